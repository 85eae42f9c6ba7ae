"""Host logic of the profiler accommodations (tests/conftest.py, __graft_entry__.smoke): ncu's
injection environment is detected, and under it the plain-stream parity tests run first and timing
assertions are skipped; without it pytest's order stands (profiles/r02_summary.md, r02l / r02m)."""
import os

from tests import conftest

_KEYS = ("CUDA_INJECTION64_PATH", "NV_COMPUTE_PROFILER_PERFWORKS_DIR")


def _clear(monkeypatch):
    for k in list(os.environ):
        if k.startswith("NV_NSIGHT_INJECTION") or k in _KEYS:
            monkeypatch.delenv(k)


class _Item:
    def __init__(self, nodeid, timing=False):
        self.nodeid, self.timing, self.marks = nodeid, timing, []

    def get_closest_marker(self, name):
        return object() if (name == "timing" and self.timing) else None

    def add_marker(self, m):
        self.marks.append(m)


def _items():
    return [_Item("tests/test_gpu_engine.py::test_engine_graphs_cut_launch_gap", timing=True),
            _Item("tests/test_gpu_parity.py::test_prefill_persistent_on_partition[a]"),
            _Item("tests/test_gpu_mux.py::test_mux_equals_iso"),
            _Item("tests/test_gpu_parity.py::test_decode_parity[0-1]"),
            _Item("tests/test_gpu_qkv.py::test_qkv"),
            _Item("tests/test_gpu_parity.py::test_prefill_parity[0]")]


def test_profiler_environment_detected(monkeypatch):
    _clear(monkeypatch)
    assert not conftest._under_profiler()
    monkeypatch.setenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE", "uds")
    assert conftest._under_profiler()
    _clear(monkeypatch)
    monkeypatch.setenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR", "/x")
    assert conftest._under_profiler()


def test_order_and_skips_only_under_profiler(monkeypatch):
    _clear(monkeypatch)
    items = _items()
    before = [i.nodeid for i in items]
    conftest.pytest_collection_modifyitems(None, items)
    assert [i.nodeid for i in items] == before and not any(i.marks for i in items)

    monkeypatch.setenv("NV_NSIGHT_INJECTION_PORT_BASE", "49152")
    items = _items()
    conftest.pytest_collection_modifyitems(None, items)
    ids = [i.nodeid.split("::")[1] for i in items]
    assert ids == ["test_decode_parity[0-1]", "test_prefill_parity[0]",                 # plain-stream parity
                   "test_prefill_persistent_on_partition[a]", "test_qkv",              # partition / qkv
                   "test_engine_graphs_cut_launch_gap", "test_mux_equals_iso"]        # the rest, in order
    assert [bool(i.marks) for i in items] == [False, False, False, False, True, False]
