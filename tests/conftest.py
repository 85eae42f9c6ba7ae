import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run with -m gpu on the GPU box")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    config.addinivalue_line("markers", "timing: asserts a measured duration (skipped under a kernel profiler)")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle


def _under_profiler() -> bool:
    # ncu's injection exports these to the profiled process
    return any(k.startswith("NV_NSIGHT_INJECTION") or k in ("CUDA_INJECTION64_PATH", "NV_COMPUTE_PROFILER_PERFWORKS_DIR")
               for k in os.environ)


def pytest_collection_modifyitems(config, items):
    """Under a kernel profiler only: run the plain-stream kernel parity tests first.  ncu cannot
    prepare a kernel launched on a green context's stream (nor the fused all-reduce's rank-emulating
    grid) and ends the process there, so a launch list of `pytest -m gpu` would otherwise stop at the
    first partition test.  Without a profiler the order is pytest's own."""
    if not _under_profiler():
        return
    # timing assertions mean nothing while ncu serialises and instruments every launch
    skip_t = pytest.mark.skip(reason="timing assertion: not meaningful under a kernel profiler")
    for item in items:
        if item.get_closest_marker("timing"):
            item.add_marker(skip_t)

    def rank(item):
        name = item.nodeid
        if "test_gpu_parity.py" in name and "partition" not in name:
            return 0
        if "test_gpu_qkv.py" in name or "test_gpu_parity.py" in name:
            return 1
        return 2
    items.sort(key=rank)   # stable: pytest's order inside each group
