"""CPU tests of the C-ABI library: it loads on a GPU-less host, exports every symbol
include/mux.h declares, and its host logic (allocator, split rule, N_PL, validation) matches
the oracle allocator and the paper's printed values.  No compute calls."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

from oracle.alloc import OraclePagePool, seeded_permutation

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mux():
    from paper_2504_14489_b200 import build as b
    b.build()
    import paper_2504_14489_b200 as m
    m.lib()
    return m


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mux.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mux_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(mux):
    syms = declared_symbols()
    assert len(syms) >= 25
    L = mux.lib()
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    out = os.popen(f"nm -D --defined-only {os.path.join(ROOT, 'paper_2504_14489_b200', 'libmux.so')}").read()
    exported = set(re.findall(r" T (mux_\w+)", out))
    assert set(syms) <= exported
    # only the ABI is exported (hidden visibility for internals)
    assert all(s.startswith("mux_") for s in exported)


def test_no_link_time_libcuda_dependency(mux):
    out = os.popen(f"ldd {os.path.join(ROOT, 'paper_2504_14489_b200', 'libmux.so')}").read()
    assert "libcuda.so" not in out


def _fake_pool(mux, num_pages, seed, hkv=1, d=64, layers=1):
    # fake (aligned) device pointers: allocator calls never touch storage
    return mux.binding.Pool(layers, num_pages, hkv, d, seed, device_ptrs=(0x100000, 0x200000))


def test_allocator_matches_oracle_allocator(mux):
    for n, seed in [(1, 0), (10, 42), (1000, 2504_14489), (16896, 7)]:
        p = _fake_pool(mux, n, seed)
        assert p.free_list() == seeded_permutation(n, seed)
        p.close()


def test_allocator_sequence_matches_oracle(mux):
    g = np.random.default_rng(1)
    p = _fake_pool(mux, 64, 9)
    o = OraclePagePool(64, 9)
    live = []
    for step in range(1500):
        op = int(g.integers(0, 3))
        if op == 0:
            n = int(g.integers(0, 9))
            if n > o.num_free():
                with pytest.raises(mux.MuxError) as e:
                    p.alloc(n)
                assert e.value.code == 3  # MUX_ERR_POOL_EXHAUSTED
                continue
            got = p.alloc(n)
            assert got == o.alloc(n)
            live.append(got)
        elif op == 1 and live:
            ids = live[int(g.integers(0, len(live)))]
            p.share(ids)
            o.share(ids)
            live.append(list(ids))
        elif live:
            ids = live.pop(int(g.integers(0, len(live))))
            p.free(ids)
            o.release(ids)
        assert p.num_free() == o.num_free()
    assert p.free_list() == list(o.free)
    for pg in range(64):
        assert p.refcount(pg) == o.ref[pg]


def test_allocator_rejects_bad_ids(mux):
    p = _fake_pool(mux, 8, 1)
    with pytest.raises(mux.MuxError):
        p.free([3])          # not allocated
    with pytest.raises(mux.MuxError):
        p.share([99])        # out of range


def test_pool_create_validation(mux):
    for kw, code in [(dict(d=96), 2), (dict(d=64, hkv=0), 1)]:
        with pytest.raises(mux.MuxError) as e:
            _fake_pool(mux, 8, 1, **kw)
        assert e.value.code == code
    desc = mux.binding.PoolDesc(1, 8, 32, 1, 64, 0x1000, 0x2000, 0)   # page size 32
    h = ctypes.c_void_p()
    assert mux.lib().mux_pool_create(ctypes.byref(h), ctypes.byref(desc)) == 2


def test_partition_config_rule_matches_paper(mux):
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_pins.json")))
    for e in gold["partition_config_counts"]:
        cfgs = mux.mux_partition_configs(e["total_sms"], e["granularity"], 12)
        assert len(cfgs) == e["count"], e["cite"]
        assert cfgs == [16 * (i + 1) for i in range(e["count"])]
    assert mux.mux_partition_configs(148) == [16, 32, 48, 64, 80, 96, 112, 128]
    assert mux.mux_partition_configs(32) == [16]
    with pytest.raises(mux.MuxError):
        mux.mux_partition_configs(20)


def test_n_pl_matches_paper_formula(mux):
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_pins.json")))
    for e in gold["n_pl"]:
        assert mux.mux_num_prefill_layers(e["T_d"], e["T_P"], e["N_T"], 10**6) == e["expect"], e["cite"]
    assert mux.mux_num_prefill_layers(30.0, 600.0, 80, 3) == 3     # clamped to remaining
    assert mux.mux_num_prefill_layers(30.0, 600.0, 80, 0) == 0


def test_decode_split_heuristic_and_workspace(mux):
    # launch-simulation choice (include/mux.h): uniform batches that already fill the SMs
    # stay unsplit; one long sequence spreads over the SMs; a ragged batch splits finer than a
    # uniform one of the same size; the count is capped at 64
    f = mux.mux_decode_num_splits
    assert f(64, 8, 4096, 32, [4096] * 64) == 1
    assert f(64, 8, 4096, 16, [4096] * 64) == 1
    assert f(1, 8, 4096, 32, [4096]) == 32
    assert f(1, 1, 16, 148) == 1
    assert f(1, 1, 1 << 20, 148) == 64
    ragged = [1024 + (i * 997) % 7168 for i in range(48)]
    assert f(48, 8, max(ragged), 32, ragged) > f(48, 8, max(ragged), 32, [max(ragged)] * 48)
    assert mux.mux_decode_workspace_bytes(64, 32, 128, 1) == 0
    assert mux.mux_decode_workspace_bytes(2, 4, 64, 3) >= 2 * 4 * 3 * (64 + 2) * 4


def test_version_and_error_string(mux):
    assert b"sm_100a" in mux.lib().mux_version()
    mux.lib().mux_pool_destroy(None)
    with pytest.raises(mux.MuxError):
        _fake_pool(mux, 8, 1, d=96)
    assert "head_dim" in mux.last_error()


def test_header_is_plain_c_and_cxx(tmp_path):
    """include/mux.h is a C ABI: it must compile as strict C99 and as C++11 (no torch or C++-only
    types), including the structs a caller fills (mux_side, mux_ar_peers, mux_batch)."""
    import shutil
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = ("#include \"mux.h\"\n"
           "int main(void) { mux_side s; mux_ar_peers p; mux_batch b; (void)s; (void)p; (void)b;\n"
           "  return mux_outproj_ar_ws_bytes(256, 256, 2) == 0; }\n")
    for comp, std, ext in (("gcc", "-std=c99", "c"), ("g++", "-std=c++11", "cpp")):
        if not shutil.which(comp):
            pytest.skip(f"{comp} not found")
        f = tmp_path / f"t.{ext}"
        f.write_text(src)
        r = subprocess.run([comp, std, "-Wall", "-Wextra", "-pedantic", "-Werror", "-fsyntax-only",
                            "-I", os.path.join(root, "include"), str(f)], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
