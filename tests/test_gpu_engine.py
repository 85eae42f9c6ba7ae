"""GPU tests of the f1 multiplex engine (include/mux.h "ENGINE"): a small request trace runs
through layer-wise prefill groups and decode iterations on SM partitions; afterwards every
request's KV pages in EVERY layer must hold exactly its tokens' rows (the engine's page
accounting, decode page growth and appends, checked byte for byte against oracle.append on the
same page table), token accounting must add up, and the device-clock statistics must be sane."""
import math

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

Hq, Hkv, D, NT = 8, 2, 128, 4
SRC_ROWS = 4096
REQS = [  # (id, cached r, prompt n, gen, src_base)
    (0, 0, 300, 6, 0),
    (1, 40, 129, 9, 500),
    (2, 0, 17, 3, 900),
    (3, 100, 64, 0, 1300),
    (4, 0, 1, 20, 1700),
    (5, 33, 500, 4, 2100),
    (6, 16, 16, 17, 3900),   # wraps around src_rows
]


@pytest.fixture(scope="module")
def mux():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2504_14489_b200 as m
    m.lib()
    return m


@pytest.fixture(scope="module")
def part(mux):
    p = mux.Partition(0, [16, 32, 64])
    yield p
    p.close()


def _src():
    g = synth.rng(9, synth.T_Q_PF)
    q = synth.bf16_normal(g, (SRC_ROWS, Hq, D))
    k = synth.bf16_normal(g, (SRC_ROWS, Hkv, D))
    v = synth.bf16_normal(g, (SRC_ROWS, Hkv, D))
    return q, k, v


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)


def _run(mux, part, **kw):
    import torch
    q, k, v = _src()
    pages = sum((r + n + gen + 15) // 16 for _, r, n, gen, _ in REQS) + 8
    kst = torch.full((NT, pages, Hkv, 16, D), 0x7FC0, dtype=torch.int16, device="cuda").view(torch.bfloat16)
    vst = kst.clone()
    pool = mux.Pool(NT, pages, Hkv, D, 77, kst, vst)
    w = synth.bf16_normal(synth.rng(9, synth.T_WO), (Hq * D, 256), std=1 / 32)
    eng = mux.Engine(part, pool, Hq, _dev(q), _dev(k), _dev(v), scale=1 / math.sqrt(D),
                     w_o=mux.mux_outproj_pack_w(_dev(w)), max_decode_seqs=8, max_prefill_tokens=600,
                     keep_pages=True, **kw)
    eng.submit(REQS)
    stats = eng.run()
    torch.cuda.synchronize()
    return eng, pool, stats, (k, v)


def _check_pool(eng, pool, src):
    import torch
    k_src, v_src = src
    for rid, r, n, gen, base in REQS:
        kv_len, pids = eng.request_pages(rid)
        assert kv_len == r + n + gen
        assert len(pids) == (kv_len + 15) // 16
        rows = (base + np.arange(kv_len)) % SRC_ROWS
        ek, ev = oracle.empty_pool(len(pids), Hkv, D, poison=True)
        oracle.append(ek, ev, k_src[rows], v_src[rows], np.array([0, kv_len], np.int32), np.array([kv_len], np.int32),
                      np.array([0, len(pids)], np.int32), np.arange(len(pids), dtype=np.int32))
        for layer in range(NT):
            gk = pool.k[layer][torch.tensor(pids, device="cuda")].view(torch.int16).cpu().numpy().view(np.uint16)
            gv = pool.v[layer][torch.tensor(pids, device="cuda")].view(torch.int16).cpu().numpy().view(np.uint16)
            # slots past kv_len in the last page are never written (poison on both sides)
            np.testing.assert_array_equal(gk, ek, err_msg=f"request {rid} layer {layer} K")
            np.testing.assert_array_equal(gv, ev, err_msg=f"request {rid} layer {layer} V")


def _check_stats(s):
    assert s["prefill_tokens"] == sum(n for _, _, n, _, _ in REQS)
    assert s["decode_tokens"] == sum(g for _, _, _, g, _ in REQS)
    assert s["decode_iters"] >= max(g for _, _, _, g, _ in REQS)
    assert 0.0 <= s["bubble_ratio"] <= 1.0
    assert s["makespan_us"] > 0 and s["ttft_max_us"] <= s["makespan_us"] + 1
    assert s["busy_dec_us"] > 0 and s["busy_pf_us"] > 0


def test_engine_fixed_split_groups(mux, part):
    eng, pool, s, src = _run(mux, part, fixed_split=1, fixed_pl=2)
    _check_stats(s)
    # 2-layer groups: every prefill batch takes NT/2 groups
    assert s["prefill_groups"] % (NT // 2) == 0
    tr = eng.trace()
    assert ((tr[:, 0] == 0) | (tr[:, 0] == 1)).all()
    assert (tr[:, 4] >= tr[:, 3]).all()
    _check_pool(eng, pool, src)
    eng.close()


def test_engine_best_fit_and_npl(mux, part):
    """Best-fit split + N_PL from a (synthetic) cost model: the decode side needs the 32-SM
    split for the SLO, prefill is 4x slower per layer than decode -> N_PL = 1 layer groups."""
    from paper_2504_14489_b200 import costmodel as cm
    dec, pf = {}, {}
    for i in range(3):
        ds, ps, _, _ = part.query(i)
        dec[ds] = cm.Fit(np.array([0.0, 0.0, 400.0 / (ds / 16)]), 0, 0, 1)   # us per layer
        pf[ps] = cm.Fit(np.array([0.0, 0.0, 0.0, 4 * 400.0]), 0, 0, 1)
    model = cm.CostModel(pf, dec, {ds: 1.0 for ds in dec})
    slo = 300.0 * NT  # 16 SMs: 400 us/layer fails, 32 SMs: 200 passes
    eng, pool, s, src = _run(mux, part, fixed_split=-2, cost=model, tbt_slo_us=slo)
    _check_stats(s)
    tr = eng.trace()
    dec_splits = set(tr[tr[:, 0] == 0, 1].tolist())
    # split 1 while a prefill runs, the whole GPU (-1) once no prefill work is left (R24)
    assert 1 in dec_splits and dec_splits <= {1, -1}, dec_splits
    _check_pool(eng, pool, src)
    eng.close()


@pytest.mark.parametrize("serialize", [False, True])
def test_engine_unpartitioned_and_time_sliced(mux, part, serialize):
    """fixed_split = -1: both sides on whole-GPU streams (unpartitioned), or on one stream
    (serialize: the temporal-multiplexing baseline)."""
    eng, pool, s, src = _run(mux, part, fixed_split=-1, serialize=serialize)
    _check_stats(s)
    _check_pool(eng, pool, src)
    eng.close()
