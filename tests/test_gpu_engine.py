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
from tests.helpers import check_close

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


# ------------------------------------------------------------------------------ engine outputs
# Staggered arrivals (a finished prefill merges into the RUNNING decode batch):
# (id, cached, prompt, gen, src_base, arrival_iter) - requests 3..6 arrive while decodes run.
REQS_ARR = [
    (0, 0, 300, 12, 0, 0),
    (1, 40, 129, 14, 500, 0),
    (2, 0, 17, 5, 900, 2),
    (3, 100, 64, 3, 1300, 4),
    (4, 0, 1, 9, 1700, 5),
    (5, 33, 200, 4, 2100, 7),
    (6, 16, 16, 6, 3900, 9),   # wraps around src_rows
]


def _run_logged(mux, part, reqs, *, o_f32, with_wo, **kw):
    import torch
    q, k, v = _src()
    pages = sum((r[1] + r[2] + r[3] + 15) // 16 for r in reqs) + 8
    kst = torch.full((NT, pages, Hkv, 16, D), 0x7FC0, dtype=torch.int16, device="cuda").view(torch.bfloat16)
    vst = kst.clone()
    pool = mux.Pool(NT, pages, Hkv, D, 78, kst, vst)
    rows = sum(r[2] + r[3] for r in reqs)
    o_log = torch.zeros((rows, Hq, D), dtype=torch.float32 if o_f32 else torch.bfloat16, device="cuda")
    w = synth.bf16_normal(synth.rng(9, synth.T_WO), (Hq * D, 256), std=1 / 32)
    y_log = torch.zeros((rows, 256), dtype=torch.bfloat16, device="cuda") if with_wo else None
    eng = mux.Engine(part, pool, Hq, _dev(q), _dev(k), _dev(v), scale=1 / math.sqrt(D),
                     w_o=mux.mux_outproj_pack_w(_dev(w)) if with_wo else None, max_decode_seqs=8,
                     max_prefill_tokens=600, keep_pages=True, o_log=o_log, y_log=y_log, o_f32=o_f32, **kw)
    eng.submit(reqs)
    stats = eng.run()
    torch.cuda.synchronize()
    assert stats["logged_rows"] == rows
    return eng, stats, o_log, y_log, (q, k, v), w


def _oracle_rows(reqs, out_rows, src):
    """Oracle O (float64) of every logged row: request `id`'s query at absolute position p over
    its keys 0..p, read through a page table from an oracle pool image of the request's rows."""
    q_src, k_src, v_src = src
    base = {r[0]: r[4] for r in reqs}
    L = {r[0]: r[1] + r[2] + r[3] for r in reqs}
    ref = np.zeros((len(out_rows), Hq, D))
    for rid in base:
        sel = np.nonzero(out_rows[:, 0] == rid)[0]
        if len(sel) == 0:
            continue
        rows = (base[rid] + np.arange(L[rid])) % SRC_ROWS
        npg = (L[rid] + 15) // 16
        ek, ev = oracle.empty_pool(npg, Hkv, D, poison=True)
        pids = np.random.default_rng(rid).permutation(npg).astype(np.int32)   # any page table
        oracle.append(ek, ev, k_src[rows], v_src[rows], np.array([0, L[rid]], np.int32),
                      np.array([L[rid]], np.int32), np.array([0, npg], np.int32), pids)
        pos = out_rows[sel, 1]
        qrows = q_src[(base[rid] + pos) % SRC_ROWS]
        kv_len = (pos + 1).astype(np.int32)
        pind = np.concatenate([[0], np.cumsum((kv_len + 15) // 16)]).astype(np.int32)
        ids = np.concatenate([pids[:(n + 15) // 16] for n in kv_len]).astype(np.int32)
        o, _ = oracle.attention(qrows, ek, ev, np.arange(len(sel) + 1, dtype=np.int32), kv_len, pind, ids,
                                1 / math.sqrt(D))
        ref[sel] = o
    return ref


def _check_rows_cover(reqs, out_rows):
    """every prompt row and every decode token is logged exactly once"""
    want = set()
    for rid, r, n, gen, *_ in reqs:
        want |= {(rid, r + t, 0) for t in range(n)}
        want |= {(rid, r + n + t, 1) for t in range(gen)}
    got = [tuple(int(x) for x in row) for row in out_rows]
    assert len(got) == len(set(got)) and set(got) == want


@pytest.mark.parametrize("graphs", [False, True])
def test_engine_outputs_match_oracle_staggered(mux, part, graphs):
    """f1 outputs (VERDICT r1 'next' #2): the LAST layer's attention output of every prefill row
    and every decode token, produced under the engine's growing / merged page tables with
    staggered arrivals, equals the oracle (fp32 outputs, strict R8)."""
    import torch
    eng, s, o_log, _, src, _ = _run_logged(mux, part, REQS_ARR, o_f32=True, with_wo=False, fixed_split=1,
                                           fixed_pl=2, use_graphs=graphs)
    rows = eng.out_rows()
    _check_rows_cover(REQS_ARR, rows)
    ref = _oracle_rows(REQS_ARR, rows, src)
    check_close(o_log.cpu().numpy(), ref, what=f"engine outputs graphs={graphs}")
    # arrivals: the decode batch GREW while decodes were running (a prefill merged into it)
    tr = eng.trace()
    bs = tr[tr[:, 0] == 0, 2]
    assert any(bs[i + 1] > bs[i] for i in range(1, len(bs) - 1)), bs
    assert s["ttft_max_us"] > 0 and s["gap_mean_us"] >= 0
    if graphs:
        assert s["graphs"] >= 1 and s["graph_bytes"] >= 0
    else:
        assert s["graphs"] == 0
    eng.close()


def test_engine_outproj_rows_match_oracle(mux, part):
    """with W_o: the logged bf16 attention rows are within R8's bf16 form of the oracle, and the
    logged out-projection rows equal oracle.outproj of exactly those rows (fp32 accumulate, bf16 y)."""
    eng, s, o_log, y_log, src, w = _run_logged(mux, part, REQS_ARR, o_f32=False, with_wo=True, fixed_split=0,
                                               use_graphs=True)
    import torch
    rows = eng.out_rows()
    _check_rows_cover(REQS_ARR, rows)
    o_bits = o_log.view(torch.int16).cpu().numpy().view(np.uint16)
    ref = _oracle_rows(REQS_ARR, rows, src)
    check_close(oracle.bf16_to_double(o_bits), ref, what="engine bf16 outputs", out_bf16=True)
    y_ref = oracle.outproj(o_bits.reshape(len(rows), Hq * D), w)
    y = oracle.bf16_to_double(y_log.view(torch.int16).cpu().numpy().view(np.uint16))
    check_close(y, y_ref, what="engine out-projection rows", out_bf16=True)
    eng.close()


@pytest.mark.parametrize("overlap", [False, True])
def test_engine_outputs_match_oracle_overlap(mux, part, overlap):
    """run-ahead (two decode iterations in flight) with graphs: the same oracle parity, split
    changes included (best-fit off, whole GPU once the prefills are done)."""
    eng, s, o_log, _, src, _ = _run_logged(mux, part, REQS_ARR, o_f32=True, with_wo=False, fixed_split=2,
                                           use_graphs=True, overlap=overlap)
    rows = eng.out_rows()
    _check_rows_cover(REQS_ARR, rows)
    check_close(o_log.cpu().numpy(), _oracle_rows(REQS_ARR, rows, src), what=f"engine outputs overlap={overlap}")
    eng.close()


@pytest.mark.timing
def test_engine_graphs_cut_launch_gap(mux, part):
    """f2: decode iterations as graph launches, enqueued one ahead (overlap),
    leave no host turn-around gap on the decode SMs between iterations; graph memory reported.
    Small batch / short contexts: the iteration is launch-bound, where graphs matter."""
    res = {}
    reqs = [(0, 0, 16, 40, 0, 0), (1, 0, 16, 40, 100, 0)]
    for mode in ("kernels", "graphs", "graphs+overlap"):
        eng, s, *_ = _run_logged(mux, part, reqs, o_f32=True, with_wo=False, fixed_split=1,
                                 use_graphs=mode != "kernels", overlap=mode.endswith("overlap"))
        tr = eng.trace()
        dec = tr[tr[:, 0] == 0]
        s["iter_us"] = float(np.median(dec[:, 4] - dec[:, 3])) * 1e-3
        # median interval between consecutive iteration ends (the mean also carries the few
        # iterations that first capture + instantiate a graph, ~1 ms each)
        s["tbt_median_us"] = float(np.median(np.diff(np.sort(dec[:, 4])))) * 1e-3
        res[mode] = s
        eng.close()
    for m, s in res.items():
        print(f"{m}: gap mean {s['gap_mean_us']:.1f} us max {s['gap_max_us']:.1f}, iteration {s['iter_us']:.1f} us, "
              f"tbt mean {s['tbt_mean_us']:.1f} / median {s['tbt_median_us']:.1f} us, graphs {s['graphs']} "
              f"({s['graph_bytes']} B)")
    assert res["graphs"]["graphs"] >= 1 and res["kernels"]["graphs"] == 0
    assert res["graphs+overlap"]["gap_mean_us"] < res["kernels"]["gap_mean_us"]
    assert res["graphs+overlap"]["tbt_median_us"] < res["kernels"]["tbt_median_us"]
