"""GPU parity of f4's fused out-projection GEMM + all-reduce (include/mux.h mux_outproj_allreduce,
DESIGN.md R23): with G ranks, every rank's Y must equal the all-reduce of the G partial sums
X_r . W_r, i.e. the unsharded product (oracle.outproj over the concatenated shards, float64: the
block identity of R23), within the rounding the wire type adds (each partial is rounded to bf16,
the fp32 sum once more).  Fewer GPUs than ranks: the G ranks' CTAs run in ONE launch on this
device (mux_outproj_allreduce_emulated), which exercises the same peer-store / counter protocol.
Also: every rank's Y is bitwise identical, bitwise equal to the composition of mux_outproj
(bf16 partials) and an fp32 rank-order sum, and unchanged across launches (epoch counters)."""
import math

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mux():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2504_14489_b200 as m
    m.lib()
    return m


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)


def _f64(t):
    import torch
    return t.float().cpu().numpy().astype(np.float64)


def _shards(G, T, K, N, seed):
    g = synth.rng(seed, synth.T_WO, salt=G * 1000 + K)
    xs = [synth.bf16_normal(g, (T, K)) for _ in range(G)]
    ws = [synth.bf16_normal(g, (K, N), std=1 / math.sqrt(G * K)) for _ in range(G)]
    return xs, ws


def _run(mux, G, T, K, N, epochs=2):
    import torch
    xs_h, ws_h = _shards(G, T, K, N, 7)
    xs = [_dev(x) for x in xs_h]
    ws = [mux.mux_outproj_pack_w(_dev(w)) for w in ws_h]
    wsb = mux.mux_outproj_ar_ws_bytes(T, N, G)
    stages = [torch.zeros(wsb, dtype=torch.uint8, device="cuda") for _ in range(G)]
    outs = []
    for e in range(1, epochs + 1):
        ys = [torch.full((T, N), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(G)]
        mux.mux_outproj_allreduce_emulated(xs, ws, e, stages, ys)
        torch.cuda.synchronize()
        outs.append(ys)
    return xs_h, ws_h, xs, ws, outs


@pytest.mark.parametrize("G,T,K,N", [
    (1, 300, 200, 264),      # one rank: the GEMM alone; row / column / K tails
    (2, 300, 200, 264),
    (3, 520, 136, 776),      # a world that does not divide the tile count
    (4, 1024, 512, 1024),
    (8, 640, 128, 1032),     # TP-8: more ranks than tiles of some owners
    (8, 64, 1024, 1024),     # a decode side's rows (one partial M tile), 70B TP-8 out-projection K
])
def test_fused_allreduce_matches_oracle(mux, G, T, K, N):
    import torch
    xs_h, ws_h, xs, ws, outs = _run(mux, G, T, K, N)
    ys = outs[0]
    # every rank holds the same bits, and a second launch (epoch 2) reproduces them
    y0 = ys[0].view(torch.int16)
    for r in range(1, G):
        assert torch.equal(ys[r].view(torch.int16), y0), f"rank {r} differs from rank 0"
    for r in range(G):
        assert torch.equal(outs[1][r].view(torch.int16), y0), f"epoch 2, rank {r} differs"
    # the oracle: the unsharded product (block identity, R23) in float64
    ref = oracle.outproj(np.concatenate(xs_h, axis=1), np.concatenate(ws_h, axis=0))
    parts = [oracle.outproj(xs_h[r], ws_h[r]) for r in range(G)]
    bound = 2.0 ** -8 * (sum(np.abs(p) for p in parts) + np.abs(ref)) + 1e-4
    got = _f64(ys[0])
    d = np.abs(got - ref)
    bad = ~(d <= bound)
    assert not bad.any(), f"{bad.sum()} of {d.size} elements off, max|d| {np.nanmax(d):.3e}"
    # composition: bf16 partials of mux_outproj, summed in fp32 in rank order, rounded once
    acc = None
    for r in range(G):
        p = torch.empty((T, N), dtype=torch.bfloat16, device="cuda")
        mux.mux_outproj(xs[r], ws[r], p)
        acc = p.float() if acc is None else acc + p.float()
    torch.cuda.synchronize()
    assert torch.equal(acc.bfloat16().view(torch.int16), y0), "fused result != bf16 partials summed in rank order"


def test_fused_allreduce_single_rank_production_path(mux):
    """world 1 through the per-rank entry point (the one a multi-GPU rank calls): Y == the bf16 GEMM."""
    import torch
    T, K, N = 384, 256, 512
    xs_h, ws_h = _shards(1, T, K, N, 9)
    x = _dev(xs_h[0])
    w = mux.mux_outproj_pack_w(_dev(ws_h[0]))
    stage = torch.zeros(mux.mux_outproj_ar_ws_bytes(T, N, 1), dtype=torch.uint8, device="cuda")
    y = torch.empty((T, N), dtype=torch.bfloat16, device="cuda")
    ref = torch.empty_like(y)
    for e in (1, 2, 3):
        mux.mux_outproj_allreduce(x, w, 0, e, [stage], [y])
        mux.mux_outproj(x, w, ref)
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int16), ref.view(torch.int16))


def test_fused_allreduce_automatic_epochs(mux):
    """epoch 0: each rank's kernel keeps its own launch counter in the workspace (what repeated
    mux_run_layer calls and CUDA-graph replays use); four launches give the same bits as the
    explicit-epoch run."""
    import torch
    G, T, K, N = 4, 700, 256, 520
    xs_h, ws_h, xs, ws, outs = _run(mux, G, T, K, N, epochs=1)
    wsb = mux.mux_outproj_ar_ws_bytes(T, N, G)
    stages = [torch.zeros(wsb, dtype=torch.uint8, device="cuda") for _ in range(G)]
    for it in range(4):
        ys = [torch.full((T, N), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(G)]
        mux.mux_outproj_allreduce_emulated(xs, ws, 0, stages, ys)
        torch.cuda.synchronize()
        for r in range(G):
            assert torch.equal(ys[r].view(torch.int16), outs[0][0].view(torch.int16)), f"launch {it}, rank {r}"


def test_fused_allreduce_rejects_bad_args(mux):
    import torch
    x = torch.zeros((256, 64), dtype=torch.bfloat16, device="cuda")
    w = mux.mux_outproj_pack_w(torch.zeros((64, 64), dtype=torch.bfloat16, device="cuda"))
    st = torch.zeros(mux.mux_outproj_ar_ws_bytes(256, 64, 1), dtype=torch.uint8, device="cuda")
    y = torch.empty((256, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(mux.MuxError):
        mux.mux_outproj_allreduce(x, w, 1, 1, [st], [y])          # rank outside the world


def test_fused_allreduce_cfg4_full_size(mux):
    """BASELINE cfg4 (Llama-3-70B, KV-head sharded over 8 GPUs, P:686 / P:701-702): each rank's
    out-projection of the 8192-token prefill, X [8192][Hq/8 * 128 = 1024] . W_o shard [1024][8192],
    all-reduced over 8 emulated ranks.  Every rank's Y is bitwise the composition (bf16 GEMM partials
    summed in rank order); 64 rows spread over the tiles (first / last row, tile boundaries) match the
    float64 unsharded product within the wire-type bound."""
    import torch
    G, T, K, N = 8, 8192, 1024, 8192
    g = synth.rng(4, synth.T_WO, salt=88)
    xs = [torch.from_numpy(synth.bf16_normal(g, (T, K)).view(np.int16)).cuda().view(torch.bfloat16) for _ in range(G)]
    ws_h = [synth.bf16_normal(g, (K, N), std=1 / math.sqrt(G * K)) for _ in range(G)]
    ws = [mux.mux_outproj_pack_w(_dev(w)) for w in ws_h]
    wsb = mux.mux_outproj_ar_ws_bytes(T, N, G)
    stages = [torch.zeros(wsb, dtype=torch.uint8, device="cuda") for _ in range(G)]
    ys = [torch.empty((T, N), dtype=torch.bfloat16, device="cuda") for _ in range(G)]
    mux.mux_outproj_allreduce_emulated(xs, ws, 0, stages, ys)
    acc = None
    for r in range(G):
        p = torch.empty((T, N), dtype=torch.bfloat16, device="cuda")
        mux.mux_outproj(xs[r], ws[r], p)
        acc = p.float() if acc is None else acc + p.float()
    torch.cuda.synchronize()
    comp = acc.bfloat16().view(torch.int16)
    for r in range(G):
        assert torch.equal(ys[r].view(torch.int16), comp), f"rank {r}"
    rows = synth.sample_rows(T, 64, tile=256)
    idx = torch.from_numpy(rows.astype(np.int64)).cuda()
    xs_h = [x[idx].view(torch.int16).cpu().numpy().view(np.uint16) for x in xs]
    ref = oracle.outproj(np.concatenate(xs_h, axis=1), np.concatenate(ws_h, axis=0))
    parts = [oracle.outproj(xs_h[r], ws_h[r]) for r in range(G)]
    bound = 2.0 ** -8 * (sum(np.abs(p) for p in parts) + np.abs(ref)) + 1e-4
    d = np.abs(_f64(ys[3][idx]) - ref)
    assert (d <= bound).all(), f"max|d| {d.max():.3e}"
