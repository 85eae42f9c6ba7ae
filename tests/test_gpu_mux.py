"""GPU tests of a6: green-context SM partitions and mux_run_layer (mux == isolated, bitwise;
parity with the oracle through the multiplexed path; per-side timestamps)."""
import math

import numpy as np
import pytest

import oracle
from synth import SideSpec, Shapes, make_side
from tests.helpers import check_close, gpu_build_side, oracle_build_side

pytestmark = pytest.mark.gpu


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
    p = mux.Partition(0, [16, 32, 64, 128])
    yield p
    p.close()


def test_partition_grants(mux, part):
    total = mux.mux_device_sm_count(0)
    for i, want in enumerate([16, 32, 64, 128]):
        d, p, sd, sp = part.query(i)
        assert d >= want and d % 8 == 0
        assert d + p <= total
        assert sd and sp and sd != sp
    d, p, _, _ = part.query(-1)
    assert d == p == total
    assert part.memory_bytes() >= 0


def test_stream_read_probe(mux, part):
    """The decode roofline's partition denominator (mux_stream_read): runs on a partition stream
    and on the whole GPU, more SMs read faster, bad arguments are rejected."""
    import torch
    buf = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")

    def gbs(stream, sms):
        st = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
        mux.mux_stream_read(buf, sms, st)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        n = sum(mux.mux_stream_read(buf, sms, st) for _ in range(5))
        b.record(st)
        torch.cuda.synchronize()
        return n / (a.elapsed_time(b) * 1e-3) / 1e9
    d16, _, sd16, _ = part.query(0)
    small, full = gbs(sd16, d16), gbs(None, mux.mux_device_sm_count(0))
    assert 100 < small < full, (small, full)
    assert full > 2000, full
    with pytest.raises(mux.MuxError):
        mux.mux_stream_read(buf, 0)
    with pytest.raises(mux.MuxError):
        mux.mux_stream_read(buf, 4, nbytes=1000)


def _workload(mux, Hq=8, Hkv=2, d=128):
    import torch
    pf = make_side(801, Shapes(Hq, Hkv, d, 1), SideSpec([37, 0], [300, 129]), decode=False)
    dc = make_side(802, Shapes(Hq, Hkv, d, 1), SideSpec([c - 1 for c in (700, 17, 4096)], [1, 1, 1]), decode=True)
    need = sum(pf.spec.pages_needed()) + sum(dc.spec.pages_needed())
    kst = torch.full((2, need + 8, Hkv, 16, d), 0x7FC0, dtype=torch.int16, device="cuda").view(torch.bfloat16)
    vst = kst.clone()
    pool = mux.Pool(2, need + 8, Hkv, d, 5, kst, vst)
    g_pf = gpu_build_side(mux, pf, need + 8, 5, Hkv, d, layers=2, pool=pool)
    g_dc = gpu_build_side(mux, dc, need + 8, 5, Hkv, d, layers=2, pool=pool)
    return pf, dc, pool, g_pf, g_dc


def _sides(mux, pool, g_pf, g_dc, Hq, d, pf_T, dc_B, ns=2):
    import torch
    o_pf = torch.zeros((pf_T, Hq, d), dtype=torch.float32, device="cuda")
    o_dc = torch.zeros((dc_B, Hq, d), dtype=torch.float32, device="cuda")
    wsb = mux.mux_decode_workspace_bytes(dc_B, Hq, d, ns)
    ws = torch.empty(max(16, wsb), dtype=torch.uint8, device="cuda")
    s_pf = mux.make_side(g_pf["batch"], Hq, g_pf["q"], o_pf, scale=1 / math.sqrt(d))
    s_dc = mux.make_side(g_dc["batch"], Hq, g_dc["q"], o_dc, scale=1 / math.sqrt(d), num_splits=ns, ws=ws)
    return s_pf, s_dc, o_pf, o_dc


def test_mux_equals_isolated_bitwise_and_matches_oracle(mux, part):
    import torch
    Hq, Hkv, d = 8, 2, 128
    pf, dc, pool, g_pf, g_dc = _workload(mux, Hq, Hkv, d)
    times = torch.zeros(4, dtype=torch.int64, device="cuda")
    for split in (-1, 0, 1, 2, 3):
        s_pf, s_dc, o_pf, o_dc = _sides(mux, pool, g_pf, g_dc, Hq, d, 429, 3)
        mux.mux_run_layer(part, split, pool, s_pf, s_dc, times)
        torch.cuda.synchronize()
        t = times.cpu().numpy()
        assert t[1] >= t[0] > 0 and t[3] >= t[2] > 0
        both_pf, both_dc = o_pf.cpu().numpy(), o_dc.cpu().numpy()
        s_pf, s_dc, o_pf, o_dc = _sides(mux, pool, g_pf, g_dc, Hq, d, 429, 3)
        mux.mux_run_layer(part, split, pool, s_pf, None, None)
        mux.mux_run_layer(part, split, pool, None, s_dc, None)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(both_pf, o_pf.cpu().numpy())
        np.testing.assert_array_equal(both_dc, o_dc.cpu().numpy())
    # and the multiplexed outputs match the oracle
    kimg = pool.k[0].view(torch.int16).cpu().numpy().view(np.uint16)
    vimg = pool.v[0].view(torch.int16).cpu().numpy().view(np.uint16)
    for side, g, out in ((pf, g_pf, both_pf), (dc, g_dc, both_dc)):
        ref, _ = oracle.attention(side.q, kimg, vimg, g["qo_indptr"], g["kv_len"], g["page_indptr"],
                                  g["page_ids"], 1 / math.sqrt(d))
        check_close(out, ref, what="mux output vs oracle")


def test_run_layer_multi_layer_with_append(mux, part):
    """Layer-wise prefill over 2 pool layers with append on both sides."""
    import torch
    Hq, Hkv, d = 4, 1, 64
    pf = make_side(803, Shapes(Hq, Hkv, d, 1), SideSpec([64], [128]), decode=False)
    need = sum(pf.spec.pages_needed())
    kst = torch.full((2, need + 4, Hkv, 16, d), 0x7FC0, dtype=torch.int16, device="cuda").view(torch.bfloat16)
    pool = mux.Pool(2, need + 4, Hkv, d, 9, kst, kst.clone())
    pind, pids = pool.page_tables(pf.spec.pages_needed())
    from synth import indptr
    L = pf.spec.L
    # prefix rows go in through append on both layers; the new rows are appended by run_layer
    pre = mux.Batch(indptr(pf.spec.r), pf.spec.r, [0, 4], pids[:4])
    kpre = torch.from_numpy(pf.k_cached().view(np.int16)).cuda().view(torch.bfloat16)
    vpre = torch.from_numpy(pf.v_cached().view(np.int16)).cuda().view(torch.bfloat16)
    for layer in (0, 1):
        mux.mux_append_kv(pool, layer, pre, kpre, vpre)
    batch = mux.Batch(indptr(pf.spec.n), L, pind, pids)
    q = torch.from_numpy(np.stack([pf.q, pf.q]).view(np.int16)).cuda().view(torch.bfloat16)
    kn = torch.from_numpy(np.stack([pf.k_new(), pf.k_new()]).view(np.int16)).cuda().view(torch.bfloat16)
    vn = torch.from_numpy(np.stack([pf.v_new(), pf.v_new()]).view(np.int16)).cuda().view(torch.bfloat16)
    o = torch.zeros((2, 128, Hq, d), dtype=torch.float32, device="cuda")
    s = mux.make_side(batch, Hq, q, o, k_new=kn, v_new=vn, scale=0.125, num_layers=2, append=True,
                      per_layer_inputs=True)
    mux.mux_run_layer(part, 1, pool, s, None, None)
    torch.cuda.synchronize()
    os_ = oracle_build_side(pf, need + 4, 9, Hkv, d)
    ref, _ = oracle.attention(pf.q, os_["kpool"], os_["vpool"], os_["qo_indptr"], os_["kv_len"],
                              os_["page_indptr"], os_["page_ids"], 0.125)
    for layer in (0, 1):
        check_close(o[layer].cpu().numpy(), ref, what=f"layer {layer}")


def test_run_layer_outproj_and_allreduce_hook(mux, part):
    """a7 on the multiplexed path: each layer's out-projection runs on the side's partition and
    the hook enqueues a (world-1) NCCL all-reduce of y on the same stream; y matches the
    oracle's O . W_o (on the oracle's own attention output) within the bf16 output tolerance."""
    import torch
    from paper_2504_14489_b200 import nccl
    import synth
    Hq, Hkv, d, hidden = 8, 2, 128, 384
    pf, dc, pool, g_pf, g_dc = _workload(mux, Hq, Hkv, d)
    wo_bits = synth.make_wo(801, Shapes(Hq, Hkv, d, 1, hidden=hidden))
    w_o = mux.mux_outproj_pack_w(torch.from_numpy(wo_bits.view(np.int16)).cuda().view(torch.bfloat16))
    comms = [nccl.Comm(0, 1), nccl.Comm(0, 1)]
    calls = []

    def hook_for(side, y):
        def h(s, layer, stream):
            assert s == side and stream != 0
            calls.append((s, layer))
            comms[side].all_reduce_(y, stream)
        return h
    try:
        for split in (-1, 1):
            ws = torch.empty(max(16, mux.mux_decode_workspace_bytes(3, Hq, d, 2)), dtype=torch.uint8, device="cuda")
            o_pf = torch.empty((429, Hq, d), dtype=torch.bfloat16, device="cuda")
            o_dc = torch.empty((3, Hq, d), dtype=torch.bfloat16, device="cuda")
            y_pf = torch.full((429, hidden), float("nan"), dtype=torch.float32, device="cuda")
            y_dc = torch.full((3, hidden), float("nan"), dtype=torch.float32, device="cuda")
            s_pf = mux.make_side(g_pf["batch"], Hq, g_pf["q"], o_pf, scale=1 / math.sqrt(d),
                                 w_o=w_o, y=y_pf, hook=hook_for(1, y_pf))
            s_dc = mux.make_side(g_dc["batch"], Hq, g_dc["q"], o_dc, scale=1 / math.sqrt(d), num_splits=2, ws=ws,
                                 w_o=w_o, y=y_dc, hook=hook_for(0, y_dc))
            calls.clear()
            mux.mux_run_layer(part, split, pool, s_pf, s_dc, None)
            torch.cuda.synchronize()
            assert sorted(calls) == [(0, 0), (1, 0)]
            kimg = pool.k[0].view(torch.int16).cpu().numpy().view(np.uint16)
            vimg = pool.v[0].view(torch.int16).cpu().numpy().view(np.uint16)
            for side, g, o, y in ((pf, g_pf, o_pf, y_pf), (dc, g_dc, o_dc, y_dc)):
                ref_o, _ = oracle.attention(side.q, kimg, vimg, g["qo_indptr"], g["kv_len"], g["page_indptr"],
                                            g["page_ids"], 1 / math.sqrt(d))
                # DESIGN.md R22: the out-projection consumes O in the activation dtype (bf16), so the
                # oracle's Y is bf16(O_oracle) . W_o; R8's bound then covers the GPU's O rounding flips
                o_bf16 = synth.f32_to_bf16_bits(ref_o.reshape(ref_o.shape[0], -1).astype(np.float32))
                ref_y = oracle.outproj(o_bf16, wo_bits)
                check_close(y.cpu().numpy(), ref_y, what=f"y split {split}")
                # and bitwise equal to the standalone out-proj of the side's own o
                y2 = torch.empty_like(y)
                mux.mux_outproj(o.view(o.shape[0], -1), w_o, y2)
                torch.cuda.synchronize()
                assert torch.equal(y, y2)
    finally:
        for c in comms:
            c.close()


def test_run_layer_allreduce_enqueued_from_c(mux, part):
    """a7 / §8e: libmux enqueues each layer's NCCL all-reduce of the out-projection itself
    (mux_side.ar_fn / ar_comm: the ncclAllReduce entry point + a communicator per side), on the
    side's partition stream, with no Python in the layer loop.  World 1: y is bitwise the
    standalone out-projection of the side's own attention output."""
    import torch
    from paper_2504_14489_b200 import nccl
    import synth
    Hq, Hkv, d, hidden = 8, 2, 128, 256
    pf, dc, pool, g_pf, g_dc = _workload(mux, Hq, Hkv, d)
    wo_bits = synth.make_wo(802, Shapes(Hq, Hkv, d, 1, hidden=hidden))
    w_o = mux.mux_outproj_pack_w(torch.from_numpy(wo_bits.view(np.int16)).cuda().view(torch.bfloat16))
    comms = [nccl.Comm(0, 1), nccl.Comm(0, 1)]
    try:
        for split in (-1, 0):
            ws = torch.empty(max(16, mux.mux_decode_workspace_bytes(3, Hq, d, 2)), dtype=torch.uint8, device="cuda")
            o_pf = torch.empty((429, Hq, d), dtype=torch.bfloat16, device="cuda")
            o_dc = torch.empty((3, Hq, d), dtype=torch.bfloat16, device="cuda")
            y_pf = torch.empty((429, hidden), dtype=torch.bfloat16, device="cuda")
            y_dc = torch.empty((3, hidden), dtype=torch.bfloat16, device="cuda")
            # layer 0 holds the workload's K/V (layer 1 of the pool is NaN-poisoned)
            s_pf = mux.make_side(g_pf["batch"], Hq, g_pf["q"], o_pf, scale=1 / math.sqrt(d), num_layers=1,
                                 w_o=w_o, y=y_pf, allreduce=comms[1].c_allreduce())
            s_dc = mux.make_side(g_dc["batch"], Hq, g_dc["q"], o_dc, scale=1 / math.sqrt(d), num_splits=2, ws=ws,
                                 num_layers=1, w_o=w_o, y=y_dc, allreduce=comms[0].c_allreduce())
            assert (mux.mux_side_plan(s_pf, pool.desc.num_layers)[:, 1] == 429 * hidden).all()
            mux.mux_run_layer(part, split, pool, s_pf, s_dc, None)
            torch.cuda.synchronize()
            for o, y in ((o_pf, y_pf), (o_dc, y_dc)):
                y2 = torch.empty_like(y)
                mux.mux_outproj(o.view(o.shape[0], -1), w_o, y2)
                torch.cuda.synchronize()
                assert not torch.isnan(y).any() and torch.equal(y, y2), f"split {split}"
    finally:
        for c in comms:
            c.close()


def test_run_layer_fused_allreduce_side(mux, part):
    """f4 on the multiplexed path: a side with mux_side.ar_peers runs each layer's out-projection
    and its all-reduce as ONE kernel (mux_outproj_allreduce) on the side's partition.  World 1,
    split -1 and a real split, two consecutive calls (epochs 1 and 2): y is bitwise the standalone
    out-projection of the side's own attention output."""
    import torch
    import synth
    Hq, Hkv, d, hidden = 8, 2, 128, 256
    pf, dc, pool, g_pf, g_dc = _workload(mux, Hq, Hkv, d)
    wo_bits = synth.make_wo(803, Shapes(Hq, Hkv, d, 1, hidden=hidden))
    w_o = mux.mux_outproj_pack_w(torch.from_numpy(wo_bits.view(np.int16)).cuda().view(torch.bfloat16))
    st_pf = torch.zeros(mux.mux_outproj_ar_ws_bytes(429, hidden, 1), dtype=torch.uint8, device="cuda")
    st_dc = torch.zeros(mux.mux_outproj_ar_ws_bytes(3, hidden, 1), dtype=torch.uint8, device="cuda")
    epoch = 1
    for split in (-1, 0):
        ws = torch.empty(max(16, mux.mux_decode_workspace_bytes(3, Hq, d, 2)), dtype=torch.uint8, device="cuda")
        o_pf = torch.empty((429, Hq, d), dtype=torch.bfloat16, device="cuda")
        o_dc = torch.empty((3, Hq, d), dtype=torch.bfloat16, device="cuda")
        y_pf = torch.full((429, hidden), float("nan"), dtype=torch.bfloat16, device="cuda")
        y_dc = torch.full((3, hidden), float("nan"), dtype=torch.bfloat16, device="cuda")
        s_pf = mux.make_side(g_pf["batch"], Hq, g_pf["q"], o_pf, scale=1 / math.sqrt(d), num_layers=1,
                             w_o=w_o, y=y_pf, ar_peers=(0, epoch, [st_pf], [y_pf]))
        s_dc = mux.make_side(g_dc["batch"], Hq, g_dc["q"], o_dc, scale=1 / math.sqrt(d), num_splits=2, ws=ws,
                             num_layers=1, w_o=w_o, y=y_dc, ar_peers=(0, epoch, [st_dc], [y_dc]))
        assert (mux.mux_side_plan(s_pf, pool.desc.num_layers)[:, 1] == 429 * hidden).all()
        mux.mux_run_layer(part, split, pool, s_pf, s_dc, None)
        torch.cuda.synchronize()
        epoch += 1
        for o, y, exact in ((o_pf, y_pf, True), (o_dc, y_dc, False)):
            y2 = torch.empty_like(y)
            mux.mux_outproj(o.view(o.shape[0], -1), w_o, y2)   # 3 rows: the skinny (transposed) GEMM
            torch.cuda.synchronize()
            assert not torch.isnan(y.float()).any(), f"split {split}"
            if exact:
                assert torch.equal(y.view(torch.int16), y2.view(torch.int16)), f"split {split}"
            else:   # same fp32 products, another MMA shape: within one bf16 rounding
                assert ((y.float() - y2.float()).abs() <= 2.0 ** -8 * y2.float().abs() + 1e-3).all(), f"split {split}"


def test_run_layer_fused_allreduce_multi_layer(mux, part):
    """f4 over a side of 2 layers with per-layer o / y (y_stride): each layer's out-projection +
    all-reduce is its own fused launch on automatic epochs (three consecutive mux_run_layer calls
    on one workspace); every layer's y is bitwise the standalone out-projection of that layer's o."""
    import torch
    import synth
    from synth import indptr
    Hq, Hkv, d, hidden = 4, 1, 64, 256
    pf = make_side(804, Shapes(Hq, Hkv, d, 1), SideSpec([64], [200]), decode=False)
    need = sum(pf.spec.pages_needed())
    kst = torch.full((2, need + 4, Hkv, 16, d), 0x7FC0, dtype=torch.int16, device="cuda").view(torch.bfloat16)
    pool = mux.Pool(2, need + 4, Hkv, d, 9, kst, kst.clone())
    pind, pids = pool.page_tables(pf.spec.pages_needed())
    pre = mux.Batch(indptr(pf.spec.r), pf.spec.r, [0, 4], pids[:4])
    kpre = torch.from_numpy(pf.k_cached().view(np.int16)).cuda().view(torch.bfloat16)
    vpre = torch.from_numpy(pf.v_cached().view(np.int16)).cuda().view(torch.bfloat16)
    for layer in (0, 1):
        mux.mux_append_kv(pool, layer, pre, kpre, vpre)
    batch = mux.Batch(indptr(pf.spec.n), pf.spec.L, pind, pids)
    T = pf.spec.total_new
    q = torch.from_numpy(np.stack([pf.q, pf.q]).view(np.int16)).cuda().view(torch.bfloat16)
    kn = torch.from_numpy(np.stack([pf.k_new(), pf.k_new()]).view(np.int16)).cuda().view(torch.bfloat16)
    vn = torch.from_numpy(np.stack([pf.v_new(), pf.v_new()]).view(np.int16)).cuda().view(torch.bfloat16)
    wo_bits = synth.make_wo(805, Shapes(Hq, Hkv, d, 1, hidden=hidden))
    w_o = mux.mux_outproj_pack_w(torch.from_numpy(wo_bits.view(np.int16)).cuda().view(torch.bfloat16))
    stage = torch.zeros(mux.mux_outproj_ar_ws_bytes(T, hidden, 1), dtype=torch.uint8, device="cuda")
    for call in range(3):
        o = torch.zeros((2, T, Hq, d), dtype=torch.bfloat16, device="cuda")
        y = torch.full((2, T, hidden), float("nan"), dtype=torch.bfloat16, device="cuda")
        s = mux.make_side(batch, Hq, q, o, k_new=kn, v_new=vn, scale=0.125, num_layers=2, append=True,
                          per_layer_inputs=True, w_o=w_o, y=y, ar_peers=(0, 0, [stage], [y]))
        mux.mux_run_layer(part, 1 if call % 2 else -1, pool, s, None, None)
        torch.cuda.synchronize()
        for layer in (0, 1):
            y2 = torch.empty((T, hidden), dtype=torch.bfloat16, device="cuda")
            mux.mux_outproj(o[layer].view(T, -1), w_o, y2)
            torch.cuda.synchronize()
            assert not torch.isnan(y[layer].float()).any(), f"call {call} layer {layer}"
            assert torch.equal(y[layer].view(torch.int16), y2.view(torch.int16)), f"call {call} layer {layer}"


def test_prefill_on_partition_stream_sizes_its_grid(mux, part):
    """mux_prefill_attn called directly on a green-context stream (no SM count in its signature) must
    size the persistent prefill grid to that context's SMs, exactly as mux_run_layer does with the
    partition it knows: the cfg2 prefill (one 8k causal sequence, 32 q / 8 kv heads) on the prefill side
    of the 32-SM decode split gives the same bits both ways, and the direct call is not slower than the
    run_layer one (a grid sized for the whole device would run two waves of persistent CTAs, ~1.5x)."""
    import torch
    from synth import indptr
    Hq, Hkv, d, L = 32, 8, 128, 8192
    pages = L // 16 + 4
    kst = torch.zeros((1, pages, Hkv, 16, d), dtype=torch.bfloat16, device="cuda")
    pool = mux.Pool(1, pages, Hkv, d, 5, kst, kst.clone())
    ppi, ppd = pool.page_tables([L // 16])
    gen = torch.Generator(device="cuda").manual_seed(3)
    k = torch.randn((L, Hkv, d), generator=gen, device="cuda").bfloat16()
    v = torch.randn((L, Hkv, d), generator=gen, device="cuda").bfloat16()
    q = torch.randn((L, Hq, d), generator=gen, device="cuda").bfloat16()
    batch = mux.Batch(indptr([L]), [L], ppi, ppd)
    mux.mux_append_kv(pool, 0, batch, k, v)
    scale = 1 / math.sqrt(d)
    split = 1                                  # decode 32 SMs / prefill the rest
    _, psms, _, sp = part.query(split)
    o_run = torch.empty((L, Hq, d), dtype=torch.bfloat16, device="cuda")
    o_dir = torch.empty_like(o_run)
    side = mux.make_side(batch, Hq, q, o_run, scale=scale)
    st = torch.cuda.ExternalStream(sp)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def timed(fn, a, b, stream, reps=5):
        fn()
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    cur = torch.cuda.current_stream()
    t_run = timed(lambda: mux.mux_run_layer(part, split, pool, side, None, None), ev[0], ev[1], cur)
    t_dir = timed(lambda: mux.mux_prefill_attn(pool, 0, batch, Hq, q, o_dir, None, scale=scale, stream=sp),
                  ev[2], ev[3], st)
    assert torch.equal(o_run.view(torch.int16), o_dir.view(torch.int16))
    assert pool.error_flags() == 0
    assert t_dir < 1.15 * t_run, f"direct {t_dir:.3f} ms vs run_layer {t_run:.3f} ms on {psms} SMs"
