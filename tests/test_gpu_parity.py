"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded bf16
inputs.  Integer/byte results bit-exact; attention within DESIGN.md R8's tolerance
(max-abs 2e-3 / rel 1e-2, BASELINE.json north_star)."""
import math

import numpy as np
import pytest

import oracle
import synth
from synth import SideData, SideSpec, Shapes, make_side
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


def _run(mux, side, Hq, Hkv, d, decode, num_pages=None, seed=11, o_f32=True, num_splits=0, scale=None):
    import torch
    need = sum(side.spec.pages_needed())
    num_pages = num_pages or need + 7
    gs = gpu_build_side(mux, side, num_pages, seed, Hkv, d)
    os_ = oracle_build_side(side, num_pages, seed, Hkv, d)
    # integer page tables: library allocator == oracle allocator (bit-exact)
    np.testing.assert_array_equal(gs["page_ids"], os_["page_ids"])
    np.testing.assert_array_equal(gs["page_indptr"], os_["page_indptr"])
    # pool image after append: byte-exact, including the untouched NaN-poisoned slots
    torch.cuda.synchronize()
    kimg = gs["pool"].k[0].view(torch.int16).cpu().numpy().view(np.uint16)
    vimg = gs["pool"].v[0].view(torch.int16).cpu().numpy().view(np.uint16)
    np.testing.assert_array_equal(kimg, os_["kpool"])
    np.testing.assert_array_equal(vimg, os_["vpool"])
    scale = scale if scale is not None else 1.0 / math.sqrt(d)
    T = side.spec.total_new
    o = torch.empty((T, Hq, d), dtype=torch.float32 if o_f32 else torch.bfloat16, device="cuda")
    lse = torch.empty((T, Hq), dtype=torch.float32, device="cuda")
    if decode:
        ns = num_splits or mux.mux_decode_num_splits(side.spec.num_seqs, Hkv, max(side.spec.L), 148, side.spec.L, d)
        wsb = mux.mux_decode_workspace_bytes(side.spec.num_seqs, Hq, d, ns)
        ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
        mux.mux_decode_attn(gs["pool"], 0, gs["batch"], Hq, gs["q"], o, lse, scale=scale, num_splits=ns, ws=ws)
    else:
        mux.mux_prefill_attn(gs["pool"], 0, gs["batch"], Hq, gs["q"], o, lse, scale=scale)
    torch.cuda.synchronize()
    ref, ref_lse = oracle.attention(side.q, os_["kpool"], os_["vpool"], os_["qo_indptr"], os_["kv_len"],
                                    os_["page_indptr"], os_["page_ids"], scale)
    return o.float().cpu().numpy(), lse.cpu().numpy(), ref, ref_lse, gs


def _side(cfg_salt, spec, Hq, Hkv, d, decode=False, outliers=False):
    return make_side(700 + cfg_salt, Shapes(Hq, Hkv, d, 1), spec, decode=decode, outliers=outliers)


# ----------------------------------------------------------------------------- append (a1+a2)
def test_append_and_page_tables_bitexact(mux):
    side = _side(1, SideSpec([0, 5, 40], [33, 17, 1]), 8, 2, 128)
    _run(mux, side, 8, 2, 128, decode=False)


def test_shared_page_write_rejected(mux):
    import torch
    side = _side(2, SideSpec([0], [40]), 4, 1, 64)
    gs = gpu_build_side(mux, side, 16, 3, 1, 64)
    ids = [int(x) for x in gs["page_ids"]]
    gs["pool"].share(ids[:2])
    k = torch.zeros((1, 1, 64), dtype=torch.bfloat16, device="cuda")
    b = mux.Batch([0, 1], [20], [0, 2], ids[:2])
    with pytest.raises(mux.MuxError) as e:
        mux.mux_append_kv(gs["pool"], 0, b, k, k)
    assert e.value.code == 4


# ----------------------------------------------------------------------------- decode (a4+a5)
DECODE_CASES = [
    # (d, Hq, Hkv, contexts)
    (64, 4, 1, [256, 256, 256, 256]),                  # cfg1 decode shape
    (128, 32, 8, [1, 15, 16, 17, 100, 257, 1000]),     # ragged, Llama-8B heads
    (128, 64, 8, [33, 4096]),                          # g = 8 (70B)
    (64, 16, 1, [129, 48]),                            # g = 16 (two N tiles)
    (128, 8, 8, [513]),                                # MHA g = 1
    (128, 4, 1, [3000, 17]),                           # one kv head: 8 warps share its pages (16-stage ring)
    (64, 8, 2, [2100]),                                # g = 4, two kv heads per CTA
    (128, 16, 8, [700, 1]),                            # g = 2
    (128, 8, 4, [1000, 5, 64]),                        # Hkv = 4 (2-GPU shard of Llama-8B), g = 2: HG = 4
    (128, 32, 4, [4096, 33]),                          # Hkv = 4 (2-GPU shard of Llama-70B), g = 8: HG = 4
    (128, 12, 6, [600, 17]),                           # Hkv = 6: HG = 2 (largest power of two dividing 6)
    (64, 24, 6, [300]),                                # Hkv = 6, g = 4, d64
    (128, 9, 3, [200, 31]),                            # Hkv = 3, g = 3: HG = 1
]


@pytest.mark.parametrize("splits", [1, 3, 7, 0])
@pytest.mark.parametrize("case", range(len(DECODE_CASES)))
def test_decode_parity(mux, case, splits):
    d, Hq, Hkv, ctx = DECODE_CASES[case]
    side = _side(10 + case, SideSpec([c - 1 for c in ctx], [1] * len(ctx)), Hq, Hkv, d, decode=True)
    o, lse, ref, ref_lse, _ = _run(mux, side, Hq, Hkv, d, decode=True, num_splits=splits)
    check_close(o, ref, what=f"decode case {case} splits {splits}")
    assert np.max(np.abs(lse - ref_lse)) <= 1e-3


def test_decode_bf16_output_and_outliers(mux):
    side = _side(20, SideSpec([700, 63], [1, 1]), 32, 8, 128, decode=True, outliers=True)
    o, lse, ref, ref_lse, _ = _run(mux, side, 32, 8, 128, decode=True, o_f32=False)
    check_close(o, ref, what="decode bf16 out", out_bf16=True)
    assert np.max(np.abs(lse - ref_lse)) <= 1e-3


# ----------------------------------------------------------------------------- prefill (a3)
PREFILL_CASES = [
    # (d, Hq, Hkv, r list, n list)
    (64, 4, 1, [64], [128]),                          # cfg1 prefill
    (128, 8, 2, [0], [300]),                          # several Q tiles + ragged tail, no prefix
    (128, 4, 1, [37, 0, 200], [150, 1, 77]),          # r not page/tile aligned, n = 1 row
    (128, 8, 1, [1000], [129]),                       # long prefix, g = 8
    (64, 4, 4, [5], [260]),                           # MHA, d64
    (128, 4, 2, [127, 129], [128, 255]),              # diagonal straddles two KV tiles
    (128, 4, 4, [30, 0], [200, 129]),                 # MHA d128: prefill_kernel<128, 1> (one q head per CTA)
    (128, 6, 2, [0, 50, 16], [140, 77, 1]),           # g = 3 d128: prefill_kernel<128, 1>
    (64, 6, 2, [20], [150]),                          # g = 3 d64: prefill_kernel<64, 1>
    (128, 12, 6, [17], [130]),                        # Hkv = 6, g = 2 (head pairs)
    # v6 cluster (multicast K/V, g % 4 == 0) with the K-first / adaptive producer order: one tile, one row
    (128, 8, 2, [0], [1]),
    (128, 8, 2, [16], [16]),                          # one cached page + one new page: nt = 1
    (128, 16, 4, [0, 4096, 33, 511], [1, 257, 640, 2]),   # 4 ragged sequences, 1..33 key tiles
    (128, 32, 8, [8191], [2]),                        # Llama-3-8B heads, 65 key tiles, one partial q tile
    (128, 4, 1, [256], [256]),                        # prefix and rows on 128-key tile boundaries
]


@pytest.mark.parametrize("case", range(len(PREFILL_CASES)))
def test_prefill_parity(mux, case):
    d, Hq, Hkv, r, n = PREFILL_CASES[case]
    side = _side(30 + case, SideSpec(r, n), Hq, Hkv, d)
    o, lse, ref, ref_lse, _ = _run(mux, side, Hq, Hkv, d, decode=False)
    check_close(o, ref, what=f"prefill case {case}")
    assert np.max(np.abs(lse - ref_lse)) <= 1e-3


def test_prefill_bf16_output_outliers(mux):
    side = _side(40, SideSpec([90], [200]), 8, 2, 128, outliers=True)
    o, lse, ref, ref_lse, _ = _run(mux, side, 8, 2, 128, decode=False, o_f32=False)
    check_close(o, ref, what="prefill bf16 out", out_bf16=True)


# ----------------------------------------------------------------------------- invariants on GPU
def test_page_permutation_invariance_bitwise(mux):
    side = _side(50, SideSpec([70, 3], [90, 40]), 8, 2, 128)
    a = _run(mux, side, 8, 2, 128, decode=False, num_pages=40, seed=1)[0]
    b = _run(mux, side, 8, 2, 128, decode=False, num_pages=64, seed=99)[0]
    np.testing.assert_array_equal(a, b)
    dside = _side(51, SideSpec([300, 31], [1, 1]), 8, 2, 128, decode=True)
    a = _run(mux, dside, 8, 2, 128, decode=True, num_pages=40, seed=1, num_splits=2)[0]
    b = _run(mux, dside, 8, 2, 128, decode=True, num_pages=64, seed=99, num_splits=2)[0]
    np.testing.assert_array_equal(a, b)


def test_gpu_deterministic_run_to_run(mux):
    import torch
    side = _side(52, SideSpec([10], [260]), 8, 2, 128)
    o1, _, _, _, gs = _run(mux, side, 8, 2, 128, decode=False)
    o2 = torch.empty((260, 8, 128), dtype=torch.float32, device="cuda")
    mux.mux_prefill_attn(gs["pool"], 0, gs["batch"], 8, gs["q"], o2, None)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(o1, o2.cpu().numpy())


def test_decode_deterministic_run_to_run(mux):
    """R17: decode outputs are bitwise run-to-run deterministic, unsplit and split (no float
    atomics in the split-KV merge or the combine)."""
    import torch
    side = _side(56, SideSpec([4000, 700, 15], [1, 1, 1]), 32, 8, 128, decode=True)
    for ns in (1, 5):
        o1, l1, _, _, gs = _run(mux, side, 32, 8, 128, decode=True, num_splits=ns)
        for _ in range(3):
            o2 = torch.empty((3, 32, 128), dtype=torch.float32, device="cuda")
            l2 = torch.empty((3, 32), dtype=torch.float32, device="cuda")
            ws = torch.empty(max(16, mux.mux_decode_workspace_bytes(3, 32, 128, ns)), dtype=torch.uint8, device="cuda")
            mux.mux_decode_attn(gs["pool"], 0, gs["batch"], 32, gs["q"], o2, l2, num_splits=ns, ws=ws)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(o1, o2.cpu().numpy())
            np.testing.assert_array_equal(l1, l2.cpu().numpy())


def _shared_prefix_pools(mux, Hq, Hkv, d, r, n_a, n_b, decode):
    """Two sequences A, B with the same cached prefix of r tokens (r a multiple of 16).  Layout 1:
    B's page table ALIASES A's r/16 prefix pages (mux_pool_share_pages, refcount 2); layout 2:
    private copies.  Returns (outputs, oracle reference) of both layouts."""
    import torch
    from synth import indptr
    g = synth.rng(57, synth.T_K_PF)
    pre_k = synth.bf16_normal(g, (r, Hkv, d))
    pre_v = synth.bf16_normal(g, (r, Hkv, d))
    rows = {}
    for name, n in (("a", n_a), ("b", n_b)):
        rows[name] = (synth.bf16_normal(g, (n, Hkv, d)), synth.bf16_normal(g, (n, Hkv, d)),
                      synth.bf16_normal(g, (n, Hq, d)))
    q = np.concatenate([rows["a"][2], rows["b"][2]])
    npre = r // 16
    scale = 1.0 / math.sqrt(d)
    outs = []
    pages_total = 64
    for shared in (True, False):
        kst = torch.full((1, pages_total, Hkv, 16, d), 0x7FC0, dtype=torch.int16, device="cuda").view(torch.bfloat16)
        pool = mux.Pool(1, pages_total, Hkv, d, 21, kst, kst.clone())
        la, lb = r + n_a, r + n_b
        pa = pool.alloc((la + 15) // 16)
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)  # noqa: E731
        # prefix rows: written once by A (then shared read-only with B), or into both private copies
        mux.mux_append_kv(pool, 0, mux.Batch([0, r], [r], [0, npre], pa[:npre]), dev(pre_k), dev(pre_v))
        if shared:
            pool.share(pa[:npre])
            pb = pa[:npre] + pool.alloc((lb + 15) // 16 - npre)
            assert all(pool.refcount(x) == 2 for x in pa[:npre])
        else:
            pb = pool.alloc((lb + 15) // 16)
            mux.mux_append_kv(pool, 0, mux.Batch([0, r], [r], [0, npre], pb[:npre]), dev(pre_k), dev(pre_v))
        # new rows into each sequence's own (refcount-1) pages; a write into a shared page is rejected
        kn = np.concatenate([rows["a"][0], rows["b"][0]])
        vn = np.concatenate([rows["a"][1], rows["b"][1]])
        batch = mux.Batch([0, n_a, n_a + n_b], [la, lb], [0, len(pa), len(pa) + len(pb)], pa + pb)
        mux.mux_append_kv(pool, 0, batch, dev(kn), dev(vn))
        T = n_a + n_b
        o = torch.empty((T, Hq, d), dtype=torch.float32, device="cuda")
        if decode:
            ws = torch.empty(max(16, mux.mux_decode_workspace_bytes(2, Hq, d, 3)), dtype=torch.uint8, device="cuda")
            mux.mux_decode_attn(pool, 0, batch, Hq, dev(q), o, None, num_splits=3, ws=ws)
        else:
            mux.mux_prefill_attn(pool, 0, batch, Hq, dev(q), o, None)
        torch.cuda.synchronize()
        outs.append(o.cpu().numpy())
        if shared:
            # the oracle reads the same aliased page table from the library's pool image
            kimg = pool.k[0].view(torch.int16).cpu().numpy().view(np.uint16)
            vimg = pool.v[0].view(torch.int16).cpu().numpy().view(np.uint16)
            ref, _ = oracle.attention(q, kimg, vimg, np.array([0, n_a, T], np.int32), np.array([la, lb], np.int32),
                                      np.array([0, len(pa), len(pa) + len(pb)], np.int32),
                                      np.array(pa + pb, np.int32), scale)
            with pytest.raises(mux.MuxError) as e:   # B's append into the aliased prefix page
                mux.mux_append_kv(pool, 0, mux.Batch([0, 1], [r], [0, npre], pb[:npre]), dev(kn[:1]), dev(vn[:1]))
            assert e.value.code == 4
        pool.close()
    return outs, ref


@pytest.mark.parametrize("decode", [False, True])
def test_shared_prefix_pages_gpu(mux, decode):
    """SURVEY §8(c) invariant (i), prefix reuse across requests: two sequences
    whose page tables alias the same full prefix pages (refcount 2) give bitwise the rows they
    give with private copies (reduction order depends only on logical positions), and match the
    oracle reading the aliased table."""
    Hq, Hkv, d = 8, 2, 128
    (o_sh, o_priv), ref = _shared_prefix_pools(mux, Hq, Hkv, d, r=160, n_a=1 if decode else 190,
                                               n_b=1 if decode else 77, decode=decode)
    np.testing.assert_array_equal(o_sh, o_priv)
    check_close(o_sh, ref, what=f"shared prefix ({'decode' if decode else 'prefill'})")


def test_prefix_reuse_equals_recompute_gpu(mux):
    full = _side(53, SideSpec([0], [300]), 4, 1, 128)
    o_full = _run(mux, full, 4, 1, 128, decode=False)[0]
    r = 173
    reuse = SideData(SideSpec([r], [300 - r]), full.q[r:], full.k_rows, full.v_rows)
    o_r = _run(mux, reuse, 4, 1, 128, decode=False)[0]
    check_close(o_r, o_full[r:], atol=2e-3, rtol=0, what="prefix reuse vs recompute")


def test_decode_equals_prefill_n1_gpu(mux):
    full = _side(54, SideSpec([0], [200]), 8, 2, 128)
    o_full = _run(mux, full, 8, 2, 128, decode=False)[0]
    for c in (1, 16, 17, 200):
        dec = SideData(SideSpec([c - 1], [1]), full.q[c - 1:c], [full.k_rows[0][:c]], [full.v_rows[0][:c]])
        o = _run(mux, dec, 8, 2, 128, decode=True)[0]
        check_close(o[0], o_full[c - 1], atol=2e-3, rtol=0, what=f"decode c={c} vs prefill row")


def test_empty_and_invalid_inputs_rejected(mux):
    import torch
    side = _side(55, SideSpec([0], [20]), 4, 1, 64)
    gs = gpu_build_side(mux, side, 8, 3, 1, 64)
    o = torch.empty((20, 4, 64), dtype=torch.float32, device="cuda")
    bad = mux.Batch([0, 0, 20], [0, 20], [0, 0, 2], [int(x) for x in gs["page_ids"]])  # n_b = 0
    with pytest.raises(mux.MuxError):
        mux.mux_prefill_attn(gs["pool"], 0, bad, 4, gs["q"], o)
    with pytest.raises(mux.MuxError):   # decode batch with 20 rows for 1 sequence
        mux.mux_decode_attn(gs["pool"], 0, gs["batch"], 4, gs["q"], o)
    with pytest.raises(mux.MuxError):   # Hq not a multiple of Hkv... (Hkv=1: use head_dim mismatch) layer
        mux.mux_prefill_attn(gs["pool"], 3, gs["batch"], 4, gs["q"], o)


def test_prefill_v_range_flag(mux):
    """The V cache is fp16 (R25, 'P precision'): normal data leaves the pool's error word
    clear; appending a |V| >= 65536 sets MUX_POOL_ERR_V_RANGE instead of failing silently."""
    import torch
    side = _side(60, SideSpec([10], [100]), 4, 2, 128)
    o, _, ref, _, gs = _run(mux, side, 4, 2, 128, decode=False)
    check_close(o, ref, what="prefill before range test")
    assert gs["pool"].error_flags() == 0
    v = side.v_rows[0].copy()
    v[50, 1, 7] = synth.f32_to_bf16_bits(np.array([1.0e6], np.float32))[0]
    big = SideData(side.spec, side.q, side.k_rows, [v])
    gs2 = gpu_build_side(mux, big, 16, 11, 2, 128)
    o2 = torch.empty((100, 4, 128), dtype=torch.float32, device="cuda")
    mux.mux_prefill_attn(gs2["pool"], 0, gs2["batch"], 4, gs2["q"], o2, None)
    torch.cuda.synchronize()
    assert gs2["pool"].error_flags(clear=True) & 1
    assert gs2["pool"].error_flags() == 0


# ----------------------------------------------------------------------------- out-proj (a7)
@pytest.mark.parametrize("T,K,N", [(64, 1024, 8192 // 8), (200, 256, 384), (1, 128, 256), (300, 512, 520),
                                   (128, 4096, 4096), (33, 640, 200), (129, 256, 256), (96, 128, 8)])
def test_outproj_parity(mux, T, K, N):
    """Y = O . W_o partial GEMM vs the oracle's float64 product (O6); T <= 128 takes the skinny
    (swap-AB) kernel, larger T the 128x256 tile kernel; ragged T / N tails on both."""
    import torch
    g = np.random.default_rng(T + K + N)
    x = synth.f32_to_bf16_bits(g.standard_normal((T, K)).astype(np.float32))
    w = synth.f32_to_bf16_bits((g.standard_normal((K, N)) / np.sqrt(K)).astype(np.float32))
    ref = oracle.outproj(x, w)
    xd = torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16)
    wd = mux.mux_outproj_pack_w(torch.from_numpy(w.view(np.int16)).cuda().view(torch.bfloat16))
    y = torch.empty((T, N), dtype=torch.float32, device="cuda")
    mux.mux_outproj(xd, wd, y)
    yb = torch.empty((T, N), dtype=torch.bfloat16, device="cuda")
    mux.mux_outproj(xd, wd, yb)
    torch.cuda.synchronize()
    check_close(y.cpu().numpy(), ref, atol=1e-4, rtol=1e-4, what="outproj f32")
    check_close(yb.float().cpu().numpy(), ref, what="outproj bf16", out_bf16=True)


def test_outproj_sharded_sum_equals_full(mux):
    """KV-head sharding: sum over G shards of O_g W_o,g == O W_o (block identity)."""
    import torch
    g = np.random.default_rng(5)
    T, Hq, d, hidden, G = 96, 16, 128, 512, 4
    x = synth.f32_to_bf16_bits(g.standard_normal((T, Hq * d)).astype(np.float32))
    w = synth.f32_to_bf16_bits((g.standard_normal((Hq * d, hidden)) / 40).astype(np.float32))
    full = oracle.outproj(x, w)
    acc = torch.zeros((T, hidden), dtype=torch.float32, device="cuda")
    kk = Hq * d // G
    for s in range(G):
        xs = torch.from_numpy(np.ascontiguousarray(x[:, s * kk:(s + 1) * kk]).view(np.int16)).cuda().view(torch.bfloat16)
        ws = mux.mux_outproj_pack_w(
            torch.from_numpy(np.ascontiguousarray(w[s * kk:(s + 1) * kk]).view(np.int16)).cuda().view(torch.bfloat16))
        y = torch.empty((T, hidden), dtype=torch.float32, device="cuda")
        mux.mux_outproj(xs, ws, y)
        acc += y
    torch.cuda.synchronize()
    check_close(acc.cpu().numpy(), full, atol=1e-4, rtol=1e-4, what="sharded outproj")


@pytest.mark.parametrize("K,N", [(64, 128), (200, 264), (4096, 4096)])
def test_outproj_pack_layout(mux, K, N):
    """The packed weight image equals the documented layout (include/mux.h), computed here
    element by element with numpy: tile (nt, kb) at (nt*KB + kb)*16 KiB, half h = n-block of
    64, row k, 16-byte chunk c stored at c ^ (k & 7); zero padding past K and N."""
    import torch
    g = np.random.default_rng(K * N)
    w = g.integers(0, 65536, size=(K, N), dtype=np.uint16)
    pk = mux.mux_outproj_pack_w(torch.from_numpy(w.view(np.int16)).cuda().view(torch.bfloat16))
    torch.cuda.synchronize()
    got = pk.data[0].cpu().numpy().view(np.uint16)
    KB, NT = (K + 63) // 64, (N + 127) // 128
    assert got.size * 2 == mux.mux_outproj_packed_bytes(K, N) == NT * KB * 16384
    wp = np.zeros((KB * 64, NT * 128), np.uint16)
    wp[:K, :N] = w
    # [nt][kb][h][k][pos][8]: element (k, n = nt*128 + h*64 + (pos ^ (k&7))*8 + e)
    nt, kb, h, k, pos, e = np.meshgrid(np.arange(NT), np.arange(KB), np.arange(2), np.arange(64), np.arange(8),
                                       np.arange(8), indexing="ij")
    want = wp[kb * 64 + k, nt * 128 + h * 64 + (pos ^ (k & 7)) * 8 + e].reshape(-1)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("num_sms", [8, 16])
@pytest.mark.parametrize("Hq,Hkv,d", [(32, 8, 128), (16, 4, 128), (8, 4, 64), (64, 8, 128)])
def test_decode_two_cta_small_partition_parity(mux, num_sms, Hq, Hkv, d):
    """The decode launch sized for a small partition (mux_decode_attn_sms, <= 16 SMs: two CTAs of
    4 kv heads per SM) against the oracle, ragged contexts incl. page tails, split and unsplit;
    with Hkv = 8 also bitwise equal to the whole-device launch with the same split count (both
    give each warp all pages of one kv head, so the reduction order is the same; with Hkv = 4 the
    device launch splits a head's pages over two warps)."""
    import torch
    spec = SideSpec([4095, 17, 1000, 0, 2049, 15], [1] * 6)
    side = _side(70 + num_sms + Hq, spec, Hq, Hkv, d)
    gs = gpu_build_side(mux, side, sum(spec.pages_needed()) + 4, 13, Hkv, d)
    os_ = oracle_build_side(side, sum(spec.pages_needed()) + 4, 13, Hkv, d)
    ref, _ = oracle.attention(side.q, os_["kpool"], os_["vpool"], os_["qo_indptr"], os_["kv_len"],
                              os_["page_indptr"], os_["page_ids"], 1 / math.sqrt(d))
    for ns in (1, 3):
        ws = torch.empty(max(16, mux.mux_decode_workspace_bytes(6, Hq, d, ns)), dtype=torch.uint8, device="cuda")
        o = torch.empty((6, Hq, d), dtype=torch.float32, device="cuda")
        mux.mux_decode_attn(gs["pool"], 0, gs["batch"], Hq, gs["q"], o, None, num_splits=ns, ws=ws, num_sms=num_sms)
        o_full = torch.empty_like(o)
        mux.mux_decode_attn(gs["pool"], 0, gs["batch"], Hq, gs["q"], o_full, None, num_splits=ns, ws=ws)
        torch.cuda.synchronize()
        check_close(o.cpu().numpy(), ref, what=f"decode {num_sms} SMs, {ns} splits")
        check_close(o_full.cpu().numpy(), ref, what=f"decode device launch, {ns} splits")
        if Hkv == 8:
            assert torch.equal(o, o_full), "small-partition launch != device launch"


# persistent prefill loop (prefill6p_kernel): on a small green-context partition every
# persistent unit walks many work items whose key-tile counts differ (1..nt_max), so the K / V ring
# phases, the Q hand-over barrier and the O epilogue overlap run across items of every length
@pytest.mark.parametrize("Hq,Hkv,r,n,dec_sms", [
    (32, 8, [0, 1000, 17, 64, 300], [300, 1, 129, 700, 2], 132),   # g = 4: clusters of 2 on ~16 SMs
    (12, 6, [5, 0, 260], [520, 131, 64], 128),                     # g = 2: single-CTA items on ~20 SMs
    (8, 2, [0], [1000], 100),                                      # one sequence, 8 q tiles x 1 pair per unit
])
def test_prefill_persistent_on_partition(mux, Hq, Hkv, r, n, dec_sms):
    import torch
    d = 128
    side = _side(90 + Hq + dec_sms, SideSpec(r, n), Hq, Hkv, d)
    need = sum(side.spec.pages_needed())
    gs = gpu_build_side(mux, side, need + 7, 13, Hkv, d)
    os_ = oracle_build_side(side, need + 7, 13, Hkv, d)
    scale = 1.0 / math.sqrt(d)
    T = side.spec.total_new
    part = mux.Partition(0, [dec_sms])
    try:
        _, psms, _, sp = part.query(0)
        o = torch.empty((T, Hq, d), dtype=torch.float32, device="cuda")
        lse = torch.empty((T, Hq), dtype=torch.float32, device="cuda")
        o_full = torch.empty_like(o)
        for _ in range(2):                 # a second launch over the same barriers' fresh phases
            o.fill_(float("nan"))
            mux.mux_prefill_attn(gs["pool"], 0, gs["batch"], Hq, gs["q"], o, lse, scale=scale, stream=sp)
            torch.cuda.synchronize()
        mux.mux_prefill_attn(gs["pool"], 0, gs["batch"], Hq, gs["q"], o_full, None, scale=scale)
        torch.cuda.synchronize()
    finally:
        part.close()
    assert psms <= 148 - dec_sms
    # the same items on the whole device: bitwise the same (each item is computed by one CTA / pair)
    assert torch.equal(o, o_full)
    ref, ref_lse = oracle.attention(side.q, os_["kpool"], os_["vpool"], os_["qo_indptr"], os_["kv_len"],
                                    os_["page_indptr"], os_["page_ids"], scale)
    check_close(o.cpu().numpy(), ref, what=f"persistent prefill on {psms} SMs")
    assert np.max(np.abs(lse.cpu().numpy() - ref_lse)) <= 1e-3
