"""GPU parity of f4's fused QKV projection + RoPE + KV append (include/mux.h mux_qkv_rope_append,
DESIGN.md R25/R26) against the oracle (oracle.qkv_rope, float64): the query rows it returns, the K
rows (bf16) and V rows (fp16) it writes into the paged pool through the page table, and the
untouched (NaN-poisoned) slots, which must keep their bytes."""
import math

import numpy as np
import pytest

import oracle
import synth
from synth import SideSpec, indptr

pytestmark = pytest.mark.gpu
THETA = 500000.0


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


def _bits(t):
    import torch
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def _close(gpu, ref, rel, what):
    """|gpu - ref| <= rel |ref| + 2e-4 (fp32 accumulation + fp32 table, then one rounding to the
    16-bit storage type: rel = 2^-8 for bf16, 2^-10 for fp16)"""
    d = np.abs(gpu - ref)
    bad = d > rel * np.abs(ref) + 2e-4
    assert not bad.any(), f"{what}: {bad.sum()} elements out of tolerance, max|d| {d.max():.3e}"
    return float(d.max())


@pytest.mark.parametrize("spec,Hq,Hkv,hidden", [
    (SideSpec([0, 40, 17], [300, 1, 77]), 8, 2, 256),        # ragged, cached prefixes, page tails
    (SideSpec([1000, 0], [129, 256]), 32, 8, 4096),          # Llama-3-8B projection shape
    (SideSpec([4000], [64]), 64, 8, 1024),                   # 70B head counts, positions ~4k
])
def test_qkv_rope_append_matches_oracle(mux, spec, Hq, Hkv, hidden):
    import torch
    d = 128
    T = spec.total_new
    g = synth.rng(11, synth.T_WO, salt=Hq)
    x = synth.bf16_normal(g, (T, hidden))
    w = synth.bf16_normal(g, (hidden, (Hq + 2 * Hkv) * d), std=1 / math.sqrt(hidden))
    pos = np.concatenate([r + np.arange(n) for r, n in zip(spec.r, spec.n)]).astype(np.int32)
    pages = sum(spec.pages_needed()) + 5
    kst = torch.full((2, pages, Hkv, 16, d), 0x7FC0, dtype=torch.int16, device="cuda").view(torch.bfloat16)
    vst = torch.full((2, pages, Hkv, 16, d), 0x7FC0, dtype=torch.int16, device="cuda").view(torch.float16)
    pool = mux.Pool(2, pages, Hkv, d, 21, kst, vst)
    pind, pids = pool.page_tables(spec.pages_needed())
    batch = mux.Batch(indptr(spec.n), spec.L, pind, pids)
    rope = mux.mux_rope_table(max(spec.L) + 1, d, THETA)
    q_out = torch.empty((T, Hq, d), dtype=torch.bfloat16, device="cuda")
    mux.mux_qkv_rope_append(pool, 1, batch, Hq, _dev(x), mux.mux_outproj_pack_w(_dev(w)), rope, q_out)
    torch.cuda.synchronize()
    assert pool.error_flags() == 0
    ref = oracle.qkv_rope(x, w, Hq, Hkv, d, pos, THETA)
    rq = ref[:, :Hq * d].reshape(T, Hq, d)
    rk = ref[:, Hq * d:(Hq + Hkv) * d].reshape(T, Hkv, d)
    rv = ref[:, (Hq + Hkv) * d:].reshape(T, Hkv, d)
    _close(oracle.bf16_to_double(_bits(q_out)), rq, 2.0 ** -8, "q rows")
    kimg, vimg = _bits(kst[1]), _bits(vst[1])
    assert (_bits(kst[0]) == 0x7FC0).all() and (_bits(vst[0]) == 0x7FC0).all(), "another layer was written"
    written = np.zeros(kimg.shape[:1] + kimg.shape[2:3], bool)       # [page][slot]
    row = 0
    for b, (r, n) in enumerate(zip(spec.r, spec.n)):
        ptab = pids[pind[b]:pind[b + 1]]
        for i in range(n):
            p = r + i
            pg, sl = ptab[p // 16], p % 16
            _close(oracle.bf16_to_double(kimg[pg, :, sl]), rk[row], 2.0 ** -8, f"k row {row}")
            _close(oracle.f16_to_double(vimg[pg, :, sl]), rv[row], 2.0 ** -10, f"v row {row}")
            written[pg, sl] = True
            row += 1
    # every other slot keeps its poison bytes
    assert (kimg.transpose(0, 2, 1, 3)[~written] == 0x7FC0).all()
    assert (vimg.transpose(0, 2, 1, 3)[~written] == 0x7FC0).all()


def test_qkv_rope_rejects_positions_past_the_table(mux):
    import torch
    spec = SideSpec([100], [20])
    Hq, Hkv, d, hidden = 4, 2, 128, 64
    kst = torch.zeros((1, 16, Hkv, 16, d), dtype=torch.bfloat16, device="cuda")
    vst = torch.zeros((1, 16, Hkv, 16, d), dtype=torch.float16, device="cuda")
    pool = mux.Pool(1, 16, Hkv, d, 3, kst, vst)
    pind, pids = pool.page_tables(spec.pages_needed())
    batch = mux.Batch(indptr(spec.n), spec.L, pind, pids)
    x = torch.zeros((20, hidden), dtype=torch.bfloat16, device="cuda")
    w = mux.mux_outproj_pack_w(torch.zeros((hidden, (Hq + 2 * Hkv) * d), dtype=torch.bfloat16, device="cuda"))
    q_out = torch.empty((20, Hq, d), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(mux.MuxError):
        mux.mux_qkv_rope_append(pool, 0, batch, Hq, x, w, mux.mux_rope_table(64, d), q_out)


@pytest.mark.parametrize("T,hidden,inter", [(300, 256, 384), (129, 1024, 2048), (64, 4096, 14336)])
def test_ffn_swiglu_matches_oracle(mux, T, hidden, inter):
    """f4 FFN (R27): the gate/up GEMM with its silu * up epilogue and the down GEMM against the
    oracle: H (bf16) within one bf16 rounding of the float64 h, Y within the rounding of H plus
    fp32 accumulation."""
    import torch
    g = synth.rng(12, synth.T_WO, salt=T)
    x = synth.bf16_normal(g, (T, hidden))
    w1 = synth.bf16_normal(g, (hidden, inter), std=1 / math.sqrt(hidden))
    w3 = synth.bf16_normal(g, (hidden, inter), std=1 / math.sqrt(hidden))
    w2 = synth.bf16_normal(g, (inter, hidden), std=1 / math.sqrt(inter))
    w13 = mux.mux_ffn_pack_w13(_dev(w1), _dev(w3))
    w2p = mux.mux_outproj_pack_w(_dev(w2))
    h = torch.empty((T, inter), dtype=torch.bfloat16, device="cuda")
    y = torch.empty((T, hidden), dtype=torch.bfloat16, device="cuda")
    mux.mux_ffn_swiglu(_dev(x), w13, w2p, h, y)
    torch.cuda.synchronize()
    rh, ry = oracle.ffn_swiglu(x, w1, w3, w2)
    _close(oracle.bf16_to_double(_bits(h)), rh, 2.0 ** -8, "h")
    gy = oracle.bf16_to_double(_bits(y))
    d = np.abs(gy - ry)
    tol = 2.0 ** -7 * np.abs(ry) + 1e-2 * np.sqrt(np.mean(ry ** 2))
    assert (d <= tol).all(), f"y: {(d > tol).sum()} elements out of tolerance, max|d| {d.max():.3e}"


@pytest.mark.parametrize("decode", [False, True])
def test_full_layer_side_equals_the_composed_calls(mux, decode):
    """mux_side's full-layer mode (fused QKV + RoPE + append -> attention -> out-projection ->
    FFN per layer) through mux_run_layer gives bitwise the outputs of the same steps called one by
    one (each of which is checked against the oracle above and in test_gpu_parity.py)."""
    import torch
    Hq, Hkv, d, hidden, inter, layers = 8, 2, 128, 256, 384, 2
    spec = SideSpec([33, 0, 200], [1, 1, 1]) if decode else SideSpec([0, 40], [150, 77])
    T = spec.total_new
    g = synth.rng(13, synth.T_WO, salt=int(decode))
    x = _dev(synth.bf16_normal(g, (T, hidden)))
    w_qkv = mux.mux_outproj_pack_w(_dev(synth.bf16_normal(g, (hidden, (Hq + 2 * Hkv) * d), std=0.06)))
    w_o = mux.mux_outproj_pack_w(_dev(synth.bf16_normal(g, (Hq * d, hidden), std=0.03)))
    w13 = mux.mux_ffn_pack_w13(_dev(synth.bf16_normal(g, (hidden, inter), std=0.06)),
                               _dev(synth.bf16_normal(g, (hidden, inter), std=0.06)))
    w2 = mux.mux_outproj_pack_w(_dev(synth.bf16_normal(g, (inter, hidden), std=0.05)))
    rope = mux.mux_rope_table(max(spec.L) + 1, d)
    outs = []
    for fused in (True, False):
        pages = sum(spec.pages_needed()) + 4
        kst = torch.zeros((layers, pages, Hkv, 16, d), dtype=torch.bfloat16, device="cuda")
        vst = torch.zeros((layers, pages, Hkv, 16, d), dtype=torch.float16, device="cuda")
        pool = mux.Pool(layers, pages, Hkv, d, 9, kst, vst)
        pind, pids = pool.page_tables(spec.pages_needed())
        # the cached prefix of every layer (same bytes in both runs)
        for l in range(layers):
            kst[l].normal_(generator=torch.Generator(device="cuda").manual_seed(l))
            vst[l].normal_(generator=torch.Generator(device="cuda").manual_seed(100 + l))
        batch = mux.Batch(indptr(spec.n), spec.L, pind, pids)
        q = torch.empty((T, Hq, d), dtype=torch.bfloat16, device="cuda")
        o = torch.empty((T, Hq, d), dtype=torch.bfloat16, device="cuda")
        y = torch.empty((T, hidden), dtype=torch.bfloat16, device="cuda")
        h = torch.empty((T, inter), dtype=torch.bfloat16, device="cuda")
        fy = torch.empty((T, hidden), dtype=torch.bfloat16, device="cuda")
        ws = torch.empty(1 << 22, dtype=torch.uint8, device="cuda")
        if fused:
            part = mux.Partition(0, [16])
            side = mux.make_side(batch, Hq, q, o, scale=1 / math.sqrt(d), layer0=0, num_layers=layers, w_o=w_o, y=y,
                                 num_splits=2 if decode else 0, ws=ws if decode else None,
                                 qkv=(x, w_qkv, rope), ffn=(w13, w2, h, fy))
            mux.mux_run_layer(part, 0, pool, None if decode else side, side if decode else None)
            torch.cuda.synchronize()
            part.close()
        else:
            for l in range(layers):
                mux.mux_qkv_rope_append(pool, l, batch, Hq, x, w_qkv, rope, q)
                if decode:
                    mux.mux_decode_attn(pool, l, batch, Hq, q, o, None, scale=1 / math.sqrt(d), num_splits=2, ws=ws)
                else:
                    mux.mux_prefill_attn(pool, l, batch, Hq, q, o, None, scale=1 / math.sqrt(d))
                mux.mux_outproj(o.view(T, -1), w_o, y)
                mux.mux_ffn_swiglu(y, w13, w2, h, fy)
            torch.cuda.synchronize()
        outs.append([_bits(t) for t in (q, o, y, fy, kst, vst.view(torch.bfloat16))])
    for a, b, name in zip(outs[0], outs[1], ("q", "o", "y", "ffn y", "K pool", "V pool")):
        np.testing.assert_array_equal(a, b, err_msg=name)
