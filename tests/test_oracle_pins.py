"""Pins of the CPU oracle against things other than itself (SURVEY.md §8(c) 'What pins each part'):
dense numpy brute force, closed forms, invariants, a hand-derived golden example and
allocator test vectors.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle.alloc import (OraclePagePool, PoolExhausted, SplitMix64, build_page_tables,
                          seeded_permutation, slot_of)
import synth
from synth import SideData, SideSpec, Shapes, f32_to_bf16_bits, indptr, make_side
from tests.helpers import dense_attention, oracle_build_side, rel_err

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _side(seed, spec, Hq, Hkv, d, outliers=False):
    return make_side(900 + seed, Shapes(Hq, Hkv, d, 1), spec, decode=False, outliers=outliers)


def _oracle(side, Hq, Hkv, d, num_pages=None, seed=7, scale=None, rows=None):
    need = sum(side.spec.pages_needed())
    st = oracle_build_side(side, num_pages or need + 5, seed, Hkv, d)
    scale = scale if scale is not None else 1.0 / math.sqrt(d)
    out, lse = oracle.attention(side.q, st["kpool"], st["vpool"], st["qo_indptr"], st["kv_len"],
                                st["page_indptr"], st["page_ids"], scale, rows=rows)
    return out, lse, st


# ---------------------------------------------------------------- dense brute force
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("Hq,Hkv", [(4, 1), (8, 2), (4, 4)])
def test_oracle_matches_dense_bruteforce(d, Hq, Hkv):
    g = np.random.default_rng(d * 100 + Hq * 10 + Hkv)
    spec = synth.small_random_spec(g, 3, max_r=100, max_n=40)
    side = _side(d + Hq, spec, Hq, Hkv, d)
    out, lse, _ = _oracle(side, Hq, Hkv, d)
    ref, ref_lse = dense_attention(side, Hq, Hkv, d, 1.0 / math.sqrt(d))
    assert rel_err(out, ref) < 1e-12
    assert np.max(np.abs(lse - ref_lse)) < 1e-12


def test_oracle_matches_dense_outliers_and_long():
    Hq, Hkv, d = 8, 2, 128
    side = _side(5, SideSpec([0, 200, 17], [320, 3, 50]), Hq, Hkv, d, outliers=True)
    out, lse, _ = _oracle(side, Hq, Hkv, d)
    ref, ref_lse = dense_attention(side, Hq, Hkv, d, 1.0 / math.sqrt(d))
    assert rel_err(out, ref) < 1e-12
    assert np.max(np.abs(lse - ref_lse)) < 1e-11


def test_oracle_sampled_rows_equal_full():
    Hq, Hkv, d = 4, 1, 64
    side = _side(6, SideSpec([10, 0], [40, 33]), Hq, Hkv, d)
    full, full_lse, st = _oracle(side, Hq, Hkv, d)
    rows = np.array([0, 5, 39, 40, 72], np.int32)
    out, lse = oracle.attention(side.q, st["kpool"], st["vpool"], st["qo_indptr"], st["kv_len"],
                                st["page_indptr"], st["page_ids"], 1 / 8.0, rows=rows)
    np.testing.assert_array_equal(out, full[rows])
    np.testing.assert_array_equal(lse, full_lse[rows])


# ---------------------------------------------------------------- golden hand example
def test_golden_tiny_attention():
    gold = json.load(open(os.path.join(GOLDEN, "tiny_attention.json")))
    q = f32_to_bf16_bits(np.array(gold["q"], np.float32)[:, None, :])
    k = f32_to_bf16_bits(np.array(gold["k"], np.float32)[:, None, :])
    v = f32_to_bf16_bits(np.array(gold["v"], np.float32)[:, None, :])
    side = SideData(SideSpec([0], [2]), q, [k], [v])
    out, lse, _ = _oracle(side, 1, 1, 2, scale=1.0)
    e = math.e
    np.testing.assert_allclose(out[0, 0], [1.0, 2.0], rtol=0, atol=1e-15)
    np.testing.assert_allclose(out[1, 0], [(1 + 3 * e) / (1 + e), (2 - e) / (1 + e)], rtol=1e-15)
    assert abs(lse[0, 0] - 2.0) < 1e-15
    assert abs(lse[1, 0] - math.log(1 + e)) < 1e-15


# ---------------------------------------------------------------- closed forms
def _with(side, q=None, k=None, v=None):
    return SideData(side.spec, side.q if q is None else q,
                    side.k_rows if k is None else k, side.v_rows if v is None else v)


def test_closed_form_zero_query_gives_prefix_mean():
    Hq, Hkv, d = 4, 2, 64
    side = _side(11, SideSpec([5, 0], [20, 7]), Hq, Hkv, d)
    side = _with(side, q=np.zeros_like(side.q))
    out, lse, _ = _oracle(side, Hq, Hkv, d)
    row = 0
    for b in range(2):
        V = oracle.bf16_to_double(side.v_rows[b])
        for i in range(side.spec.n[b]):
            p = side.spec.r[b] + i
            for h in range(Hq):
                np.testing.assert_allclose(out[row, h], V[: p + 1, h // 2].mean(axis=0), rtol=1e-12, atol=1e-14)
                assert abs(lse[row, h] - math.log(p + 1)) < 1e-12
            row += 1


def test_closed_form_equal_keys_give_prefix_mean():
    Hq, Hkv, d = 2, 1, 64
    side = _side(12, SideSpec([3], [9]), Hq, Hkv, d)
    k = [np.repeat(side.k_rows[0][:1], 12, axis=0)]
    side = _with(side, k=k)
    out, _, _ = _oracle(side, Hq, Hkv, d)
    V = oracle.bf16_to_double(side.v_rows[0])
    for i in range(9):
        np.testing.assert_allclose(out[i, 0], V[: 3 + i + 1, 0].mean(axis=0), rtol=1e-12, atol=1e-14)


def test_closed_form_constant_values():
    Hq, Hkv, d = 4, 1, 128
    side = _side(13, SideSpec([30], [17]), Hq, Hkv, d)
    c = side.v_rows[0][0:1]
    side = _with(side, v=[np.repeat(c, 47, axis=0)])
    out, _, _ = _oracle(side, Hq, Hkv, d)
    cc = oracle.bf16_to_double(c)[0, 0]
    for h in range(Hq):
        np.testing.assert_allclose(out[:, h], np.broadcast_to(cc, out[:, h].shape), rtol=1e-13)


def test_closed_form_single_visible_key():
    Hq, Hkv, d = 2, 1, 64
    side = _side(14, SideSpec([0], [1]), Hq, Hkv, d)
    out, lse, _ = _oracle(side, Hq, Hkv, d)
    V = oracle.bf16_to_double(side.v_rows[0][0, 0])
    K = oracle.bf16_to_double(side.k_rows[0][0, 0])
    for h in range(Hq):
        np.testing.assert_array_equal(out[0, h], V)
        s0 = float(np.dot(oracle.bf16_to_double(side.q[0, h]), K)) / 8.0
        assert abs(lse[0, h] - s0) < 1e-13


def test_closed_form_aligned_key_dominates():
    Hq, Hkv, d = 1, 1, 64
    side = _side(15, SideSpec([40], [1]), Hq, Hkv, d)
    qf = oracle.bf16_to_double(side.q[0, 0])
    k = side.k_rows[0].copy()
    j = 17
    # K_j = 30 * sqrt(d) * q/|q|^2 ... scaled so that s_j exceeds every other score by > 40
    kj = qf / np.dot(qf, qf) * 8.0 * 400.0
    k[j, 0] = f32_to_bf16_bits(kj.astype(np.float32))
    side = _with(side, k=[k])
    out, _, _ = _oracle(side, Hq, Hkv, d)
    V = oracle.bf16_to_double(side.v_rows[0][j, 0])
    np.testing.assert_allclose(out[0, 0], V, rtol=0, atol=1e-12)


# ---------------------------------------------------------------- invariants
def test_invariant_page_permutation_bitwise():
    Hq, Hkv, d = 4, 1, 64
    side = _side(21, SideSpec([37, 0, 15], [29, 60, 1]), Hq, Hkv, d)
    a, la, _ = _oracle(side, Hq, Hkv, d, num_pages=40, seed=1)
    b, lb, _ = _oracle(side, Hq, Hkv, d, num_pages=64, seed=99)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(la, lb)


def test_invariant_prefix_reuse_equals_recompute():
    Hq, Hkv, d = 4, 2, 64
    full = _side(22, SideSpec([0], [90]), Hq, Hkv, d)
    out_full, lse_full, _ = _oracle(full, Hq, Hkv, d)
    r = 53
    reuse = SideData(SideSpec([r], [90 - r]), full.q[r:], full.k_rows, full.v_rows)
    out_r, lse_r, _ = _oracle(reuse, Hq, Hkv, d)
    np.testing.assert_array_equal(out_r, out_full[r:])
    np.testing.assert_array_equal(lse_r, lse_full[r:])


def test_invariant_decode_is_prefill_with_n1():
    Hq, Hkv, d = 8, 2, 128
    full = _side(23, SideSpec([0], [70]), Hq, Hkv, d)
    out_full, _, _ = _oracle(full, Hq, Hkv, d)
    for c in (1, 16, 17, 70):
        dec = SideData(SideSpec([c - 1], [1]), full.q[c - 1:c], [full.k_rows[0][:c]], [full.v_rows[0][:c]])
        out, _, _ = _oracle(dec, Hq, Hkv, d)
        np.testing.assert_array_equal(out[0], out_full[c - 1])


def test_invariant_softmax_rows_sum_to_one():
    Hq, Hkv, d = 4, 1, 64
    side = _side(24, SideSpec([20], [12]), Hq, Hkv, d)
    _, lse, _ = _oracle(side, Hq, Hkv, d)
    K = oracle.bf16_to_double(side.k_rows[0])[:, 0]
    Q = oracle.bf16_to_double(side.q)
    for i in range(12):
        for h in range(Hq):
            s = K[: 20 + i + 1] @ Q[i, h] / 8.0
            assert abs(np.exp(s - lse[i, h]).sum() - 1.0) < 1e-12


def test_invariant_gqa_equals_replicated_mha():
    Hq, Hkv, d = 8, 2, 64
    side = _side(25, SideSpec([9], [20]), Hq, Hkv, d)
    out, _, _ = _oracle(side, Hq, Hkv, d)
    rep = SideData(side.spec, side.q, [np.repeat(side.k_rows[0], 4, axis=1)], [np.repeat(side.v_rows[0], 4, axis=1)])
    out_mha, _, _ = _oracle(rep, Hq, Hq, d)
    np.testing.assert_array_equal(out, out_mha)


@pytest.mark.parametrize("cuts", [[0, 16, 33, 50], [0, 1, 2, 50], [0, 0, 25, 25, 50]])
def test_invariant_split_combine_equals_unsplit(cuts):
    Hq, Hkv, d = 4, 1, 128
    side = _side(26, SideSpec([49], [1]), Hq, Hkv, d)
    out, lse, st = _oracle(side, Hq, Hkv, d)
    pages = st["page_ids"]
    for h in range(Hq):
        parts = [oracle.partial(side.q[0, h], st["kpool"], st["vpool"], 0, pages, a, b, 1 / math.sqrt(d))
                 for a, b in zip(cuts[:-1], cuts[1:])]
        o, l_ = oracle.combine(np.stack([p[0] for p in parts]), np.array([p[1] for p in parts]),
                               np.array([p[2] for p in parts]))
        np.testing.assert_allclose(o, out[0, h], rtol=1e-12, atol=1e-14)
        assert abs(l_ - lse[0, h]) < 1e-12


def test_invariant_shared_prefix_pages():
    """Two sequences whose page tables alias the same (full) prefix pages give the same rows
    as with private copies (SURVEY.md §8(c) invariant (i))."""
    Hq, Hkv, d = 4, 1, 64
    base = _side(27, SideSpec([32, 32], [5, 9]), Hq, Hkv, d)
    k2 = base.k_rows[1].copy(); k2[:32] = base.k_rows[0][:32]
    v2 = base.v_rows[1].copy(); v2[:32] = base.v_rows[0][:32]
    side = SideData(base.spec, base.q, [base.k_rows[0], k2], [base.v_rows[0], v2])
    private, _, _ = _oracle(side, Hq, Hkv, d)
    # shared: seq 1 reuses seq 0's two prefix pages (refcount), own pages for the tail
    pool = OraclePagePool(20, 3)
    p0 = pool.alloc(3)
    pool.share(p0[:2])
    p1 = p0[:2] + pool.alloc(1)
    kimg, vimg = oracle.empty_pool(20, Hkv, d)
    L = [37, 41]
    oracle.append(kimg, vimg, np.concatenate([base.k_rows[0], k2[32:]]), np.concatenate([base.v_rows[0], v2[32:]]),
                  indptr([37, 9]), np.array(L, np.int32), indptr([3, 3]), np.array(p0 + p1, np.int32))
    out, _ = oracle.attention(side.q, kimg, vimg, indptr([5, 9]), np.array(L, np.int32), indptr([3, 3]),
                              np.array(p0 + p1, np.int32), 1 / 8.0)
    np.testing.assert_array_equal(out, private)


def test_outproj_sharded_sum_equals_unsharded():
    g = np.random.default_rng(3)
    T, Hq, d, hidden, G = 5, 8, 16, 32, 4
    o = g.standard_normal((T, Hq * d))
    w = f32_to_bf16_bits(g.standard_normal((Hq * d, hidden)).astype(np.float32))
    full = oracle.outproj(o, w)
    parts = sum(oracle.outproj(o[:, k * Hq * d // G:(k + 1) * Hq * d // G], w[k * Hq * d // G:(k + 1) * Hq * d // G])
                for k in range(G))
    np.testing.assert_allclose(parts, full, rtol=1e-12, atol=1e-12)
    # and against an explicit triple loop on one element
    wd = oracle.bf16_to_double(w)
    assert abs(full[2, 7] - sum(o[2, c] * wd[c, 7] for c in range(Hq * d))) < 1e-12


# ---------------------------------------------------------------- append (O2)
def test_append_byte_image_matches_naive_loop():
    Hq, Hkv, d = 4, 2, 64
    side = _side(31, SideSpec([0, 0, 0], [17, 1, 40]), Hq, Hkv, d)
    st = oracle_build_side(side, 12, 5, Hkv, d)
    # naive per-element reconstruction of the expected image from the slot formula (O2)
    kref = np.full((12, Hkv, 16, d), 0x7FC0, np.uint16)
    pind, pids = st["page_indptr"], st["page_ids"]
    for b in range(3):
        pages = list(pids[pind[b]:pind[b + 1]])
        for t in range(side.spec.L[b]):
            s = slot_of(pages, t)
            for h in range(Hkv):
                for c in range(d):
                    kref[s // 16, h, s % 16, c] = side.k_rows[b][t, h, c]
    np.testing.assert_array_equal(st["kpool"], kref)
    # V: the same slots, stored as fp16 (R25): numpy's float32 -> float16 (round to nearest even)
    vref = np.full((12, Hkv, 16, d), 0x7FC0, np.uint16)
    for b in range(3):
        pages = list(pids[pind[b]:pind[b + 1]])
        for t in range(side.spec.L[b]):
            s = slot_of(pages, t)
            vref[s // 16, :, s % 16, :] = synth.bf16_bits_to_f32(side.v_rows[b][t]).astype(np.float16).view(np.uint16)
    np.testing.assert_array_equal(st["vpool"], vref)


def test_v_fp16_storage_is_exact_for_bf16_inputs():
    """R25: every bf16 value in fp16's normal range [2^-14, 65504] survives the V cache exactly, and
    larger magnitudes clamp to +-65504 (a plain-C conversion in the oracle, pinned by numpy)."""
    bits = np.arange(0, 1 << 16, dtype=np.uint32).astype(np.uint16)
    x = synth.bf16_bits_to_f32(bits).astype(np.float64)
    ok = np.isfinite(x) & (np.abs(x) >= 2.0 ** -14) & (np.abs(x) <= 65504)
    n = bits.size                                  # one token per bf16 bit pattern, d = 8
    k, v = oracle.empty_pool(n // 16, 1, 8, poison=True)
    oracle.append(k, v, np.zeros((n, 1, 8), np.uint16), np.repeat(bits.reshape(n, 1, 1), 8, axis=2),
                  np.array([0, n], np.int32), np.array([n], np.int32), np.array([0, n // 16], np.int32),
                  np.arange(n // 16, dtype=np.int32))
    got = oracle.f16_to_double(v[:, 0, :, 0].reshape(-1))
    np.testing.assert_array_equal(got[ok], x[ok])
    big = np.isfinite(x) & (np.abs(x) > 65504)
    np.testing.assert_array_equal(got[big], np.sign(x[big]) * 65504.0)


# ---------------------------------------------------------------- allocator (O1)
def test_splitmix64_reference_vector():
    g = SplitMix64(0)
    assert g.next() == 0xE220A8397B1DCDAF


def test_allocator_permutation_and_all_or_nothing():
    perm = seeded_permutation(1000, 42)
    assert sorted(perm) == list(range(1000)) and perm != list(range(1000))
    pool = OraclePagePool(10, 42)
    a = pool.alloc(4)
    assert a == seeded_permutation(10, 42)[:4]
    with pytest.raises(PoolExhausted):
        pool.alloc(7)
    assert pool.num_free() == 6
    b = pool.alloc(6)
    assert sorted(a + b) == list(range(10))


def test_allocator_fifo_and_refcounts_bruteforce():
    g = np.random.default_rng(0)
    pool = OraclePagePool(64, 9)
    live = {}
    ref = [0] * 64
    free = list(seeded_permutation(64, 9))
    for step in range(2000):
        op = g.integers(0, 3)
        if op == 0:
            n = int(g.integers(0, 8))
            if n > len(free):
                with pytest.raises(PoolExhausted):
                    pool.alloc(n)
                continue
            got = pool.alloc(n)
            assert got == free[:n]
            free = free[n:]
            for p in got:
                ref[p] = 1
            live[step] = got
        elif op == 1 and live:
            k = list(live)[int(g.integers(0, len(live)))]
            pool.share(live[k])
            for p in live[k]:
                ref[p] += 1
            live[-step - 1] = list(live[k])
        elif live:
            k = list(live)[int(g.integers(0, len(live)))]
            pool.release(live[k])
            for p in live.pop(k):
                ref[p] -= 1
                if ref[p] == 0:
                    free.append(p)
        assert pool.ref == ref
        assert list(pool.free) == free


def test_page_tables_cover_lengths():
    pool = OraclePagePool(100, 1)
    ind, ids = build_page_tables(pool, SideSpec([0, 0, 0, 0], [1, 16, 17, 33]).pages_needed())
    assert ind == [0, 1, 2, 4, 7]
    assert len(set(ids)) == len(ids)


# ---------------------------------------------------------------- f4: QKV projection + RoPE (R26)
def _qkv_inputs(seed, T=5, hidden=96, Hq=4, Hkv=2, d=128):
    g = synth.rng(seed, synth.T_WO)
    x = synth.bf16_normal(g, (T, hidden))
    w = synth.bf16_normal(g, (hidden, (Hq + 2 * Hkv) * d), std=1 / np.sqrt(hidden))
    return x, w


def test_qkv_rope_position_zero_is_the_plain_projection():
    """RoPE at position 0 is the identity, so the oracle is X . W (numpy float64 matmul)."""
    x, w = _qkv_inputs(1)
    out = oracle.qkv_rope(x, w, 4, 2, 128, np.zeros(5, np.int32), 500000.0)
    ref = oracle.bf16_to_double(x) @ oracle.bf16_to_double(w)
    np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)


def test_qkv_rope_rotation_closed_forms():
    """Llama rotate-half convention: pair c rotates by pos * theta^(-2c/d); pair 0 turns by exactly
    pos radians; value heads are not rotated; every pair keeps its norm."""
    Hq, Hkv, d = 4, 2, 128
    x, w = _qkv_inputs(2, Hq=Hq, Hkv=Hkv)
    pos = np.array([1, 7, 100, 4095, 32767], np.int32)
    y = oracle.bf16_to_double(x) @ oracle.bf16_to_double(w)
    out = oracle.qkv_rope(x, w, Hq, Hkv, d, pos, 500000.0)
    for t in range(5):
        for h in range(Hq + Hkv):
            a, b = y[t, h * d:h * d + 64], y[t, h * d + 64:(h + 1) * d]
            oa, ob = out[t, h * d:h * d + 64], out[t, h * d + 64:(h + 1) * d]
            np.testing.assert_allclose(oa ** 2 + ob ** 2, a ** 2 + b ** 2, rtol=1e-10, atol=1e-12)
            p = float(pos[t])
            assert abs(oa[0] - (a[0] * math.cos(p) - b[0] * math.sin(p))) < 1e-9      # pair 0: omega = 1
            assert abs(ob[0] - (b[0] * math.cos(p) + a[0] * math.sin(p))) < 1e-9
            w1 = 500000.0 ** (-2.0 / d)                                                   # pair 1
            assert abs(oa[1] - (a[1] * math.cos(p * w1) - b[1] * math.sin(p * w1))) < 1e-9
    v0 = (Hq + Hkv) * d
    np.testing.assert_allclose(out[:, v0:], y[:, v0:], rtol=1e-12, atol=1e-12)


def test_qkv_rope_scores_depend_on_relative_position_only():
    """The defining property of rotary embeddings: q(m) . k(n) depends on m - n only (same token
    contents at (m, n) and (m + s, n + s) give the same score)."""
    Hq, Hkv, d = 2, 2, 128
    x, w = _qkv_inputs(3, T=2, Hq=Hq, Hkv=Hkv)
    xs = np.concatenate([x, x, x], axis=0)                  # rows: (q tok, k tok) at 3 offsets
    pos = np.array([10, 3, 10 + 500, 3 + 500, 10 + 30000, 3 + 30000], np.int32)
    out = oracle.qkv_rope(np.concatenate([xs[0::2][:, None], xs[1::2][:, None]], 1).reshape(6, -1), w, Hq, Hkv,
                          d, pos, 500000.0)
    q = out[0::2, 0:d]                                      # query head 0 of the q token
    k = out[1::2, Hq * d:Hq * d + d]                        # key head 0 of the k token
    s = (q * k).sum(axis=1)
    np.testing.assert_allclose(s, s[0], rtol=1e-9, atol=1e-9)


# ---------------------------------------------------------------- f4: SwiGLU FFN (R27)
def test_ffn_swiglu_matches_numpy_and_closed_forms():
    """h = silu(x W1) * (x W3) against numpy (scipy's expit as the sigmoid), y = bf16(h) W2 against a
    numpy matmul of the rounded h; silu(0) = 0 and silu(a) -> a for large a."""
    import scipy.special
    g = synth.rng(4, synth.T_WO)
    T, hidden, inter = 6, 64, 256
    x = synth.bf16_normal(g, (T, hidden))
    w1, w3 = synth.bf16_normal(g, (hidden, inter), std=0.2), synth.bf16_normal(g, (hidden, inter), std=0.2)
    w2 = synth.bf16_normal(g, (inter, hidden), std=0.1)
    h, y = oracle.ffn_swiglu(x, w1, w3, w2)
    a = oracle.bf16_to_double(x) @ oracle.bf16_to_double(w1)
    b = oracle.bf16_to_double(x) @ oracle.bf16_to_double(w3)
    np.testing.assert_allclose(h, a * scipy.special.expit(a) * b, rtol=1e-12, atol=1e-12)
    hb = oracle.bf16_to_double(synth.f32_to_bf16_bits(h.astype(np.float32)))
    np.testing.assert_allclose(y, hb @ oracle.bf16_to_double(w2), rtol=1e-9, atol=1e-9)
    z = np.zeros((1, hidden), np.uint16)                      # x = 0 -> silu(0) * 0 = 0
    assert not oracle.ffn_swiglu(z, w1, w3, w2)[1].any()
