"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain double-precision CPU reference of the MuxWise hot path (arXiv 2504.14489):
paged append (O2), prefill/decode attention over the paged pool (O3/O4), split
combine (O5), out-projection (O6), the page allocator (O1, oracle/alloc.py) and the
QKV projection + RoPE and the SwiGLU FFN of f4 (qkv_rope, ffn_swiglu).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg, --impl reference)
may import this package.  The product path (paper_2504_14489_b200) never imports it and
it never imports the product path; the two share only the seeded input generators in
synth/.  Parity status of every function: pinned.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", _SO, src, "-lm"])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.oracle_append.argtypes = [P, P, i64, ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int, P, P, P, P]
        L.oracle_attention.argtypes = [P, i64, ctypes.c_int, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       P, P, P, P, dbl, P, i64, P, P]
        L.oracle_partial.argtypes = [P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, dbl, i64, i64, P, P, P]
        L.oracle_combine.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, P, P]
        L.oracle_qkv_rope.argtypes = [P, i64, ctypes.c_int, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, dbl, P]
        L.oracle_qkv_rope.restype = ctypes.c_int
        L.oracle_ffn_swiglu.argtypes = [P, i64, ctypes.c_int, P, P, P, ctypes.c_int, P, P]
        L.oracle_ffn_swiglu.restype = ctypes.c_int
        L.oracle_num_threads.restype = ctypes.c_int
        for f in (L.oracle_append, L.oracle_attention, L.oracle_partial, L.oracle_combine):
            f.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def num_threads() -> int:
    return lib().oracle_num_threads()


def append(kpool: np.ndarray, vpool: np.ndarray, k_new, v_new, new_indptr, kv_len, page_indptr, page_ids):
    """O2.  kpool/vpool: uint16 [num_pages, Hkv, 16, d] (ONE layer), modified in place.  K rows are
    copied (bf16 bits); V rows are stored as fp16 bits (R25)."""
    assert kpool.dtype == np.uint16 and kpool.flags.c_contiguous and vpool.flags.c_contiguous
    num_pages, Hkv, P, d = kpool.shape
    assert P == 16
    k_new, v_new = _c(k_new, np.uint16), _c(v_new, np.uint16)
    new_indptr, kv_len = _c(new_indptr, np.int32), _c(kv_len, np.int32)
    page_indptr, page_ids = _c(page_indptr, np.int32), _c(page_ids, np.int32)
    rc = lib().oracle_append(_p(kpool), _p(vpool), num_pages, Hkv, d, _p(k_new), _p(v_new),
                             len(kv_len), _p(new_indptr), _p(kv_len), _p(page_indptr), _p(page_ids))
    if rc != 0:
        raise ValueError("oracle_append: page id out of range")


def attention(q, kpool, vpool, qo_indptr, kv_len, page_indptr, page_ids, scale: Optional[float] = None,
              rows: Optional[np.ndarray] = None):
    """O3/O4.  q: uint16 [total_q, Hq, d]; pools: uint16 [num_pages, Hkv, 16, d] (K bf16, V fp16 bits).
    Returns (out float64 [n_rows, Hq, d], lse float64 [n_rows, Hq])."""
    q = _c(q, np.uint16)
    total_q, Hq, d = q.shape
    _, Hkv, _, d2 = kpool.shape
    assert d == d2
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    qo_indptr, kv_len = _c(qo_indptr, np.int32), _c(kv_len, np.int32)
    page_indptr, page_ids = _c(page_indptr, np.int32), _c(page_ids, np.int32)
    if rows is not None:
        rows = _c(rows, np.int32)
        n_rows = len(rows)
    else:
        n_rows = total_q
    out = np.zeros((n_rows, Hq, d), dtype=np.float64)
    lse = np.zeros((n_rows, Hq), dtype=np.float64)
    kpool, vpool = _c(kpool, np.uint16), _c(vpool, np.uint16)
    rc = lib().oracle_attention(_p(q), total_q, Hq, _p(kpool), _p(vpool), Hkv, d, len(kv_len),
                                _p(qo_indptr), _p(kv_len), _p(page_indptr), _p(page_ids), float(scale),
                                _p(rows) if rows is not None else None, n_rows, _p(out), _p(lse))
    if rc != 0:
        raise ValueError(f"oracle_attention rc={rc}")
    return out, lse


def partial(q_row, kpool, vpool, kh: int, pages, j0: int, j1: int, scale: float):
    """State (o normalised, m, l) of one (row, head) over key positions [j0, j1)."""
    q_row = _c(q_row, np.uint16)
    _, Hkv, _, d = kpool.shape
    pages = _c(pages, np.int32)
    o = np.zeros(d, dtype=np.float64)
    m = ctypes.c_double()
    l = ctypes.c_double()
    lib().oracle_partial(_p(q_row), _p(_c(kpool, np.uint16)), _p(_c(vpool, np.uint16)), Hkv, d, kh,
                         _p(pages), float(scale), j0, j1, _p(o), ctypes.byref(m), ctypes.byref(l))
    return o, m.value, l.value


def combine(o_s, m_s, l_s):
    """O5 split combine of S partial states -> (o, lse)."""
    o_s, m_s, l_s = _c(o_s, np.float64), _c(m_s, np.float64), _c(l_s, np.float64)
    S, d = o_s.shape
    o = np.zeros(d, dtype=np.float64)
    lse = ctypes.c_double()
    lib().oracle_combine(S, d, _p(o_s), _p(m_s), _p(l_s), _p(o), ctypes.byref(lse))
    return o, lse.value


def outproj(o_rows: np.ndarray, w_o_bits: np.ndarray) -> np.ndarray:
    """O6: Y = O . W_o in float64, on the full (unsharded) heads.
    o_rows: [T, Hq*d] float64 (or bf16 bits as uint16); w_o_bits: [Hq*d, hidden] bf16 bits."""
    if o_rows.dtype == np.uint16:
        o_rows = bf16_to_double(o_rows)
    return np.matmul(o_rows.astype(np.float64), bf16_to_double(w_o_bits))


def f16_to_double(bits: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(bits, dtype=np.uint16).view(np.float16).astype(np.float64)


def qkv_rope(x_bits: np.ndarray, w_bits: np.ndarray, Hq: int, Hkv: int, d: int, pos, theta: float) -> np.ndarray:
    """f4: y = x . w (float64) with RoPE(pos) on the query and key heads (R26).
    x_bits [T][hidden], w_bits [hidden][(Hq + 2 Hkv) d] bf16 bits.  Returns float64 [T][(Hq+2Hkv) d]."""
    x_bits, w_bits = _c(x_bits, np.uint16), _c(w_bits, np.uint16)
    T, hidden = x_bits.shape
    assert w_bits.shape == (hidden, (Hq + 2 * Hkv) * d)
    pos = _c(pos, np.int32)
    out = np.zeros((T, (Hq + 2 * Hkv) * d), np.float64)
    lib().oracle_qkv_rope(_p(x_bits), T, hidden, _p(w_bits), Hq, Hkv, d, _p(pos), float(theta), _p(out))
    return out


def ffn_swiglu(x_bits, w1_bits, w3_bits, w2_bits):
    """f4 FFN (R27): h = silu(x.w1) * (x.w3) (float64), y = bf16(h) . w2.  Returns (h, y) float64."""
    x_bits = _c(x_bits, np.uint16)
    w1_bits, w3_bits, w2_bits = _c(w1_bits, np.uint16), _c(w3_bits, np.uint16), _c(w2_bits, np.uint16)
    T, hidden = x_bits.shape
    inter = w1_bits.shape[1]
    assert w1_bits.shape == w3_bits.shape == (hidden, inter) and w2_bits.shape == (inter, hidden)
    h = np.zeros((T, inter), np.float64)
    y = np.zeros((T, hidden), np.float64)
    lib().oracle_ffn_swiglu(_p(x_bits), T, hidden, _p(w1_bits), _p(w3_bits), _p(w2_bits), inter, _p(h), _p(y))
    return h, y


def bf16_to_double(bits: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def empty_pool(num_pages: int, Hkv: int, d: int, poison: bool = True):
    """One layer of pool image, NaN-poisoned (bf16 0x7FC0) so a read of an unwritten slot shows."""
    fill = 0x7FC0 if poison else 0
    k = np.full((num_pages, Hkv, 16, d), fill, dtype=np.uint16)
    v = np.full((num_pages, Hkv, 16, d), fill, dtype=np.uint16)
    return k, v
