"""ctypes binding of include/mux.h (argument marshalling only).

Names follow the C ABI (mux_pool_create, mux_append_kv, mux_prefill_attn, mux_decode_attn,
mux_run_layer, ...).  Tensors are torch tensors: data_ptr() is passed as a plain pointer.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libmux.so")

MUX_OK = 0
MUX_DTYPE_BF16 = 0
MUX_DTYPE_F32 = 1
STATUS = {0: "MUX_OK", 1: "MUX_ERR_INVALID_ARG", 2: "MUX_ERR_UNSUPPORTED", 3: "MUX_ERR_POOL_EXHAUSTED",
          4: "MUX_ERR_SHARED_PAGE_WRITE", 5: "MUX_ERR_NO_CONFIG", 6: "MUX_ERR_CUDA", 7: "MUX_ERR_WORKSPACE"}

c_i32, c_i64, c_u64, c_p, c_f32, c_dbl, c_sz = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p,
                                                ctypes.c_float, ctypes.c_double, ctypes.c_size_t)


class MuxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class PoolDesc(ctypes.Structure):
    _fields_ = [("num_layers", c_i32), ("num_pages", c_i32), ("page_size", c_i32), ("num_kv_heads", c_i32),
                ("head_dim", c_i32), ("k_storage", c_p), ("v_storage", c_p), ("free_list_seed", c_u64)]


class BatchC(ctypes.Structure):
    _fields_ = [("num_seqs", c_i32), ("qo_indptr", c_p), ("kv_len", c_p), ("page_indptr", c_p),
                ("page_ids", c_p), ("total_q", c_i32), ("max_q", c_i32), ("max_kv", c_i32),
                ("h_qo_indptr", c_p), ("h_kv_len", c_p), ("h_page_indptr", c_p), ("h_page_ids", c_p)]


LayerHook = ctypes.CFUNCTYPE(None, c_p, c_i32, c_i32, c_p)


MUX_AR_MAX_WORLD = 8


class ArPeersC(ctypes.Structure):
    _fields_ = [("world", c_i32), ("rank", c_i32), ("epoch", ctypes.c_uint32),
                ("stage", c_p * MUX_AR_MAX_WORLD), ("y", c_p * MUX_AR_MAX_WORLD)]


class SideC(ctypes.Structure):
    _fields_ = [("batch", ctypes.POINTER(BatchC)), ("num_q_heads", c_i32), ("q", c_p), ("k_new", c_p),
                ("v_new", c_p), ("o", c_p), ("lse", c_p), ("q_stride", c_i64), ("kv_stride", c_i64),
                ("o_stride", c_i64), ("lse_stride", c_i64), ("o_dtype", c_i32), ("scale", c_f32),
                ("layer0", c_i32), ("num_layers", c_i32), ("append", c_i32), ("num_splits", c_i32),
                ("ws", c_p), ("ws_bytes", c_sz), ("w_o", c_p), ("y", c_p), ("w_stride", c_i64),
                ("y_stride", c_i64), ("hidden", c_i32), ("y_dtype", c_i32), ("hook", LayerHook),
                ("hook_user", c_p), ("ar_fn", c_p), ("ar_comm", c_p), ("attn_events", c_p),
                ("x_in", c_p), ("hidden_in", c_i32), ("w_qkv", c_p), ("rope", c_p), ("rope_max_pos", c_i32),
                ("w13", c_p), ("w2", c_p), ("ffn_h", c_p), ("ffn_y", c_p), ("ffn_inter", c_i32),
                ("ar_peers", c_p)]


class EngineDesc(ctypes.Structure):
    _fields_ = [("num_q_heads", c_i32), ("scale", c_f32), ("src_q", c_p), ("src_k", c_p), ("src_v", c_p),
                ("src_rows", c_i32), ("w_o", c_p), ("hidden", c_i32), ("max_decode_seqs", c_i32),
                ("max_prefill_tokens", c_i32), ("fixed_split", c_i32), ("n_cost", c_i32), ("dec_theta", c_p),
                ("pf_theta", c_p), ("dec_slowdown", c_p), ("tbt_slo_us", c_dbl), ("fixed_pl", c_i32),
                ("handoff", c_i32), ("keep_pages", c_i32), ("serialize", c_i32), ("use_graphs", c_i32),
                ("o_log", c_p), ("y_log", c_p), ("log_rows", c_i32), ("o_f32", c_i32), ("overlap", c_i32)]


class RequestC(ctypes.Structure):
    _fields_ = [("id", c_i32), ("cached", c_i32), ("prompt", c_i32), ("gen", c_i32), ("src_base", c_i32),
                ("arrival_iter", c_i32), ("arrival_us", c_dbl)]


class EngineStats(ctypes.Structure):
    _fields_ = [("makespan_us", c_dbl), ("prefill_tokens", c_i64), ("decode_tokens", c_i64),
                ("decode_iters", c_i32), ("prefill_groups", c_i32), ("split_changes", c_i32), ("handoffs", c_i32),
                ("busy_dec_us", c_dbl), ("busy_pf_us", c_dbl), ("bubble_ratio", c_dbl), ("bubble_ratio_dec", c_dbl),
                ("bubble_ratio_pf", c_dbl), ("tbt_mean_us", c_dbl), ("tbt_max_us", c_dbl), ("ttft_mean_us", c_dbl),
                ("ttft_max_us", c_dbl), ("gap_mean_us", c_dbl), ("gap_max_us", c_dbl), ("graphs", c_i32),
                ("graph_bytes", c_i64), ("logged_rows", c_i32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class SideTimes(ctypes.Structure):
    _fields_ = [("dec_start_ns", c_u64), ("dec_end_ns", c_u64), ("pf_start_ns", c_u64), ("pf_end_ns", c_u64)]


_lib = None


def lib():
    """Load libmux.so (in-tree).  Raises if it is missing: there is no fallback path."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO):
        raise ImportError(f"libmux.so not built ({_SO}); run __graft_entry__.build()")
    L = ctypes.CDLL(_SO)
    sig = {
        "mux_pool_create": [ctypes.POINTER(c_p), ctypes.POINTER(PoolDesc)],
        "mux_pool_destroy": [c_p],
        "mux_pool_alloc_pages": [c_p, c_i32, c_p],
        "mux_pool_share_pages": [c_p, c_i32, c_p],
        "mux_pool_free_pages": [c_p, c_i32, c_p],
        "mux_pool_num_free": [c_p, ctypes.POINTER(c_i32)],
        "mux_pool_refcount": [c_p, c_i32, ctypes.POINTER(c_i32)],
        "mux_pool_free_list": [c_p, c_p, c_i32, ctypes.POINTER(c_i32)],
        "mux_pool_storage": [c_p, ctypes.POINTER(c_p), ctypes.POINTER(c_p)],
        "mux_pool_error_flags": [c_p, ctypes.POINTER(ctypes.c_uint32), c_i32],
        "mux_append_kv": [c_p, c_i32, ctypes.POINTER(BatchC), c_p, c_p, c_p],
        "mux_prefill_attn": [c_p, c_i32, ctypes.POINTER(BatchC), c_i32, c_p, c_p, c_i32, c_p, c_f32, c_p],
        "mux_decode_attn": [c_p, c_i32, ctypes.POINTER(BatchC), c_i32, c_p, c_p, c_i32, c_p, c_f32, c_i32, c_p,
                            c_sz, c_p],
        "mux_decode_attn_sms": [c_p, c_i32, ctypes.POINTER(BatchC), c_i32, c_p, c_p, c_i32, c_p, c_f32, c_i32, c_p,
                                c_sz, c_p, c_i32],
        "mux_partition_create": [ctypes.POINTER(c_p), c_i32, c_p, c_i32],
        "mux_partition_destroy": [c_p],
        "mux_partition_query": [c_p, c_i32, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32), ctypes.POINTER(c_p),
                                ctypes.POINTER(c_p)],
        "mux_partition_memory": [c_p, ctypes.POINTER(c_i64)],
        "mux_stream_read": [c_p, c_sz, c_i32, c_p],
        "mux_run_layer": [c_p, c_i32, c_p, ctypes.POINTER(SideC), ctypes.POINTER(SideC), c_p, c_p],
        "mux_outproj": [c_p, c_p, c_p, c_i32, c_i32, c_i32, c_i32, c_p],
        "mux_outproj_sms": [c_p, c_p, c_p, c_i32, c_i32, c_i32, c_i32, c_p, c_i32],
        "mux_outproj_pack_w": [c_p, c_p, c_i32, c_i32, c_p],
        "mux_outproj_allreduce": [c_p, c_p, c_i32, c_i32, c_i32, ctypes.POINTER(ArPeersC), c_i32, c_p],
        "mux_outproj_allreduce_emulated": [ctypes.POINTER(c_p), ctypes.POINTER(c_p), c_i32, c_i32, c_i32,
                                           ctypes.POINTER(ArPeersC), c_p],
        "mux_ipc_alloc": [c_sz, ctypes.POINTER(c_p), c_p],
        "mux_ipc_open": [c_p, ctypes.POINTER(c_p)],
        "mux_ipc_close": [c_p],
        "mux_ipc_free": [c_p],
        "mux_side_plan": [ctypes.POINTER(SideC), c_i32, c_p, c_i32, ctypes.POINTER(c_i32)],
        "mux_rope_table": [c_p, c_i32, c_i32, c_dbl, c_p],
        "mux_ffn_pack_w13": [c_p, c_p, c_p, c_i32, c_i32, c_p],
        "mux_ffn_swiglu": [c_p, c_p, c_p, c_p, c_p, c_i32, c_i32, c_i32, c_p],
        "mux_qkv_rope_append": [c_p, c_i32, ctypes.POINTER(BatchC), c_i32, c_p, c_i32, c_p, c_p, c_i32, c_p, c_p],
        "mux_engine_create": [ctypes.POINTER(c_p), c_p, c_p, ctypes.POINTER(EngineDesc)],
        "mux_engine_submit": [c_p, ctypes.POINTER(RequestC), c_i32],
        "mux_engine_run": [c_p, ctypes.POINTER(EngineStats)],
        "mux_engine_request_pages": [c_p, c_i32, ctypes.POINTER(c_i32), c_p, c_i32, ctypes.POINTER(c_i32)],
        "mux_engine_trace": [c_p, c_p, c_i32, ctypes.POINTER(c_i32)],
        "mux_engine_out_rows": [c_p, c_p, c_i32, ctypes.POINTER(c_i32)],
        "mux_engine_destroy": [c_p],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.mux_decode_workspace_bytes.argtypes = [c_i32, c_i32, c_i32, c_i32]
    L.mux_decode_workspace_bytes.restype = c_sz
    L.mux_outproj_ar_ws_bytes.argtypes = [c_i32, c_i32, c_i32]
    L.mux_outproj_ar_ws_bytes.restype = c_sz
    L.mux_outproj_packed_bytes.argtypes = [c_i32, c_i32]
    L.mux_outproj_packed_bytes.restype = c_sz
    L.mux_decode_num_splits.argtypes = [c_i32, c_i32, c_i32, c_p, c_i32, c_i32]
    L.mux_decode_num_splits.restype = c_i32
    L.mux_partition_configs.argtypes = [c_i32, c_i32, c_i32, c_p, c_i32]
    L.mux_partition_configs.restype = c_i32
    L.mux_num_prefill_layers.argtypes = [c_dbl, c_dbl, c_i32, c_i32]
    L.mux_num_prefill_layers.restype = c_i32
    L.mux_partition_count.argtypes = [c_p]
    L.mux_partition_count.restype = c_i32
    L.mux_device_sm_count.argtypes = [c_i32]
    L.mux_device_sm_count.restype = c_i32
    L.mux_last_error.restype = ctypes.c_char_p
    L.mux_version.restype = ctypes.c_char_p
    _lib = L
    return L


def last_error() -> str:
    return lib().mux_last_error().decode()


def _check(rc: int):
    if rc != MUX_OK:
        raise MuxError(rc, last_error())


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _np32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


# ------------------------------------------------------------------------------ pool
class Pool:
    """A paged KV pool (a1).  Storage: torch bf16 tensors [layers, pages, Hkv, 16, d] passed
    to the library (or library-owned when k/v are None)."""

    def __init__(self, num_layers: int, num_pages: int, num_kv_heads: int, head_dim: int, seed: int,
                 k=None, v=None, device_ptrs: Optional[tuple] = None):
        self.desc = PoolDesc(num_layers, num_pages, 16, num_kv_heads, head_dim, None, None, seed)
        if k is not None:
            self.desc.k_storage, self.desc.v_storage = _ptr(k), _ptr(v)
        elif device_ptrs is not None:
            self.desc.k_storage, self.desc.v_storage = device_ptrs
        self.k, self.v = k, v
        h = c_p()
        _check(lib().mux_pool_create(ctypes.byref(h), ctypes.byref(self.desc)))
        self.h = h

    def close(self):
        if self.h:
            lib().mux_pool_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def alloc(self, n: int) -> List[int]:
        out = np.zeros(max(n, 1), np.int32)
        _check(lib().mux_pool_alloc_pages(self.h, n, out.ctypes.data))
        return [int(x) for x in out[:n]]

    def share(self, ids: Sequence[int]):
        a = _np32(ids)
        _check(lib().mux_pool_share_pages(self.h, len(a), a.ctypes.data))

    def free(self, ids: Sequence[int]):
        a = _np32(ids)
        _check(lib().mux_pool_free_pages(self.h, len(a), a.ctypes.data))

    def num_free(self) -> int:
        n = c_i32()
        _check(lib().mux_pool_num_free(self.h, ctypes.byref(n)))
        return n.value

    def refcount(self, page: int) -> int:
        n = c_i32()
        _check(lib().mux_pool_refcount(self.h, page, ctypes.byref(n)))
        return n.value

    def free_list(self) -> List[int]:
        n = c_i32()
        _check(lib().mux_pool_free_list(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros(max(1, n.value), np.int32)
        _check(lib().mux_pool_free_list(self.h, out.ctypes.data, n.value, ctypes.byref(n)))
        return [int(x) for x in out[:n.value]]

    def error_flags(self, clear: bool = False) -> int:
        f = ctypes.c_uint32()
        _check(lib().mux_pool_error_flags(self.h, ctypes.byref(f), 1 if clear else 0))
        return f.value

    def page_tables(self, pages_needed: Sequence[int]):
        ind, ids = [0], []
        for n in pages_needed:
            ids.extend(self.alloc(n))
            ind.append(len(ids))
        return ind, ids


def mux_pool_create(num_layers, num_pages, num_kv_heads, head_dim, seed, k=None, v=None) -> Pool:
    return Pool(num_layers, num_pages, num_kv_heads, head_dim, seed, k, v)


# ------------------------------------------------------------------------------ batch
class Batch:
    """Batch descriptor (device CSR arrays as torch int32 tensors + host copies for validation)."""

    def __init__(self, qo_indptr, kv_len, page_indptr, page_ids, device="cuda", host_check: bool = True):
        import torch
        self.h_qo = _np32(qo_indptr)
        self.h_kv = _np32(kv_len)
        self.h_pind = _np32(page_indptr)
        self.h_pids = _np32(page_ids) if len(page_ids) else np.zeros(1, np.int32)
        self.num_seqs = len(self.h_kv)
        self.total_q = int(self.h_qo[-1])
        n = np.diff(self.h_qo)
        self.max_q = int(n.max())
        self.max_kv = int(self.h_kv.max())
        self.d_qo = torch.from_numpy(self.h_qo).to(device)
        self.d_kv = torch.from_numpy(self.h_kv).to(device)
        self.d_pind = torch.from_numpy(self.h_pind).to(device)
        self.d_pids = torch.from_numpy(self.h_pids).to(device)
        self.c = BatchC(self.num_seqs, _ptr(self.d_qo), _ptr(self.d_kv), _ptr(self.d_pind), _ptr(self.d_pids),
                        self.total_q, self.max_q, self.max_kv,
                        self.h_qo.ctypes.data if host_check else None, self.h_kv.ctypes.data if host_check else None,
                        self.h_pind.ctypes.data if host_check else None,
                        self.h_pids.ctypes.data if host_check else None)

    @property
    def ref(self):
        return ctypes.byref(self.c)


def mux_append_kv(pool: Pool, layer: int, batch: Batch, k_new, v_new, stream=None):
    _check(lib().mux_append_kv(pool.h, layer, batch.ref, _ptr(k_new), _ptr(v_new), _stream(stream)))


def mux_prefill_attn(pool: Pool, layer: int, batch: Batch, num_q_heads: int, q, o, lse=None,
                     scale: Optional[float] = None, stream=None):
    import torch
    scale = scale if scale is not None else 1.0 / float(np.sqrt(pool.desc.head_dim))
    od = MUX_DTYPE_F32 if o.dtype == torch.float32 else MUX_DTYPE_BF16
    _check(lib().mux_prefill_attn(pool.h, layer, batch.ref, num_q_heads, _ptr(q), _ptr(o), od, _ptr(lse),
                                  scale, _stream(stream)))


def mux_decode_attn(pool: Pool, layer: int, batch: Batch, num_q_heads: int, q, o, lse=None,
                    scale: Optional[float] = None, num_splits: int = 0, ws=None, stream=None, num_sms: int = 0):
    """a4 decode attention; num_sms > 0: launch sized for the partition the stream runs on
    (mux_decode_attn_sms), else for the whole device (mux_decode_attn)."""
    import torch
    scale = scale if scale is not None else 1.0 / float(np.sqrt(pool.desc.head_dim))
    od = MUX_DTYPE_F32 if o.dtype == torch.float32 else MUX_DTYPE_BF16
    ws_bytes = ws.numel() * ws.element_size() if ws is not None else 0
    if num_sms > 0:
        _check(lib().mux_decode_attn_sms(pool.h, layer, batch.ref, num_q_heads, _ptr(q), _ptr(o), od, _ptr(lse),
                                         scale, num_splits, _ptr(ws), ws_bytes, _stream(stream), num_sms))
        return
    _check(lib().mux_decode_attn(pool.h, layer, batch.ref, num_q_heads, _ptr(q), _ptr(o), od, _ptr(lse), scale,
                                 num_splits, _ptr(ws), ws_bytes, _stream(stream)))


def mux_decode_workspace_bytes(num_seqs: int, num_q_heads: int, head_dim: int, num_splits: int) -> int:
    return int(lib().mux_decode_workspace_bytes(num_seqs, num_q_heads, head_dim, num_splits))


def mux_decode_num_splits(num_seqs: int, num_kv_heads: int, max_kv: int, num_sms: int, kv_len=None,
                          head_dim: int = 128) -> int:
    """Balanced split-KV split count (include/mux.h); kv_len = the batch's contexts (host)."""
    a = _np32(kv_len) if kv_len is not None else None
    return int(lib().mux_decode_num_splits(num_seqs, num_kv_heads, head_dim, a.ctypes.data if a is not None else None,
                                           max_kv, num_sms))


def mux_partition_configs(total_sms: int, granularity: int = 16, min_side: int = 12) -> List[int]:
    n = lib().mux_partition_configs(total_sms, granularity, min_side, None, 0)
    if n < 0:
        raise MuxError(-n, last_error())
    out = np.zeros(n, np.int32)
    lib().mux_partition_configs(total_sms, granularity, min_side, out.ctypes.data, n)
    return [int(x) for x in out]


def mux_num_prefill_layers(t_decode: float, t_prefill: float, n_layers_model: int, remaining: int) -> int:
    return int(lib().mux_num_prefill_layers(t_decode, t_prefill, n_layers_model, remaining))


class PackedW:
    """A [K][N] bf16 weight re-laid out by mux_outproj_pack_w (include/mux.h).  `data` is a
    uint8 device tensor [layers][packed_bytes] (layers = 1 for a single matrix)."""

    def __init__(self, data, K: int, N: int):
        self.data, self.K, self.N = data, K, N

    @property
    def layer_bytes(self) -> int:
        return int(self.data[0].numel())


def mux_outproj_packed_bytes(K: int, N: int) -> int:
    return int(lib().mux_outproj_packed_bytes(K, N))


def mux_outproj_pack_w(w, stream=None) -> PackedW:
    """Pack w [K][N] (or [layers][K][N]) bf16 for mux_outproj / mux_side.w_o."""
    import torch
    w3 = w if w.dim() == 3 else w.unsqueeze(0)
    L_, K, N = w3.shape
    nb = mux_outproj_packed_bytes(K, N)
    out = torch.empty((L_, nb), dtype=torch.uint8, device=w.device)
    for i in range(L_):
        _check(lib().mux_outproj_pack_w(_ptr(w3[i].contiguous()), _ptr(out[i]), K, N, _stream(stream)))
    return PackedW(out, K, N)


def mux_outproj(x, w: PackedW, y, stream=None, num_sms: int = 0):
    """a7 partial GEMM: y[T][N] = x[T][K] . W[K][N] (bf16 in, fp32 accumulate, y bf16 or fp32);
    W packed by mux_outproj_pack_w."""
    import torch
    T, K = x.shape
    assert isinstance(w, PackedW), "mux_outproj takes a PackedW (mux_outproj_pack_w)"
    N = w.N
    assert K == w.K and tuple(y.shape) == (T, N)
    yd = MUX_DTYPE_F32 if y.dtype == torch.float32 else MUX_DTYPE_BF16
    _check(lib().mux_outproj_sms(_ptr(x), _ptr(w.data), _ptr(y), yd, T, K, N, _stream(stream), num_sms))


def mux_outproj_ar_ws_bytes(T: int, N: int, world: int) -> int:
    return int(lib().mux_outproj_ar_ws_bytes(T, N, world))


def _ar_peers(world: int, rank: int, epoch: int, stages, ys) -> ArPeersC:
    assert 1 <= world <= MUX_AR_MAX_WORLD and len(stages) == world and len(ys) == world
    pr = ArPeersC()
    pr.world, pr.rank, pr.epoch = world, rank, epoch
    for r in range(world):
        pr.stage[r] = stages[r] if isinstance(stages[r], int) else _ptr(stages[r])
        pr.y[r] = ys[r] if isinstance(ys[r], int) else _ptr(ys[r])
    return pr


class IpcBuffer:
    """Device memory shareable through CUDA IPC (mux_ipc_alloc); `handle` (64 bytes) maps it in
    another process with IpcBuffer.open(handle).  `tensor(shape, dtype)` views it as a torch tensor."""

    def __init__(self, nbytes: int = 0, handle: bytes | None = None):
        self.ptr = c_p()
        if handle is None:
            h = ctypes.create_string_buffer(64)
            _check(lib().mux_ipc_alloc(nbytes, ctypes.byref(self.ptr), h))
            self.handle, self.owned, self.nbytes = h.raw, True, nbytes
        else:
            _check(lib().mux_ipc_open(handle, ctypes.byref(self.ptr)))
            self.handle, self.owned, self.nbytes = handle, False, nbytes

    @classmethod
    def open(cls, handle: bytes, nbytes: int):
        return cls(nbytes, handle)

    @property
    def address(self) -> int:
        return int(self.ptr.value or 0)

    def tensor(self, shape, dtype):
        import torch
        n = 1
        for x in shape:
            n *= int(x)
        itemsize = torch.empty((), dtype=dtype).element_size()
        assert n * itemsize <= self.nbytes
        typestr = {torch.bfloat16: "<i2", torch.uint8: "|u1", torch.float32: "<f4"}[dtype]

        class _Iface:
            __cuda_array_interface__ = {"shape": tuple(int(x) for x in shape), "typestr": typestr,
                                        "data": (self.address, False), "version": 3}
        t = torch.as_tensor(_Iface(), device="cuda")
        return t.view(dtype) if dtype == torch.bfloat16 else t

    def close(self):
        if self.address:
            _check(lib().mux_ipc_free(self.ptr) if self.owned else lib().mux_ipc_close(self.ptr))
            self.ptr = c_p()


def mux_outproj_allreduce(x, w: PackedW, rank: int, epoch: int, stages, ys, stream=None, num_sms: int = 0):
    """f4: y_r = sum over ranks of x_r . W_r, the GEMM and the all-reduce in ONE kernel (include/mux.h).
    stages / ys: per-rank staging workspaces and outputs as device addresses (ints) or tensors valid
    in this process (peers' buffers mapped by CUDA IPC); epoch: shared launch counter, 1, 2, ..."""
    T, K = x.shape
    pr = _ar_peers(len(stages), rank, epoch, stages, ys)
    _check(lib().mux_outproj_allreduce(_ptr(x), _ptr(w.data), T, K, w.N, ctypes.byref(pr), num_sms,
                                       _stream(stream)))


def mux_outproj_allreduce_emulated(xs, ws, epoch: int, stages, ys, stream=None):
    """The same kernel with all len(xs) ranks' CTAs in one launch on this device (every buffer local)."""
    G = len(xs)
    T, K = xs[0].shape
    pr = _ar_peers(G, 0, epoch, stages, ys)
    xa = (c_p * G)(*[_ptr(x) for x in xs])
    wa = (c_p * G)(*[_ptr(w.data) for w in ws])
    _check(lib().mux_outproj_allreduce_emulated(xa, wa, T, K, ws[0].N, ctypes.byref(pr), _stream(stream)))


def mux_device_sm_count(device: int = 0) -> int:
    return int(lib().mux_device_sm_count(device))


def mux_stream_read(src, num_ctas: int, stream=None, nbytes: int | None = None) -> int:
    """Read-bandwidth probe (include/mux.h): stream `src` (a device tensor) through shared memory
    with 32 KiB bulk copies on `num_ctas` CTAs.  `stream`: a raw cudaStream_t (e.g. a partition
    stream from Partition.query) or None for torch's current stream.  Returns the bytes read."""
    nb = (nbytes if nbytes is not None else src.numel() * src.element_size()) // 32768 * 32768
    _check(lib().mux_stream_read(c_p(src.data_ptr()), nb, num_ctas, c_p(_stream(stream))))
    return nb


# ------------------------------------------------------------------------------ partitions
class Partition:
    def __init__(self, device: int, decode_sms: Sequence[int]):
        a = _np32(decode_sms) if len(decode_sms) else np.zeros(1, np.int32)
        h = c_p()
        _check(lib().mux_partition_create(ctypes.byref(h), device, a.ctypes.data, len(decode_sms)))
        self.h = h
        self.n = len(decode_sms)

    def query(self, idx: int):
        d, p, sd, sp = c_i32(), c_i32(), c_p(), c_p()
        _check(lib().mux_partition_query(self.h, idx, ctypes.byref(d), ctypes.byref(p), ctypes.byref(sd),
                                         ctypes.byref(sp)))
        return d.value, p.value, sd.value, sp.value

    def memory_bytes(self) -> int:
        b = c_i64()
        _check(lib().mux_partition_memory(self.h, ctypes.byref(b)))
        return b.value

    def close(self):
        if self.h:
            lib().mux_partition_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mux_partition_create(device: int, decode_sms: Sequence[int]) -> Partition:
    return Partition(device, decode_sms)


def make_side(batch: Batch, num_q_heads: int, q, o, k_new=None, v_new=None, lse=None, scale: float = 1.0,
              layer0: int = 0, num_layers: int = 1, append: bool = False, num_splits: int = 0, ws=None,
              per_layer_inputs: bool = False, w_o=None, y=None, hook=None, allreduce=None,
              attn_events=None, qkv=None, ffn=None, ar_peers=None) -> SideC:
    """Build a mux_side.  per_layer_inputs: q/k_new/v_new/o/lse carry a leading layer dim
    and layer i uses slice i (stride = one slice); otherwise every layer reuses the buffers.
    allreduce: (fn address, comm handle) of the NCCL all-reduce the library enqueues after every
    layer's out-projection (nccl.Comm.c_allreduce()).  attn_events: 2 * num_layers raw
    cudaEvent_t handles (EventSet) recorded around every layer's attention."""
    import torch

    def stride(t):
        if t is None or not per_layer_inputs:
            return 0
        return t[0].numel() * t.element_size()

    s = SideC()
    s.batch = ctypes.pointer(batch.c)
    s.num_q_heads = num_q_heads
    s.q, s.k_new, s.v_new, s.o, s.lse = _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(o), _ptr(lse)
    s.q_stride, s.kv_stride, s.o_stride, s.lse_stride = stride(q), stride(k_new), stride(o), stride(lse)
    s.o_dtype = MUX_DTYPE_F32 if o.dtype == torch.float32 else MUX_DTYPE_BF16
    s.scale = scale
    s.layer0, s.num_layers = layer0, num_layers
    s.append = 1 if append else 0
    s.num_splits = num_splits
    s.ws = _ptr(ws)
    s.ws_bytes = ws.numel() * ws.element_size() if ws is not None else 0
    if w_o is not None:
        assert isinstance(w_o, PackedW), "w_o must be packed (mux_outproj_pack_w)"
        s.w_o, s.y = _ptr(w_o.data), _ptr(y)
        s.w_stride = w_o.layer_bytes if w_o.data.shape[0] > 1 else 0
        s.y_stride = y[0].numel() * y.element_size() if y.dim() == 3 else 0
        s.hidden = int(w_o.N)
        s.y_dtype = MUX_DTYPE_F32 if y.dtype == torch.float32 else MUX_DTYPE_BF16
    cb = None
    if hook is not None:
        # hook(side, layer_index, stream_handle) -> None; enqueue work on that stream
        cb = LayerHook(lambda user, side, layer, stream: hook(int(side), int(layer), int(stream or 0)))
        s.hook = cb
    if allreduce is not None:
        s.ar_fn, s.ar_comm = allreduce
    ev_arr = None
    if attn_events is not None:
        assert len(attn_events) >= 2 * num_layers
        ev_arr = (c_p * len(attn_events))(*attn_events.handles())
        s.attn_events = ctypes.cast(ev_arr, c_p)
    if qkv is not None:   # f4: (x_in, w_qkv PackedW, rope table) -> fused projection + RoPE + append
        x_in, w_qkv, rope = qkv
        s.x_in, s.hidden_in, s.w_qkv = _ptr(x_in), int(x_in.shape[1]), _ptr(w_qkv.data)
        s.rope, s.rope_max_pos = _ptr(rope), int(rope.shape[0])
        s.append = 0
    if ffn is not None:   # f4: (w13 PackedW, w2 PackedW, h scratch, y_ffn) -> SwiGLU FFN after out-proj
        w13, w2, fh, fy = ffn
        s.w13, s.w2, s.ffn_h, s.ffn_y, s.ffn_inter = _ptr(w13.data), _ptr(w2.data), _ptr(fh), _ptr(fy), int(w13.N // 2)
    if ar_peers is not None:   # f4: (rank, epoch, stages, ys) -> out-projection + all-reduce in one kernel
        rank, epoch, stages, ys = ar_peers
        pr = _ar_peers(len(stages), rank, epoch, stages, ys)
        s.ar_peers = ctypes.addressof(pr)
        ar_peers = (ar_peers, pr)
    s._keep = (batch, q, o, k_new, v_new, lse, ws, w_o, y, cb, ev_arr, attn_events, qkv, ffn, ar_peers)
    return s


def mux_rope_table(max_pos: int, head_dim: int = 128, theta: float = 500000.0, stream=None):
    """Device RoPE table (cos, sin) [max_pos][head_dim/2] float32 pairs for mux_qkv_rope_append."""
    import torch
    t = torch.empty((max_pos, head_dim // 2, 2), dtype=torch.float32, device="cuda")
    _check(lib().mux_rope_table(_ptr(t), max_pos, head_dim, float(theta), _stream(stream)))
    return t


def mux_qkv_rope_append(pool: Pool, layer: int, batch: Batch, num_q_heads: int, x, w_qkv: "PackedW", rope, q_out,
                        stream=None):
    """f4: Y = X . W_qkv, RoPE on the q / k heads, q -> q_out (bf16), k / v -> the pool slots (one kernel)."""
    assert isinstance(w_qkv, PackedW), "w_qkv must be packed (mux_outproj_pack_w)"
    T, hidden = x.shape
    assert w_qkv.K == hidden
    _check(lib().mux_qkv_rope_append(pool.h, layer, ctypes.byref(batch.c), num_q_heads, _ptr(x), hidden,
                                     _ptr(w_qkv.data), _ptr(rope), int(rope.shape[0]), _ptr(q_out), _stream(stream)))


def mux_ffn_pack_w13(w1, w3, stream=None) -> "PackedW":
    """Weight prep of the SwiGLU FFN: W1 and W3 [hidden][inter] bf16 interleaved in 128-column blocks
    and packed (mux_ffn_pack_w13) -> PackedW of [hidden][2 inter]."""
    import torch
    hidden, inter = w1.shape
    assert tuple(w3.shape) == (hidden, inter)
    lib().mux_ffn_w13_packed_bytes.restype = c_sz
    nbytes = lib().mux_ffn_w13_packed_bytes(hidden, inter)
    out = torch.empty((1, nbytes), dtype=torch.uint8, device="cuda")
    _check(lib().mux_ffn_pack_w13(_ptr(w1), _ptr(w3), _ptr(out), hidden, inter, _stream(stream)))
    return PackedW(out, hidden, 2 * inter)


def mux_ffn_swiglu(x, w13: "PackedW", w2: "PackedW", h, y, stream=None):
    """f4 FFN: h = silu(x W1) * (x W3) (one GEMM + epilogue), y = h W2."""
    T, hidden = x.shape
    inter = w13.N // 2
    assert w13.K == hidden and w2.K == inter and w2.N == hidden
    assert tuple(h.shape) == (T, inter) and tuple(y.shape) == (T, hidden)
    _check(lib().mux_ffn_swiglu(_ptr(x), _ptr(w13.data), _ptr(w2.data), _ptr(h), _ptr(y), T, hidden, inter,
                                _stream(stream)))


def mux_side_plan(side: SideC, pool_layers: int) -> np.ndarray:
    """[(pool layer, all-reduce elements)] in the order libmux would enqueue them (host only)."""
    n = c_i32()
    _check(lib().mux_side_plan(ctypes.byref(side), pool_layers, None, 0, ctypes.byref(n)))
    out = np.zeros((max(1, n.value), 2), np.int64)
    _check(lib().mux_side_plan(ctypes.byref(side), pool_layers, out.ctypes.data, n.value, ctypes.byref(n)))
    return out[:n.value]


class EventSet:
    """n timing-enabled CUDA events as raw handles (created through the CUDA runtime torch loaded),
    for mux_side.attn_events; durations(i) = ms between events 2i and 2i+1 after a sync."""

    def __init__(self, n: int):
        import torch
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        s = torch.cuda.Stream()
        for e in self.ev:          # materialise the cudaEvent_t (torch creates it on first record)
            e.record(s)
        s.synchronize()

    def __len__(self):
        return len(self.ev)

    def handles(self):
        return [int(e.cuda_event) for e in self.ev]

    def durations_ms(self, pairs: int):
        return [self.ev[2 * i].elapsed_time(self.ev[2 * i + 1]) for i in range(pairs)]


def mux_run_layer(part: Partition, split_idx: int, pool: Pool, prefill: Optional[SideC], decode: Optional[SideC],
                  times=None, join_stream=None):
    _check(lib().mux_run_layer(part.h, split_idx, pool.h, ctypes.byref(prefill) if prefill is not None else None,
                               ctypes.byref(decode) if decode is not None else None, _ptr(times),
                               _stream(join_stream)))


# ------------------------------------------------------------------------------ engine (f1)
class Engine:
    """The bubble-less multiplex engine (include/mux.h).  src_q/k/v: device
    bf16 source rows of the synthetic activations; cost: optional costmodel.CostModel (per split
    fits in partition order) for best-fit splits and N_PL."""

    def __init__(self, part: "Partition", pool: Pool, num_q_heads: int, src_q, src_k, src_v, *,
                 scale: float, w_o: "PackedW" = None, max_decode_seqs: int = 256,
                 max_prefill_tokens: int = 16384, fixed_split: int = -2, cost=None, tbt_slo_us: float = 1e30,
                 fixed_pl: int = 0, handoff: bool = True, keep_pages: bool = False, serialize: bool = False,
                 use_graphs: bool = False, o_log=None, y_log=None, o_f32: bool = False, overlap: bool = False):
        d = EngineDesc()
        d.num_q_heads, d.scale = num_q_heads, scale
        d.src_q, d.src_k, d.src_v = _ptr(src_q), _ptr(src_k), _ptr(src_v)
        d.src_rows = int(src_q.shape[0])
        if w_o is not None:
            d.w_o, d.hidden = _ptr(w_o.data), int(w_o.N)
        d.max_decode_seqs, d.max_prefill_tokens = max_decode_seqs, max_prefill_tokens
        d.fixed_split, d.tbt_slo_us, d.fixed_pl = fixed_split, tbt_slo_us, fixed_pl
        d.handoff, d.keep_pages, d.serialize = int(handoff), int(keep_pages), int(serialize)
        d.use_graphs, d.o_f32, d.overlap = int(use_graphs), int(o_f32), int(overlap)
        if o_log is not None:
            d.o_log, d.log_rows = _ptr(o_log), int(o_log.shape[0])
            if y_log is not None:
                d.y_log = _ptr(y_log)
        self._keep = [src_q, src_k, src_v, w_o, o_log, y_log]
        if cost is not None:
            n = part.n
            dec = np.zeros((n, 3))
            pf = np.zeros((n, 4))
            sl = np.ones(n)
            for i in range(n):
                ds, ps, _, _ = part.query(i)
                dec[i] = cost.decode[ds].theta
                pf[i] = cost.prefill[ps].theta
                sl[i] = cost.max_slowdown_dec.get(ds, 1.0)
            self._cost = (np.ascontiguousarray(dec), np.ascontiguousarray(pf), np.ascontiguousarray(sl))
            d.n_cost = n
            d.dec_theta, d.pf_theta, d.dec_slowdown = (a.ctypes.data for a in self._cost)
        self.desc = d
        h = c_p()
        _check(lib().mux_engine_create(ctypes.byref(h), part.h, pool.h, ctypes.byref(d)))
        self.h = h

    def submit(self, reqs):
        """reqs: iterable of (id, cached, prompt, gen, src_base[, arrival_iter[, arrival_us]])."""
        arr = (RequestC * len(reqs))(*[RequestC(*r) for r in reqs])
        _check(lib().mux_engine_submit(self.h, arr, len(reqs)))

    def run(self) -> dict:
        st = EngineStats()
        _check(lib().mux_engine_run(self.h, ctypes.byref(st)))
        return st.as_dict()

    def request_pages(self, rid: int):
        kv, n = c_i32(), c_i32()
        _check(lib().mux_engine_request_pages(self.h, rid, ctypes.byref(kv), None, 0, ctypes.byref(n)))
        out = np.zeros(max(1, n.value), np.int32)
        _check(lib().mux_engine_request_pages(self.h, rid, ctypes.byref(kv), out.ctypes.data, n.value, ctypes.byref(n)))
        return kv.value, [int(x) for x in out[:n.value]]

    def trace(self):
        n = c_i32()
        _check(lib().mux_engine_trace(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros((max(1, n.value), 6), np.int64)
        _check(lib().mux_engine_trace(self.h, out.ctypes.data, n.value, ctypes.byref(n)))
        return out[:n.value]

    def out_rows(self):
        """[(request id, absolute position, decode?)] of the rows in o_log / y_log."""
        n = c_i32()
        _check(lib().mux_engine_out_rows(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros((max(1, n.value), 3), np.int32)
        _check(lib().mux_engine_out_rows(self.h, out.ctypes.data, n.value, ctypes.byref(n)))
        return out[:n.value]

    def close(self):
        if getattr(self, "h", None):
            lib().mux_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
