"""Minimal NCCL binding (ctypes over the NCCL shipped with torch) for the multi-GPU step.

torch's ProcessGroupNCCL enqueues collectives on its own internal streams; the multiplexed
engine needs each side's all-reduce of the out-projection partial sums on
that side's green-context stream, so that the NCCL kernels run on the side's own SM
partition and stay ordered after its layer's GEMM.  One communicator per side (two
concurrent collectives on one communicator from two streams could serialise or deadlock).
torch.distributed (any backend) is used only to broadcast the ncclUniqueId.
"""
from __future__ import annotations

import ctypes
import glob
import os

_lib = None

NCCL_BF16, NCCL_F32 = 9, 7
NCCL_SUM = 0


class _UniqueId(ctypes.Structure):
    _fields_ = [("internal", ctypes.c_char * 128)]


def lib():
    global _lib
    if _lib is None:
        import nvidia
        cands = []
        for p in nvidia.__path__:
            cands += glob.glob(os.path.join(p, "nccl", "lib", "libnccl.so*"))
        cands += ["libnccl.so.2"]
        last = None
        for c in cands:
            try:
                _lib = ctypes.CDLL(c)
                break
            except OSError as e:  # pragma: no cover
                last = e
        if _lib is None:
            raise ImportError(f"NCCL not found: {last}")
        _lib.ncclGetUniqueId.argtypes = [ctypes.POINTER(_UniqueId)]
        _lib.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, _UniqueId, ctypes.c_int]
        _lib.ncclAllReduce.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_void_p, ctypes.c_void_p]
        _lib.ncclCommDestroy.argtypes = [ctypes.c_void_p]
        _lib.ncclGetErrorString.restype = ctypes.c_char_p
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        raise RuntimeError(f"{what}: NCCL error {rc}: {lib().ncclGetErrorString(rc).decode()}")


def uid_bytes(uid: _UniqueId) -> bytes:
    """All 128 bytes of an ncclUniqueId (it is binary: `bytes(uid.internal)` would stop at the
    first NUL, as ctypes reads c_char arrays as C strings, and hand other ranks a corrupt id)."""
    return ctypes.string_at(ctypes.addressof(uid), ctypes.sizeof(_UniqueId))


def uid_from_bytes(b: bytes) -> _UniqueId:
    assert len(b) == ctypes.sizeof(_UniqueId), len(b)
    uid = _UniqueId()
    ctypes.memmove(ctypes.addressof(uid), b, len(b))
    return uid


class Comm:
    """A NCCL communicator over all ranks of the default torch.distributed group."""

    def __init__(self, rank: int, world: int):
        import torch.distributed as dist
        uid = _UniqueId()
        if rank == 0:
            _check(lib().ncclGetUniqueId(ctypes.byref(uid)), "ncclGetUniqueId")
        if world > 1:
            obj = [uid_bytes(uid) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = uid_from_bytes(obj[0])
        self.comm = ctypes.c_void_p()
        _check(lib().ncclCommInitRank(ctypes.byref(self.comm), world, uid, rank), "ncclCommInitRank")

    def all_reduce_(self, t, stream: int):
        """In-place sum all-reduce of tensor t, enqueued on the raw CUDA stream handle `stream`."""
        import torch
        dt = {torch.bfloat16: NCCL_BF16, torch.float32: NCCL_F32}[t.dtype]
        _check(lib().ncclAllReduce(t.data_ptr(), t.data_ptr(), t.numel(), dt, NCCL_SUM, self.comm, stream),
               "ncclAllReduce")

    def c_allreduce(self):
        """(ncclAllReduce address, comm) for mux_side.ar_fn / ar_comm: the library enqueues each
        layer's all-reduce from C on the side's stream (no Python in the layer loop)."""
        return ctypes.cast(lib().ncclAllReduce, ctypes.c_void_p).value, self.comm.value

    def close(self):
        if self.comm:
            lib().ncclCommDestroy(self.comm)
            self.comm = ctypes.c_void_p()


class PeerSet:
    """f4 fused all-reduce buffers (include/mux.h mux_outproj_allreduce): this rank's staging
    workspace and output Y allocated for CUDA IPC, their handles exchanged over the default
    torch.distributed group (any backend), and every other rank's buffers mapped into this
    process.  `peers()` gives the (rank, epoch, stages, ys) tuple for make_side(ar_peers=...)
    with epoch 0 (the kernel's own launch counter).  The fused kernel needs every rank on its
    own GPU (its CTAs wait on the other ranks' stores)."""

    def __init__(self, rank: int, world: int, T: int, N: int):
        import torch
        import torch.distributed as dist
        from .binding import IpcBuffer, mux_outproj_ar_ws_bytes
        self.rank, self.world, self.T, self.N = rank, world, T, N
        ws_bytes = mux_outproj_ar_ws_bytes(T, N, world)
        y_bytes = T * N * 2
        self.mine, self.opened = [], []
        self.stage_addr, self.y_addr, self.y_bufs = [], [], []

        def agree(ok: bool, err):
            # every rank reaches every exchange, so a failure on one rank fails all of them together
            # (a rank that raised alone would leave the others blocked in the next collective)
            if world == 1:
                if not ok:
                    raise err
                return
            flags = [None] * world
            dist.all_gather_object(flags, ok)
            if not all(flags):
                self.close()
                raise RuntimeError(f"PeerSet: ranks {[r for r, f in enumerate(flags) if not f]} failed: {err!r}")

        err = None
        try:
            self.mine = [IpcBuffer(ws_bytes), IpcBuffer(y_bytes)]
            handles = [(self.mine[0].handle, self.mine[1].handle)]
        except Exception as e:
            err, handles = e, [None]
        if world > 1:
            allh = [None] * world
            dist.all_gather_object(allh, handles[0])
            handles = allh
        agree(err is None and all(h is not None for h in handles), err)
        try:
            for r in range(world):
                if r == rank:
                    st, y = self.mine
                else:
                    st, y = IpcBuffer.open(handles[r][0], ws_bytes), IpcBuffer.open(handles[r][1], y_bytes)
                    self.opened += [st, y]
                self.stage_addr.append(st.address)
                self.y_addr.append(y.address)
                self.y_bufs.append(y)
        except Exception as e:
            err = e
        agree(err is None, err)
        self.y = self.mine[1].tensor((T, N), torch.bfloat16)   # this rank's reduced output

    def peers(self):
        return (self.rank, 0, list(self.stage_addr), list(self.y_addr))

    def close(self):
        for b in self.opened + self.mine:
            b.close()
        self.opened, self.mine, self.y_bufs = [], [], []
