"""Multi-process (gloo, world_size 2, CPU) tests of the KV-head-sharded path's host logic:
shard ranges, replicated page tables (hash all-gather), and that sharded attention + sharded
out-projection + all-reduce reproduces the unsharded oracle result."""
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2504_14489_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from synth import Shapes, SideSpec
        from tests.helpers import oracle_build_side
        Hq, Hkv, d, hidden = 8, 2, 64, 96
        spec = SideSpec([40, 0], [30, 9])
        full = synth.make_side(77, Shapes(Hq, Hkv, d, 1), spec, decode=False)
        # each rank: its kv heads / q heads of the same seeded workload
        ka, kb = shard.kv_head_range(rank, world, Hkv)
        qa, qb = shard.q_head_range(rank, world, Hq, Hkv)
        mine = synth.SideData(spec, full.q[:, qa:qb], [k[:, ka:kb] for k in full.k_rows],
                              [v[:, ka:kb] for v in full.v_rows])
        st = oracle_build_side(mine, 16, 5, kb - ka, d)
        h = shard.page_table_hash(st["page_indptr"], st["page_ids"])
        hs = [None] * world
        dist.all_gather_object(hs, h)
        o, _ = oracle.attention(mine.q, st["kpool"], st["vpool"], st["qo_indptr"], st["kv_len"],
                                st["page_indptr"], st["page_ids"], 1 / math.sqrt(d))
        g = np.random.default_rng(3)
        wo = synth.f32_to_bf16_bits((g.standard_normal((Hq * d, hidden)) / 30).astype(np.float32))
        ra, rb = shard.wo_row_range(rank, world, Hq, Hkv, d)
        y = torch.from_numpy(oracle.outproj(o.reshape(o.shape[0], -1), wo[ra:rb]))
        dist.all_reduce(y)
        if rank == 0:
            stf = oracle_build_side(full, 16, 5, Hkv, d)
            of, _ = oracle.attention(full.q, stf["kpool"], stf["vpool"], stf["qo_indptr"], stf["kv_len"],
                                     stf["page_indptr"], stf["page_ids"], 1 / math.sqrt(d))
            yf = oracle.outproj(of.reshape(of.shape[0], -1), wo)
            q.put((len(set(hs)), float(np.max(np.abs(y.numpy() - yf))), float(np.max(np.abs(of[:, qa:qb] - o)))))
    finally:
        dist.destroy_process_group()


def test_kv_head_sharded_layer_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    assert all(p.exitcode == 0 for p in ps)
    n_hashes, dy, do = q.get(timeout=5)
    assert n_hashes == 1            # identical page tables on both ranks
    assert do == 0.0                # head-sharded attention == the same heads of the full one (bitwise)
    assert dy < 1e-12               # sharded out-proj + all-reduce == unsharded O . W_o


def test_shard_ranges():
    assert shard.kv_head_range(1, 4, 8) == (2, 4)
    assert shard.q_head_range(1, 4, 64, 8) == (16, 32)
    assert shard.wo_row_range(3, 8, 64, 8, 128) == (24 * 128, 32 * 128)
    with pytest.raises(ValueError):
        shard.kv_head_range(0, 3, 8)
    assert shard.page_table_hash([0, 2], [5, 7]) != shard.page_table_hash([0, 2], [7, 5])


def _uid_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2504_14489_b200 import nccl
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        raw = bytes([(7 * i) % 5 for i in range(128)])      # binary, NULs at every 5th byte
        uid = nccl.uid_from_bytes(raw) if rank == 0 else nccl._UniqueId()
        obj = [nccl.uid_bytes(uid) if rank == 0 else None]  # the exchange nccl.Comm performs
        dist.broadcast_object_list(obj, src=0)
        got = nccl.uid_bytes(nccl.uid_from_bytes(obj[0]))
        res = [None] * world
        dist.all_gather_object(res, got == raw)
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


def test_nccl_unique_id_broadcast_keeps_binary_bytes():
    """nccl.Comm hands rank 0's ncclUniqueId to the other ranks through torch.distributed; the id
    is binary, so the bytes must survive embedded NULs (world 2, gloo)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_uid_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
    assert res == [True, True]


def _plan_worker(rank, world, port, q):
    """Each rank builds ITS shard of the cfg4 step's two sides (Hq/world q heads, hidden 8192,
    C-side all-reduce set) for 3 steps of the layer-rotating decode side, asks libmux (host dry
    run, mux_side_plan) for the collective schedule it would enqueue, and all-gathers it."""
    import torch
    import torch.distributed as dist
    import paper_2504_14489_b200 as mux
    import synth
    from synth import indptr
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = synth.get_config(4)
        S = c.shapes
        Hq = S.Hq // world
        NT = S.n_layers_model
        D = torch.tensor([37 if rank == 0 else 0])
        dist.broadcast(D, 0)                     # rank 0 decides the decode layers (as bench.py)
        D = int(D.item())
        plans = {}
        for name, spec in (("pf", c.prefill), ("dc", c.decode)):
            pages = [(l + 15) // 16 for l in spec.L]
            pind = np.concatenate([[0], np.cumsum(pages)]).astype(np.int32)
            b = mux.Batch(indptr(spec.n), spec.L, pind, np.arange(pind[-1], dtype=np.int32), device="cpu")
            x = torch.zeros((spec.total_new, Hq, S.d), dtype=torch.bfloat16)
            y = torch.zeros((spec.total_new, S.hidden), dtype=torch.bfloat16)
            w = mux.PackedW(torch.zeros((1, 16), dtype=torch.uint8), Hq * S.d, S.hidden)
            for k in range(3):
                l0, nl = (0, NT) if name == "pf" else ((k * D) % NT, D)
                side = mux.make_side(b, Hq, x, x, k_new=x, v_new=x, layer0=l0, num_layers=nl, append=True,
                                     w_o=w, y=y, allreduce=(0x1, 0x1))
                plans[(name, k)] = mux.mux_side_plan(side, NT).tolist()
        allp = [None] * world
        dist.all_gather_object(allp, plans)
        if rank == 0:
            q.put(allp)
    finally:
        dist.destroy_process_group()


def test_collective_order_identical_across_ranks():
    """NCCL needs every rank to issue the same all-reduces in the same order on each side's
    communicator: the per-side schedules libmux would enqueue (layer order, element
    counts) for three steps of the sharded cfg4 workload are identical on both gloo ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_plan_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    allp = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
    assert allp[0] == allp[1]
    pf, dc = allp[0][("pf", 0)], allp[0][("dc", 1)]
    assert [l for l, _ in pf] == list(range(80)) and all(n == 8192 * 8192 for _, n in pf)
    assert [l for l, _ in dc] == [(37 + i) % 80 for i in range(37)] and all(n == 64 * 8192 for _, n in dc)


def _peerset_worker(rank, world, port, q, fail_open_on=-1):
    """nccl.PeerSet over gloo with a host-only stand-in for the CUDA IPC buffers: every rank must
    end up with the same per-rank address table, its own buffers at its own index and every other
    rank's buffers opened from THAT rank's handles (f4 fused all-reduce peers)."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_14489_b200 import binding, nccl

        class FakeIpc:
            made = 0

            def __init__(self, nbytes=0, handle=None):
                if handle is None:
                    FakeIpc.made += 1
                    self.handle = f"r{rank}b{FakeIpc.made}".encode().ljust(64, b"\0")
                    self.owner = rank
                else:
                    self.handle, self.owner = handle, int(handle[1:2])
                self.nbytes = nbytes

            @classmethod
            def open(cls, handle, nbytes):
                if rank == fail_open_on:
                    raise OSError("peer access refused (test)")
                return cls(nbytes, handle)

            @property
            def address(self):   # a stand-in "mapped address": the allocation's identity
                return int.from_bytes(self.handle.rstrip(b"\0")[-2:], "little") + (self.owner << 32)

            def tensor(self, shape, dtype):
                return None

            def close(self):
                pass

        binding.IpcBuffer = FakeIpc
        binding.mux_outproj_ar_ws_bytes = lambda T, N, G: 4096
        import paper_2504_14489_b200.binding as b2
        assert b2.IpcBuffer is FakeIpc
        try:
            ps = nccl.PeerSet(rank, world, 300, 264)
        except RuntimeError as e:
            q.put((rank, "raised", str(e)))
            return
        rk, epoch, stages, ys = ps.peers()
        owners = [a >> 32 for a in stages] + [a >> 32 for a in ys]
        q.put((rank, rk, epoch, owners, stages, ys))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_peer_set_exchange_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3
    ps = [ctx.Process(target=_peerset_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in ps:
        item = q.get(timeout=120)
        res[item[0]] = item
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert len(res[r]) == 6, res[r]
        _, rk, epoch, owners, stages, ys = res[r]
        assert rk == r and epoch == 0
        assert owners == list(range(world)) * 2            # slot r holds rank r's buffers
        assert stages == res[0][4] and ys == res[0][5]      # the same table on every rank


def test_peer_set_failure_is_collective_gloo():
    """one rank cannot map its peers: every rank raises (none is left blocked in a collective), so
    bench.py falls back to NCCL on all ranks together"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3
    ps = [ctx.Process(target=_peerset_worker, args=(r, world, port, q, 1)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in ps:
        item = q.get(timeout=120)
        res[item[0]] = item
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert res[r][1] == "raised" and "ranks [1] failed" in res[r][2], res[r]
