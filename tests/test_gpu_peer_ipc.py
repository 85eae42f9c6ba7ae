"""f4 peer buffers across processes (nccl.PeerSet over CUDA IPC, include/mux.h mux_ipc_*): two
ranks (processes, gloo for the handle exchange) on this one GPU allocate their staging / Y
buffers, exchange handles and map each other's; each writes a rank-specific pattern into the
OTHER rank's Y through the mapped address and reads it back from its own.  No kernel waits on the
other process (the fused kernel itself needs one GPU per rank; its protocol is tested with
emulated ranks in test_gpu_outproj_ar.py).  World 1: the fused kernel through PeerSet buffers."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2504_14489_b200 import nccl
        ps = nccl.PeerSet(rank, world, 300, 264)
        other = 1 - rank
        # write into the other rank's Y (peer address), then let it read its own
        ys_other = torch.full((300, 264), float(rank + 1), dtype=torch.bfloat16, device="cuda")
        ps.y_bufs[other].tensor((300, 264), torch.bfloat16).copy_(ys_other)
        torch.cuda.synchronize()
        dist.barrier()
        got = ps.y.float().cpu().numpy()
        q.put((rank, bool(np.all(got == float(other + 1)))))
        dist.barrier()
        ps.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_peer_buffers_two_processes():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


def test_peer_set_world1_fused_kernel():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2504_14489_b200 as mux
    from paper_2504_14489_b200 import nccl
    T, K, N = 300, 256, 264
    g = np.random.default_rng(5)
    x = torch.from_numpy(g.standard_normal((T, K), dtype=np.float32)).cuda().bfloat16()
    w = mux.mux_outproj_pack_w(torch.from_numpy(g.standard_normal((K, N), dtype=np.float32) / 16).cuda().bfloat16())
    ps = nccl.PeerSet(0, 1, T, N)
    ref = torch.empty((T, N), dtype=torch.bfloat16, device="cuda")
    mux.mux_outproj(x, w, ref)
    for _ in range(3):
        rank, epoch, stages, ys = ps.peers()
        mux.mux_outproj_allreduce(x, w, rank, epoch, stages, ys)
        torch.cuda.synchronize()
        assert torch.equal(ps.y.view(torch.int16), ref.view(torch.int16))
    ps.close()
