"""Dev tool: the fused out-proj + all-reduce kernel with G ranks emulated in one launch on ONE GPU
(cfg4 per-rank shapes) vs the G GEMMs alone.  All ranks' staging / all-gather traffic lands in one
HBM here, so this bounds the protocol's overhead on one device; it says nothing about NVLink."""
import math
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14489_b200 as mux  # noqa: E402

G, T, K, N = [int(x) for x in os.environ.get("SHAPE", "8,8192,1024,8192").split(",")]
xs = [torch.randn((T, K), device="cuda").bfloat16() for _ in range(G)]
ws = [mux.mux_outproj_pack_w((torch.randn((K, N), device="cuda") / math.sqrt(G * K)).bfloat16()) for _ in range(G)]
stages = [torch.zeros(mux.mux_outproj_ar_ws_bytes(T, N, G), dtype=torch.uint8, device="cuda") for _ in range(G)]
ys = [torch.empty((T, N), dtype=torch.bfloat16, device="cuda") for _ in range(G)]


def timed(f, it=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e-3


t_f = timed(lambda: mux.mux_outproj_allreduce_emulated(xs, ws, 0, stages, ys))
sms = mux.mux_device_sm_count(0)


def gemms():
    for r in range(G):
        mux.mux_outproj(xs[r], ws[r], ys[r])


t_g = timed(gemms)
fl = 2.0 * T * K * N * G
print(f"G={G} T={T} K={K} N={N}: fused emulated {t_f*1e6:.0f} us ({fl/t_f/1e12:.0f} TF/s), "
      f"{G} GEMMs alone (each on the whole GPU) {t_g*1e6:.0f} us ({fl/t_g/1e12:.0f} TF/s)", flush=True)
