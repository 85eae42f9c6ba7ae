"""Dev tool: out-projection GEMM time vs the SM count its grid is sized for (wave quantisation)."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14489_b200 as mux  # noqa: E402
from quick_perf import timed  # noqa: E402

T, K, N = [int(x) for x in os.environ.get("SHAPE", "8192,4096,4096").split(",")]
x = torch.randn((T, K), device="cuda").bfloat16()
w = mux.mux_outproj_pack_w((torch.randn((K, N), device="cuda") / 64).bfloat16())
y = torch.empty((T, N), dtype=torch.bfloat16, device="cuda")
for sms in (148, 140, 132, 128, 116):
    t = timed(lambda: mux.mux_outproj(x, w, y, num_sms=sms), iters=20)
    print(f"T={T} K={K} N={N} grid for {sms} SMs: {t*1e6:.1f} us {2*T*K*N/t/1e12:.0f} TF/s", flush=True)
