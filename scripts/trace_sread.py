"""Dev tool (trace build): per-warp timing of head B's S reads in the heaviest prefill v6 CTA:
when each of the 8 softmax warps starts waiting for S_B(j), and when its S is in registers,
relative to the lead warp's view of S_B(j) ready."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14489_b200 as mux  # noqa: E402
Hq, Hkv, d, N = 32, 8, 128, 8192
pages = N // 16 + 16
k = torch.randn((1, pages, Hkv, 16, d), device="cuda").to(torch.bfloat16)
v = torch.randn((1, pages, Hkv, 16, d), device="cuda").to(torch.float16)
pool = mux.Pool(1, pages, Hkv, d, 1, k, v)
pi, pd = pool.page_tables([N // 16])
b = mux.Batch([0, N], [N], pi, pd)
q = torch.randn((N, Hq, d), device="cuda").to(torch.bfloat16)
o = torch.empty((N, Hq, d), device="cuda", dtype=torch.bfloat16)
mux.mux_prefill_attn(pool, 0, b, Hq, q, o)
tr = torch.zeros(40 * 256, dtype=torch.int64, device="cuda")
os.environ["MUX_PF_TRACE"] = str(tr.data_ptr())
mux.mux_prefill_attn(pool, 0, b, Hq, q, o)
torch.cuda.synchronize()
t = tr.view(40, 256).cpu().numpy().astype(np.int64)
nt = 64
mid = slice(8, nt - 4)
sB = t[1, :nt]
print("warp (wq, sub): median over tiles 8-60 of [wait start, S in regs] relative to S_B(j) seen by the lead warp")
for w in range(8):
    ws = np.median((t[32 + w, :nt] - sB)[mid])
    rd = np.median((t[24 + w, :nt] - sB)[mid])
    print(f"  wq {w // 2} sub {w % 2}: wait starts {ws:7.0f}   S in registers {rd:7.0f}")
print("slowest S read", np.median((t[24:32, :nt].max(axis=0) - sB)[mid]))
# MMA issuer (events 21 loop top, 20 QK_B(j) MMAs issued, 18 PV_B(j-1) MMAs issued, 19 committed,
# 10 QK_A(j+1) S free seen, 11 K(j+1) seen, 8 QK_A issue start) relative to S_B(j) seen
for name, ev, shift in (("loop top", 21, 0), ("QK_B(j) issued", 20, 0), ("PV_B(j-1) start", 7, 0),
                        ("PV_B(j-1) MMAs issued", 18, 0), ("PV_B(j-1) committed", 19, 0), ("S free seen", 10, 0),
                        ("K(j+1) seen", 11, 0)):
    print(f"  MMA {name:24s} {np.median((t[ev, :nt] - sB)[mid]):7.0f}")
print("  MMA QK_A(j+1) issue start", np.median((t[8, 1:nt] - sB[:nt - 1])[mid]))
print("  MMA PV_A(j) start        ", np.median((t[6, :nt] - sB)[mid]))
