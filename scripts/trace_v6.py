"""Dev tool: cycle trace of the heaviest prefill v6 CTA (qt = 63, head group 0) at cfg2 size: per
128-key tile and head, when QK is issued, S is ready, the row max is done, P is written, PV issued."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14489_b200 as mux  # noqa: E402
Hq, Hkv, d, N = 32, 8, 128, 8192
pages = N // 16 + 16
k = torch.randn((1, pages, Hkv, 16, d), device="cuda").to(torch.bfloat16)
v = torch.randn((1, pages, Hkv, 16, d), device="cuda").to(torch.float16)   # V cache: fp16 (R25)
pool = mux.Pool(1, pages, Hkv, d, 1, k, v)
pi, pd = pool.page_tables([N // 16])
b = mux.Batch([0, N], [N], pi, pd)
q = torch.randn((N, Hq, d), device="cuda").to(torch.bfloat16)
o = torch.empty((N, Hq, d), device="cuda", dtype=torch.bfloat16)
mux.mux_prefill_attn(pool, 0, b, Hq, q, o)
tr = torch.zeros(24 * 256, dtype=torch.int64, device="cuda")
os.environ["MUX_PF_TRACE"] = str(tr.data_ptr())
mux.mux_prefill_attn(pool, 0, b, Hq, q, o)
torch.cuda.synchronize()
t = tr.view(24, 256).cpu().numpy().astype(np.int64)
np.save("gpurun_out/trace_v6.npy", t)
nt = 64
t0 = t[t > 0].min()
ev = {"qkA": 8, "qkB": 9, "sA": 0, "sB": 1, "maxA": 2, "maxB": 3, "expA": 12, "expB": 13, "pvA": 6, "pvB": 7}
print("j  " + " ".join(f"{n:>7s}" for n in ev))
for j in list(range(0, 4)) + list(range(30, 34)) + list(range(nt - 3, nt)):
    print(f"{j:2d} " + " ".join(f"{(t[e, j] - t0) if t[e, j] else -1:7d}" for e in ev.values()))
mid = slice(8, nt - 4)
for h, (qk, s, mx, ex, pv, pw) in enumerate([(8, 0, 2, 12, 6, 4), (9, 1, 3, 13, 7, 5)]):
    print(f"head {h}: period(S ready) {np.median(np.diff(t[s, :nt])[mid]):.0f}  qk->S {np.median((t[s]-t[qk])[mid]):.0f}"
          f"  S->max {np.median((t[mx]-t[s])[mid]):.0f}  max->P written {np.median((t[ex]-t[mx])[mid]):.0f}"
          f"  (max->PV(j-1) seen done {np.median((t[pw]-t[mx])[mid]):.0f})"
          f"  P->PV issue {np.median((t[pv]-t[ex])[mid]):.0f}")
print("B's S after A's S:", np.median((t[1] - t[0])[mid]), " A's QK(j+1) after B's S(j):",
      np.median((t[8, 1:nt] - t[1, :nt - 1])[mid]))
# producer side: K(j) / V(j) TMA issue times (after their ring slot was released)
kl, vl = t[10, :nt], t[11, :nt]
if (kl > 0).all() and (vl > 0).all():
  print("K(j) issued -> QK_A(j) issued", np.median((t[8, :nt] - kl)[mid]), " K(j) issued after QK_B(j-2) issued",
      np.median((kl[2:] - t[9, :nt - 2])[mid]))
  print("V(j) issued -> PV_A(j) issued", np.median((t[6, :nt] - vl)[mid]), " V(j) issued after PV_B(j-3) issued",
      np.median((vl[3:] - t[7, :nt - 3])[mid]))

# MMA issuer waits (v6 trace slots 10/11: QK_A(j+1) S free / K(j+1) landed; 14/15: PV_B(j-1) P ready / V ready)
if (t[10, 8:nt - 4] > 0).all():
    print("iteration j: MMA thread times relative to S_B(j) ready:")
    print("  PV_B(j-1) P_B ready", np.median((t[14, :nt] - t[1, :nt])[mid]),
          " V(j-1) ready", np.median((t[15, :nt] - t[1, :nt])[mid]),
          " PV_B(j-1) issued", np.median((t[7, :nt - 1] - t[1, 1:nt])[mid]))
    print("  QK_A(j+1) S free", np.median((t[10, :nt] - t[1, :nt])[mid]),
          " K(j+1) landed", np.median((t[11, :nt] - t[1, :nt])[mid]),
          " QK_A(j+1) issued", np.median((t[8, 1:nt] - t[1, :nt - 1])[mid]))

# producer (slots 16/17: K(j) / V(j) loads issued once their ring slot was free), relative to S_B(j)
if (t[16, 8:nt - 4] > 0).all():
    print("producer relative to S_B(j): K(j+1) issued", np.median((t[16, 1:nt] - t[1, :nt - 1])[mid]),
          " V(j) issued", np.median((t[17, :nt] - t[1, :nt])[mid]),
          " V(j+1) issued", np.median((t[17, 1:nt] - t[1, :nt - 1])[mid]))
    print("  K(j+1) issued -> landed (MMA saw it)", np.median((t[11, :nt - 1] - t[16, 1:nt])[mid]))
