"""Dev tool: cycle trace of the heaviest prefill CTA (qt = last tile, heads 0/1) at cfg2 size."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14489_b200 as mux
Hq, Hkv, d, N = 32, 8, 128, int(os.environ.get("NPF", 8192))
pages = N // 16 + 16
k = torch.randn((1, pages, Hkv, 16, d), device="cuda").to(torch.bfloat16)
v = torch.randn((1, pages, Hkv, 16, d), device="cuda").to(torch.bfloat16)
pool = mux.Pool(1, pages, Hkv, d, 1, k, v)
pi, pd = pool.page_tables([N // 16])
b = mux.Batch([0, N], [N], pi, pd)
q = torch.randn((N, Hq, d), device="cuda").to(torch.bfloat16)
o = torch.empty((N, Hq, d), device="cuda", dtype=torch.bfloat16)
mux.mux_prefill_attn(pool, 0, b, Hq, q, o)
tr = torch.zeros(16 * 256, dtype=torch.int64, device="cuda")
os.environ["MUX_PF_TRACE"] = str(tr.data_ptr())
mux.mux_prefill_attn(pool, 0, b, Hq, q, o)
torch.cuda.synchronize()
del os.environ["MUX_PF_TRACE"]
t = tr.view(16, 256).cpu().numpy().astype(np.int64)
nt = (N + 63) // 64  # sub-tiles (v5: 64-key S sub-tiles)
t0 = t[t > 0].min()
names = ["sfull0", "sfull1", "pass1_0", "pass1_1", "pfull0", "pfull1", "pv0", "pv1", "qk0", "qk1", "kload", "vload", "exp0", "exp1", "qkret0", "swait0"]
print("j " + " ".join(f"{n:>8s}" for n in names))
for j in list(range(0, 6)) + list(range(nt - 4, nt)):
    print(f"{j:2d} " + " ".join(f"{(t[e, j] - t0) if t[e, j] else -1:8d}" for e in range(16)))
sf = t[0, 1:nt] - t[0, :nt - 1]
print("period sfull0 median", np.median(sf[5:]), "softmax0 (sfull->pfull) median", np.median((t[4] - t[0])[5:nt]),
      "pass1 median", np.median((t[2] - t[0])[5:nt]), "pfull0->pv0", np.median((t[6] - t[4])[5:nt]),
      "pv0->sfull0(next)", np.median((t[0, 6:nt] - t[6, 5:nt - 1])),
      "pass1->exp", np.median((t[12] - t[2])[5:nt]), "exp->pfull", np.median((t[4] - t[12])[5:nt]), "vload->conv", np.median((t[14] - t[11])[5:nt]), "conv->pfull0", np.median((t[4] - t[14])[5:nt]))
