import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2504_14489_b200 as mux
Hq, Hkv, d, N = 32, 8, 128, 8192
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
t = tr.view(16, 256).cpu().numpy().astype(np.int64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, -1)
print("tile  kload  vload")
for j in range(56, 64): print(j, t[10, j], t[11, j])
if os.environ.get("V6"):
    print("j | qkA sfullA passA expA pvA || qkB sfullB passB expB pvB || mma: wait_sfreeB seen | kload vload")
    for j in range(50, 64):
        print(j, "|", t[8, j], t[0, j], t[2, j], t[12, j], t[6, j], "||", t[9, j], t[1, j], t[3, j], t[13, j], t[7, j],
              "||", t[14, j], t[15, j], "|", t[10, j], t[11, j])
else:
    print("u swait0 sfull0 pass1_0 exp0 pfull0 | qk0 qkret0 pv0 || sfull1 pass1_1 exp1 pfull1 | qk1 pv1")
    for u in range(100, 128):
        print(u, t[15, u], t[0, u], t[2, u], t[12, u], t[4, u], "|", t[8, u], t[14, u], t[6, u], "||",
              t[1, u], t[3, u], t[13, u], t[5, u], "|", t[9, u], t[7, u])
