"""One decode launch with 16 CTAs (16 sequences x 4096, one split) on the full GPU: the per-SM
behaviour of a 16-SM decode partition, in a form ncu can capture (developer tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_14489_b200 as mux
Hq, Hkv, d, B, C = 32, 8, 128, 16, 4096
pages = B * C // 16 + 16
k = torch.randn((1, pages, Hkv, 16, d), device="cuda").to(torch.bfloat16)
v = torch.randn_like(k)
pool = mux.Pool(1, pages, Hkv, d, 1, k, v)
pi, pd = pool.page_tables([C // 16] * B)
b = mux.Batch(list(range(B + 1)), [C] * B, pi, pd)
q = torch.randn((B, Hq, d), device="cuda").to(torch.bfloat16)
o = torch.empty((B, Hq, d), device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    mux.mux_decode_attn(pool, 0, b, Hq, q, o, None, num_splits=1)
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    mux.mux_decode_attn(pool, 0, b, Hq, q, o, None, num_splits=1)
e.record()
torch.cuda.synchronize()
t = a.elapsed_time(e) / 10 * 1e-3
print(f"16 CTAs: {t*1e6:.1f} us  {B*C*Hkv*d*4/t/1e9:.0f} GB/s  {B*C*Hkv*d*4/t/1e9/16:.1f} GB/s/SM")
