"""One launch each of the cfg2 prefill (n=8192) and decode (B=64 @ 4096) kernels, for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14489_b200 as mux  # noqa: E402

Hq, Hkv, d, B, C, N = 32, 8, 128, 64, 4096, int(os.environ.get("NPF", 8192))
num_pages = B * C // 16 + N // 16 + 16
k = torch.randn((1, num_pages, Hkv, 16, d), device="cuda").to(torch.bfloat16)
v = torch.randn((1, num_pages, Hkv, 16, d), device="cuda").to(torch.float16)
pool = mux.Pool(1, num_pages, Hkv, d, 1, k, v)
pi, pd = pool.page_tables([C // 16] * B)
db = mux.Batch(list(range(B + 1)), [C] * B, pi, pd)
q = torch.randn((B, Hq, d), device="cuda").to(torch.bfloat16)
o = torch.empty((B, Hq, d), device="cuda", dtype=torch.bfloat16)
ppi, ppd = pool.page_tables([N // 16])
pb = mux.Batch([0, N], [N], ppi, ppd)
qp = torch.randn((N, Hq, d), device="cuda").to(torch.bfloat16)
op = torch.empty((N, Hq, d), device="cuda", dtype=torch.bfloat16)
which = sys.argv[1] if len(sys.argv) > 1 else "both"
for _ in range(2):
    if which in ("both", "decode"):
        mux.mux_decode_attn(pool, 0, db, Hq, q, o, None, num_splits=1)
    if which in ("both", "prefill"):
        mux.mux_prefill_attn(pool, 0, pb, Hq, qp, op, None)
torch.cuda.synchronize()
print("done")
