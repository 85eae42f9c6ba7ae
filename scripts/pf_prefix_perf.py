"""Dev tool: prefill attention with cached prefixes (K/V beyond L2): cfg2 with an 8k prefix, a
cfg3-like multi-turn batch (r = 9 n), two long-prefix chunks; CUDA-event timed, TF/s."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14489_b200 as mux  # noqa: E402
from quick_perf import timed  # noqa: E402

Hq, Hkv, d = 32, 8, 128
tag = os.environ.get("TAG", "")
cases = {"r8k_n8k": ([8192], [8192]), "cfg3like": ([9216, 13824, 6912, 18432], [1024, 1536, 768, 2048]),
         "2x_r8k_n1k": ([8192, 8192], [1024, 1024])}
for name, (r, n) in cases.items():
    L = [a + b for a, b in zip(r, n)]
    pages = [(x + 15) // 16 for x in L]
    tot = sum(pages) + 16
    k = torch.randn((1, tot, Hkv, 16, d), device="cuda").to(torch.bfloat16)
    v = torch.randn((1, tot, Hkv, 16, d), device="cuda").to(torch.float16)
    pool = mux.Pool(1, tot, Hkv, d, 1, k, v)
    pi, pd = pool.page_tables(pages)
    qo = [0]
    for x in n:
        qo.append(qo[-1] + x)
    b = mux.Batch(qo, L, pi, pd)
    T = qo[-1]
    q = torch.randn((T, Hq, d), device="cuda").to(torch.bfloat16)
    o = torch.empty((T, Hq, d), device="cuda", dtype=torch.bfloat16)
    t = timed(lambda: mux.mux_prefill_attn(pool, 0, b, Hq, q, o), iters=5)
    flops = sum(4 * d * Hq * (nn * rr + nn * (nn + 1) / 2) for rr, nn in zip(r, n))
    print(f"{tag} {name}: {t*1e6:.1f} us {flops/t/1e12:.1f} TF/s", flush=True)
    del pool, k, v
