"""Dev tool: prefill attention alone (cfg2 shapes, Llama-3-8B heads) at NPF tokens, CUDA-event timed."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14489_b200 as mux  # noqa: E402

Hq, Hkv, d = 32, 8, 128
tag = os.environ.get("TAG", "")
for n in [int(x) for x in os.environ.get("NPFS", "8192,32768").split(",")]:
    pages = (n + 15) // 16 + 16
    k = torch.randn((1, pages, Hkv, 16, d), device="cuda").to(torch.bfloat16)
    v = torch.randn((1, pages, Hkv, 16, d), device="cuda").to(torch.float16)
    pool = mux.Pool(1, pages, Hkv, d, 1, k, v)
    pi, pd = pool.page_tables([(n + 15) // 16])
    b = mux.Batch([0, n], [n], pi, pd)
    q = torch.randn((n, Hq, d), device="cuda").to(torch.bfloat16)
    o = torch.empty((n, Hq, d), device="cuda", dtype=torch.bfloat16)
    f = lambda: mux.mux_prefill_attn(pool, 0, b, Hq, q, o)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    it = 20 if n <= 8192 else 5
    best = 1e9
    for rep in range(3):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(it):
            f()
        e.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(e) / it * 1e-3)
    flops = 4 * d * Hq * (n * (n + 1) / 2)
    print(f"{tag} n={n}: {best*1e6:.1f} us {flops/best/1e12:.1f} TF/s", flush=True)
    del pool, k, v
