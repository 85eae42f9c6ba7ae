"""Dev tool: prefill attention alone on the prefill green context of several SM splits (cfg2 shapes)."""
import math
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14489_b200 as mux  # noqa: E402
from quick_perf import timed  # noqa: E402

Hq, Hkv, d = 32, 8, 128
n = int(os.environ.get("NPF", 8192))
pages = n // 16 + 16
k = torch.randn((1, pages, Hkv, 16, d), device="cuda").to(torch.bfloat16)
v = torch.randn((1, pages, Hkv, 16, d), device="cuda").to(torch.float16)
pool = mux.Pool(1, pages, Hkv, d, 1, k, v)
pi, pd = pool.page_tables([n // 16])
b = mux.Batch([0, n], [n], pi, pd)
q = torch.randn((n, Hq, d), device="cuda").to(torch.bfloat16)
o = torch.empty((n, Hq, d), device="cuda", dtype=torch.bfloat16)
decs = [int(x) for x in os.environ.get("DECS", "8,16,24,32").split(",")]
part = mux.Partition(0, decs)
s_pf = mux.make_side(b, Hq, q, o, scale=1 / math.sqrt(d))
flops = 4 * d * Hq * (n * (n + 1) / 2)
tag = os.environ.get("TAG", "")
for i in [-1] + list(range(len(decs))):
    if i >= 0:
        dsms, psms, _, _ = part.query(i)
    else:
        dsms, psms = 0, 148
    t = timed(lambda: mux.mux_run_layer(part, i, pool, s_pf, None), iters=10)
    print(f"{tag} split {i}: pf {psms} SMs {t*1e6:.1f} us {flops/t/1e12:.0f} TF/s  per-SM {flops/t/1e12/psms*148:.0f}", flush=True)

# cold-cache variants on split 0: each launch after an L2 flush (everything cold), or after a flush
# followed by a read of the layer's K/V (K/V in L2, Q cold: the bench's situation after append)
if os.environ.get("COLD"):
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    kv_sink = torch.empty_like(k)
    vv_sink = torch.empty_like(v)
    i = int(os.environ.get("COLD_SPLIT", 0))
    st = torch.cuda.Stream()
    for mode in ("hot", "cold", "kv_hot"):
        ts = []
        for rep in range(8):
            if mode != "hot":
                flush.zero_()
            if mode == "kv_hot":
                kv_sink.copy_(k)
                vv_sink.copy_(v)
            torch.cuda.synchronize()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            mux.mux_run_layer(part, i, pool, s_pf, None)
            e.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(e) * 1e-3)
        t = sorted(ts)[len(ts) // 2]
        print(f"{tag} split {i} {mode}: {t*1e6:.1f} us {flops/t/1e12:.0f} TF/s", flush=True)
