"""Quick kernel timings at BASELINE config 2 sizes (developer tool, not the bench)."""
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14489_b200 as mux  # noqa: E402


def timed(fn, iters=10, stream=None):
    stream = stream or torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(iters):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e-3


def main():
    Hq, Hkv, d = 32, 8, 128
    B, C = 64, 4096
    n_pf = int(os.environ.get("NPF", 8192))
    layers = 2
    dc_pages = B * (C // 16)
    pf_pages = (n_pf + 15) // 16
    num_pages = dc_pages + pf_pages + 16
    k = torch.randn((layers, num_pages, Hkv, 16, d), device="cuda").to(torch.bfloat16)
    v = torch.randn((layers, num_pages, Hkv, 16, d), device="cuda").to(torch.float16)   # V cache: fp16 (R25)
    pool = mux.Pool(layers, num_pages, Hkv, d, 1, k, v)
    pind, pids = pool.page_tables([C // 16] * B)
    dbatch = mux.Batch(list(range(B + 1)), [C] * B, pind, pids)
    q = torch.randn((B, Hq, d), device="cuda").to(torch.bfloat16)
    o = torch.empty((B, Hq, d), device="cuda", dtype=torch.bfloat16)
    for ns in (1, 2, 4):
        wsb = mux.mux_decode_workspace_bytes(B, Hq, d, ns)
        ws = torch.empty(max(16, wsb), dtype=torch.uint8, device="cuda")
        lay = [0]

        def run():
            mux.mux_decode_attn(pool, lay[0], dbatch, Hq, q, o, None, num_splits=ns, ws=ws)
            lay[0] ^= 1
        t = timed(run)
        byts = B * C * Hkv * d * 4 + 2 * B * Hq * d * 2 + 4 * B * (C // 16)
        print(f"decode B={B} C={C} splits={ns}: {t*1e6:.1f} us  {byts/t/1e9:.0f} GB/s", flush=True)

    ppind, ppids = pool.page_tables([pf_pages])
    pbatch = mux.Batch([0, n_pf], [n_pf], ppind, ppids)
    qp = torch.randn((n_pf, Hq, d), device="cuda").to(torch.bfloat16)
    op = torch.empty((n_pf, Hq, d), device="cuda", dtype=torch.bfloat16)
    t = timed(lambda: mux.mux_prefill_attn(pool, 0, pbatch, Hq, qp, op, None), iters=5)
    flops = 4 * d * Hq * (n_pf * (n_pf + 1) / 2)
    print(f"prefill n={n_pf}: {t*1e6:.1f} us  {flops/t/1e12:.1f} TFLOP/s", flush=True)

    part = mux.Partition(0, [16, 32, 48, 64, 96])
    for i in range(5):
        dsms, psms, sd, sp = part.query(i)
        wsb = mux.mux_decode_workspace_bytes(B, Hq, d, 4)
        ws = torch.empty(max(16, wsb), dtype=torch.uint8, device="cuda")
        s_dc = mux.make_side(dbatch, Hq, q, o, scale=1 / math.sqrt(d), num_splits=0, ws=ws)
        s_pf = mux.make_side(pbatch, Hq, qp, op, scale=1 / math.sqrt(d))
        td = timed(lambda: mux.mux_run_layer(part, i, pool, None, s_dc), iters=5)
        tp = timed(lambda: mux.mux_run_layer(part, i, pool, s_pf, None), iters=3)
        tm = timed(lambda: mux.mux_run_layer(part, i, pool, s_pf, s_dc), iters=3)
        print(f"split {i}: dec {dsms} SMs {td*1e6:.0f} us | pf {psms} SMs {tp*1e6:.0f} us | mux {tm*1e6:.0f} us",
              flush=True)


if __name__ == "__main__":
    main()


def outproj_perf():
    for T, K, N in ((8192, 4096, 4096), (64, 4096, 4096), (128, 8192, 8192), (8192, 1024, 8192), (8192, 8192, 8192)):
        x = torch.randn((T, K), device="cuda").to(torch.bfloat16)
        w = (torch.randn((K, N), device="cuda") / 64).to(torch.bfloat16)
        wp = mux.mux_outproj_pack_w(w)
        y = torch.empty((T, N), device="cuda", dtype=torch.bfloat16)
        t = timed(lambda: mux.mux_outproj(x, wp, y), iters=10)
        ref = (x.float() @ w.float())
        err = (y.float() - ref).abs().max().item()
        tb = timed(lambda: torch.matmul(x, w), iters=10)
        print(f"outproj T={T} K={K} N={N}: {t*1e6:.1f} us {2*T*K*N/t/1e12:.1f} TFLOP/s (cuBLAS {2*T*K*N/tb/1e12:.1f}) max|d| {err:.3g}",
              flush=True)


if __name__ == "__main__" and os.environ.get("OUTPROJ"):
    outproj_perf()
