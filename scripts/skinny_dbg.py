"""Time the out-proj kernels on skinny (decode-side) shapes inside a CUDA graph (no Python
launch overhead in the number).  The round-1 experiments behind the skinny kernel's stage size
(k-blocks per stage 1/2/4, loads or MMAs disabled, X by cp.async instead of TMA) used this
script with temporary switches in outproj.cu; results are in profiles/r01_summary.md."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_14489_b200 as mux
for T, K, N in ((64, 4096, 4096), (64, 4096, 16384), (128, 4096, 4096)):
    x = torch.randn((T, K), device="cuda").to(torch.bfloat16)
    w = (torch.randn((K, N), device="cuda") / 64).to(torch.bfloat16)
    wp = mux.mux_outproj_pack_w(w)
    y = torch.empty((T, N), device="cuda", dtype=torch.float32)
    for _ in range(3):
        mux.mux_outproj(x, wp, y)
    torch.cuda.synchronize()
    err = (y - x.float() @ w.float()).abs().max().item()
    # CUDA graph of 20 launches: the kernel time without the Python launch overhead
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                mux.mux_outproj(x, wp, y, stream=s)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 20 * 1e-3
    print(f"T={T} N={N}: {t*1e6:.1f} us ({K*N*2/t/1e9:.0f} GB/s W) err {err:.2g}", end="; ")
