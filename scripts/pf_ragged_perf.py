"""Prefill attention timing on the BASELINE configs' prefill batches (cfg2: one 8k sequence; cfg3: four
sequences n ~ U[512, 2048] with r = 9n cached; cfg5: one 32k sequence), whole GPU (developer tool)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2504_14489_b200 as mux  # noqa: E402

for cfg in (2, 3, 5):
    wl = bench.Workload(cfg, 0, 1, layers=2)
    q, o = wl.pf_q, wl.pf_o
    run = lambda: mux.mux_prefill_attn(wl.pool, 0, wl.pf_batch, wl.Hq, q, o, None, scale=wl.scale)  # noqa: E731
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        run()
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 5 * 1e-3
    print(f"cfg{cfg} prefill n={wl.pf_spec.n} r={wl.pf_spec.r}: {t*1e6:.1f} us {wl.prefill_flops_layer()/t/1e12:.1f} TFLOP/s",
          flush=True)
    del wl
    torch.cuda.empty_cache()
