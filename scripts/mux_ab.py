"""Developer A/B of one multiplexed step (not the bench): BASELINE cfg (default 2) on a fixed
split, D decode layers per step; prints step ms, mean prefill / decode attention launch us inside
the step (CUDA events on the partition streams) and the prefill attention alone on its partition."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2504_14489_b200 as mux  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--dec-sms", type=int, default=8)
ap.add_argument("--dc-layers", type=int, default=19)
ap.add_argument("--steps", type=int, default=6)
a = ap.parse_args()
wl = bench.Workload(a.config, 0, 1)
NT = wl.layers
part = mux.Partition(0, [a.dec_sms])
K = a.steps
ev_pf = [mux.EventSet(2 * NT) for _ in range(K)]
ev_dc = [mux.EventSet(2 * a.dc_layers) for _ in range(K)]
sides = [wl.sides(a.dec_sms, a.dc_layers, (k * a.dc_layers) % NT, ev_pf[k], ev_dc[k]) for k in range(K)]
times = torch.zeros((K, 4), dtype=torch.int64, device="cuda")
for k in range(3):
    mux.mux_run_layer(part, 0, wl.pool, sides[k][0], sides[k][1], times[k])
torch.cuda.synchronize()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for k in range(K):
    mux.mux_run_layer(part, 0, wl.pool, sides[k][0], sides[k][1], times[k])
e1.record(st)
torch.cuda.synchronize()
pf = np.concatenate([e.durations_ms(NT) for e in ev_pf]) * 1e3
dc = np.concatenate([e.durations_ms(a.dc_layers) for e in ev_dc]) * 1e3
tt = times.cpu().numpy()
alone = bench.time_kernel_alone(mux, part, wl, 0, "pf")[0] * 1e6
print(f"step {e0.elapsed_time(e1) / K:.2f} ms | prefill attn {pf.mean():.1f} us (alone {alone:.1f}) | "
      f"decode attn {dc.mean():.1f} us | pf side {np.mean(tt[:, 3] - tt[:, 2]) * 1e-6:.2f} ms, "
      f"dc side {np.mean(tt[:, 1] - tt[:, 0]) * 1e-6:.2f} ms")
part.close()
