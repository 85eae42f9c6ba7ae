"""One multiplexed bench step (cfg2, fixed split, DC_LAYERS decode layers) for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2504_14489_b200 as mux

split = int(os.environ.get("SPLIT", 0))
wl = bench.Workload(2, 0, 1)
part = mux.Partition(0, mux.mux_partition_configs(mux.mux_device_sm_count(0), 16, 12))
dsms = part.query(split)[0]
pf, dc, ns = wl.sides(dsms, int(os.environ.get("DC_LAYERS", 22)))
torch.cuda.synchronize()
for _ in range(int(os.environ.get("STEPS", 1))):
    mux.mux_run_layer(part, split, wl.pool, pf, dc, None)
torch.cuda.synchronize()
print("done split", split, "dec_sms", dsms, "num_splits", ns)
