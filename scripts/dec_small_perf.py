"""Decode layer time on small decode partitions (8-32 SMs) for the BASELINE decode batches:
cfg2 64 x 4096 (g = 4), cfg4 64 x 4096 with 70B heads (g = 8), cfg5 256 x 2048 (developer tool)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2504_14489_b200 as mux  # noqa: E402

part = mux.Partition(0, [8, 16, 24, 32])
for cfg in (2, 4, 5):
    wl = bench.Workload(cfg, 0, 1, layers=2)
    line = []
    for i in range(4):
        dsms, _, sd, _ = part.query(i)
        st = torch.cuda.ExternalStream(sd)
        ns = mux.mux_decode_num_splits(wl.dc_spec.num_seqs, wl.Hkv, max(wl.dc_spec.L), dsms, wl.dc_spec.L, wl.d)
        wsb = mux.mux_decode_workspace_bytes(wl.dc_spec.num_seqs, wl.Hq, wl.d, ns)
        ws = torch.empty(max(16, wsb), dtype=torch.uint8, device="cuda")
        lay = [0]

        def run():
            mux.mux_decode_attn(wl.pool, lay[0], wl.dc_batch, wl.Hq, wl.dc_q, wl.dc_o, None, num_splits=ns, ws=ws,
                                stream=sd)
            lay[0] ^= 1
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(6):
            run()
        b.record(st)
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / 6 * 1e-3
        line.append(f"{dsms} SMs {t*1e6:.0f} us ({wl.decode_bytes_layer()/t/1e9:.0f} GB/s, S={ns})")
    print(f"cfg{cfg} decode B={wl.dc_spec.num_seqs} g={wl.Hq // wl.Hkv}: " + " | ".join(line), flush=True)
    del wl
    torch.cuda.empty_cache()
