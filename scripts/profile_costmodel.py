"""Fit MuxWise's solo-run predictors (Eq.1 / Eq.2) and the contention guard's max
slowdown to THIS library's per-layer times on B200, per SM partition.

Per split of mux_partition_configs(148) (+ the full GPU): time one attention layer (append +
attention (+ combine) + out-projection, Llama-3-8B shapes) with the other side idle, over a
grid of prefill batches (n, r) and decode batches (bs, context); fit Eq.1 / Eq.2 by NNLS on
relative error; then co-run a small grid of (prefill, decode) pairs on each split and record
per-side slowdowns.  Writes gpurun_out/costmodel.json (samples + fits + guard).

usage (GPU box): python scripts/profile_costmodel.py [--quick]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_14489_b200 as mux  # noqa: E402
from paper_2504_14489_b200 import costmodel as cm  # noqa: E402
from synth import indptr  # noqa: E402

Hq, Hkv, D, HIDDEN = 32, 8, 128, 4096
POOL_LAYERS = 2


def prefill_grid(quick):
    g = []
    for n in ([512, 2048, 8192] if quick else [256, 1024, 2048, 4096, 8192]):
        for mult in ([0, 1, 4] if n <= 4096 else [0, 1]):
            g.append(([n * mult], [n]))
    g += [([0, 0], [2048, 2048]), ([0] * 4, [1024] * 4), ([4096, 0], [512, 4096]), ([8192] * 2, [1024] * 2),
          ([0] * 8, [512] * 8), ([2000, 300, 7000], [700, 1500, 333])]
    return g


def decode_grid(quick):
    g = []
    for bs in ([16, 64, 128] if quick else [8, 32, 64, 128]):
        for ctx in [1024, 4096, 8192]:
            g.append([ctx - 1] * bs)
    rng = np.random.default_rng(7)
    for bs in (48, 96):
        g.append([int(x) - 1 for x in rng.integers(1024, 8193, size=bs)])
    return g


class Bench:
    def __init__(self):
        max_pages = 128 * 8192 // 16 + 2 * 40960 // 16 + 64
        self.k = torch.empty((POOL_LAYERS, max_pages, Hkv, 16, D), dtype=torch.bfloat16, device="cuda").normal_()
        self.v = torch.empty_like(self.k, dtype=torch.float16).normal_()   # V cache: fp16 (R25)
        self.pool = mux.Pool(POOL_LAYERS, max_pages, Hkv, D, 11, self.k, self.v)
        self.w = mux.mux_outproj_pack_w((torch.randn((Hq * D, HIDDEN), device="cuda") / 64).to(torch.bfloat16))
        self.scale = 1 / math.sqrt(D)

    def side(self, r, n, decode, num_layers, ns=0):
        L = [a + b for a, b in zip(r, n)]
        pind, pids = self.pool.page_tables([(x + 15) // 16 for x in L])
        b = mux.Batch(indptr(n), L, pind, pids)
        T = sum(n)
        q = torch.randn((T, Hq, D), device="cuda").to(torch.bfloat16)
        kn = torch.randn((T, Hkv, D), device="cuda").to(torch.bfloat16)
        vn = torch.randn((T, Hkv, D), device="cuda").to(torch.bfloat16)
        o = torch.empty((T, Hq, D), dtype=torch.bfloat16, device="cuda")
        y = torch.empty((T, HIDDEN), dtype=torch.bfloat16, device="cuda")
        ws = None
        if decode:
            wsb = mux.mux_decode_workspace_bytes(len(n), Hq, D, 64)
            ws = torch.empty(max(16, wsb), dtype=torch.uint8, device="cuda")
        s = mux.make_side(b, Hq, q, o, k_new=kn, v_new=vn, scale=self.scale, layer0=0, num_layers=num_layers,
                          append=True, num_splits=ns, ws=ws, w_o=self.w, y=y)
        return s, pids

    def free(self, pids):
        self.pool.free(pids)


def time_run(part, split, pool, pf, dc, reps):
    times = torch.zeros(4, dtype=torch.int64, device="cuda")
    mux.mux_run_layer(part, split, pool, pf, dc, times)
    torch.cuda.synchronize()
    dec, pre = [], []
    for _ in range(reps):
        mux.mux_run_layer(part, split, pool, pf, dc, times)
        torch.cuda.synchronize()
        t = times.cpu().numpy()
        dec.append((t[1] - t[0]) * 1e-3)
        pre.append((t[3] - t[2]) * 1e-3)
    return float(np.median(dec)), float(np.median(pre))  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default="gpurun_out/costmodel.json")
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    B = Bench()
    total = mux.mux_device_sm_count(0)
    configs = mux.mux_partition_configs(total, 16, 12)
    part = mux.Partition(0, configs)
    splits = list(range(len(configs))) + [-1]
    pg, dg = prefill_grid(args.quick), decode_grid(args.quick)
    LAY = 4
    samples = {"prefill": [], "decode": []}
    t0 = time.time()
    for sp in splits:
        dsms, psms, _, _ = part.query(sp)
        for r, n in pg:
            s, pids = B.side(r, n, False, LAY)
            _, tp = time_run(part, sp, B.pool, s, None, 3)
            B.free(pids)
            samples["prefill"].append({"sms": psms, "split": sp, "r": r, "n": n, "us_per_layer": tp / LAY})
        for r in dg:
            s, pids = B.side(r, [1] * len(r), True, LAY)
            td, _ = time_run(part, sp, B.pool, None, s, 3)
            B.free(pids)
            samples["decode"].append({"sms": dsms, "split": sp, "r": r, "us_per_layer": td / LAY})
        print(f"split {sp} ({dsms}/{psms}) done at {time.time() - t0:.0f}s", flush=True)

    def fits(kind):
        out = {}
        for sms in sorted({s["sms"] for s in samples[kind]}):
            rows = [s for s in samples[kind] if s["sms"] == sms]
            if kind == "prefill":
                X = np.stack([cm.prefill_features(s["r"], s["n"]) for s in rows])
            else:
                X = np.stack([cm.decode_features(s["r"]) for s in rows])
            out[sms] = cm.fit(X, np.array([s["us_per_layer"] for s in rows]))
        return out
    model = cm.CostModel(fits("prefill"), fits("decode"))

    def wave_fits(kind):   # Eq.1w / Eq.2w (costmodel.prefill_wave_features / decode_wave_features)
        out = {}
        for sms in sorted({s["sms"] for s in samples[kind]}):
            rows = [s for s in samples[kind] if s["sms"] == sms]
            X = np.stack([cm.prefill_wave_features(s["r"], s["n"], sms) if kind == "prefill"
                          else cm.decode_wave_features(s["r"], sms) for s in rows])
            f = cm.fit(X, np.array([s["us_per_layer"] for s in rows]))
            out[str(sms)] = {"theta": f.theta.tolist(), "max_dev": f.max_dev, "mean_dev": f.mean_dev, "n": f.n}
        return out
    wave = {"prefill_eq1w": wave_fits("prefill"), "decode_eq2w": wave_fits("decode")}

    # contention guard: co-run pairs on each split; side windows balanced with the solo model
    pairs_pf = [([0], [2048]), ([0], [8192]), ([8192] * 4, [1024] * 4)]
    pairs_dc = [[4095] * 64, [8191] * 128, [1023] * 32]
    guard = []
    for sp in splits[:-1]:
        dsms, psms, _, _ = part.query(sp)
        for r, n in pairs_pf:
            for rd in pairs_dc:
                tp = model.t_prefill(psms, r, n)
                td = model.t_decode(dsms, rd)
                # each side's layer count so that both windows are ~8 x the longer layer
                span = 8 * max(tp, td)
                lp, ld = max(1, round(span / tp)), max(1, round(span / td))
                s_pf, p1 = B.side(r, n, False, lp)
                s_dc, p2 = B.side(rd, [1] * len(rd), True, ld)
                iso_d, _ = time_run(part, sp, B.pool, None, s_dc, 2)
                _, iso_p = time_run(part, sp, B.pool, s_pf, None, 2)
                mx_d, mx_p = time_run(part, sp, B.pool, s_pf, s_dc, 2)
                B.free(p1)
                B.free(p2)
                guard.append({"split": sp, "dec_sms": dsms, "pf_sms": psms, "pf": [r, n], "dc_bs": len(rd),
                              "dc_ctx": rd[0] + 1, "slowdown_dec": mx_d / iso_d, "slowdown_pf": mx_p / iso_p})
        print(f"guard split {sp} done at {time.time() - t0:.0f}s", flush=True)
    for g in guard:
        model.max_slowdown_dec[g["dec_sms"]] = max(model.max_slowdown_dec.get(g["dec_sms"], 1.0), g["slowdown_dec"])
        model.max_slowdown_pf[g["pf_sms"]] = max(model.max_slowdown_pf.get(g["pf_sms"], 1.0), g["slowdown_pf"])
    out = {"model": model.to_json(), "wave_aware": wave, "samples": samples, "guard": guard,
           "shapes": {"Hq": Hq, "Hkv": Hkv, "d": D, "hidden": HIDDEN}}
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    for kind, d in (("prefill Eq.1", model.prefill), ("decode Eq.2", model.decode)):
        for sms, ft in sorted(d.items()):
            print(f"{kind} {sms:3d} SMs: theta {np.array2string(ft.theta, precision=4)} "
                  f"max dev {100 * ft.max_dev:.1f}% mean {100 * ft.mean_dev:.1f}% (n={ft.n})")
    for kind, d in wave.items():
        for sms, ft in d.items():
            print(f"{kind} {int(sms):3d} SMs: max dev {100 * ft['max_dev']:.1f}% mean {100 * ft['mean_dev']:.1f}%")
    print("max slowdown dec", model.max_slowdown_dec)
    print("max slowdown pf", model.max_slowdown_pf)
    part.close()


if __name__ == "__main__":
    main()
