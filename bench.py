"""bench.py — multiplexed prefill+decode attention throughput on B200 (BASELINE.json metric).

Workload (N=1): BASELINE config 2 = Llama-3-8B attention shapes (Hq=32, Hkv=8, d=128,
N_T=32 layers): one 8192-token prefill (r=0) co-running with a decode batch of 64
sequences at context 4096, on disjoint green-context SM partitions (SM-split sweep over
the 8 configs of the 16-SM rule).

A STEP is one multiplexed window through the whole hot path (all §8(a) rows):
  decode side : `iters` decode iterations x 32 layers, each layer = mux_append_kv (the
                current token) + split-KV decode attention (+ combine) + out-projection
                partial GEMM (+ NCCL all-reduce of it on the decode communicator when N > 1);
  prefill side: the 8k prefill through all 32 layers, layer by layer, each layer =
                mux_append_kv (8192 new K/V rows) + tcgen05 prefill attention + out-projection
                (+ all-reduce on the prefill communicator when N > 1),
both enqueued by ONE mux_run_layer call (decode first) on the chosen SM split.
`iters` balances the two sides with the paper's N_PL rule evaluated on the
isolated timings of that split, so neither side idles (bubble-less).

metric value = model-equivalent attention tok/s = (8192 + 64*iters) tokens / step time
(each token passes all 32 attention layers).  e2e = the same through the public API with
the step's inputs (new-token Q/K/V, one layer's worth, reused by every layer: the QKV
projections are outside this hot path) copied from pinned host memory and the last
layer's outputs copied back inside the timed region.

Multi-GPU (torchrun, N>1): KV-head sharding (§8(e)) — each rank holds Hkv/N kv heads,
Hq/N q heads and the matching rows of W_o of the same workload (strong scaling); attention
needs no collective; each layer's out-projection partial sums are all-reduced (bf16, NCCL)
on the side's own green-context stream through a per-side communicator.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "multiplexed prefill+decode tok/s per B200; decode HBM GB/s + prefill TC util"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return dict(PEAKS_FALLBACK), "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clocks and clock-event (throttle) reasons DURING the timed region: NVML
    every 20 ms (nvidia_ml_py), falling back to nvidia-smi every 200 ms."""
    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    REASON_BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
                   0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []       # (sm_mhz, max_mhz, set(reasons))
        self.source = None
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.source = "nvml 20 ms"
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                bits = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((float(sm), float(mx), {n for b, n in self.REASON_BITS.items() if bits & b}))
                self._stop.wait(0.02)
        finally:
            pynvml.nvmlShutdown()

    def _run_smi(self):
        self.source = "nvidia-smi 200 ms"
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                s = [x.strip() for x in out.split(",")]
                if len(s) >= 8 and s[0].replace(".", "").isdigit():
                    self.samples.append((float(s[0]), float(s[1]),
                                         {names[i] for i in range(4) if s[4 + i] == "Active"}))
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        try:
            self._run_nvml()
        except Exception:
            if not self._stop.is_set():
                self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"]}
        sm = [s[0] for s in self.samples]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(set().union(*[s[2] for s in self.samples])), "samples": len(self.samples),
                "sm_mhz_min": min(sm), "source": self.source}


# ----------------------------------------------------------------------------- workload
class Workload:
    """cfg2 (or another BASELINE config) laid out in one pool of N_T layers on this rank."""

    def __init__(self, cfg: int, rank: int, world: int, layers: int | None = None):
        import torch
        import paper_2504_14489_b200 as mux
        import synth
        self.mux = mux
        c = synth.get_config(cfg)
        S = c.shapes
        assert S.Hkv % world == 0, "KV-head sharding needs world | Hkv"
        self.cfg = c
        self.Hkv = S.Hkv // world
        self.Hq = S.Hq // world
        self.d = S.d
        self.layers = layers or S.n_layers_model
        self.n_layers_model = S.n_layers_model
        self.pf_spec, self.dc_spec = c.prefill, c.decode
        pages = sum(self.pf_spec.pages_needed()) + sum(self.dc_spec.pages_needed()) + 16
        self.num_pages = pages
        dev = torch.device("cuda")
        g = torch.Generator(device=dev)
        g.manual_seed(synth.BASE_SEED + 1000 * cfg + rank)
        shape = (self.layers, pages, self.Hkv, 16, self.d)
        # the cached prefix / decode context of every layer: resident synthetic KV (N(0,1) bf16)
        self.kpool = torch.empty(shape, dtype=torch.bfloat16, device=dev)
        self.vpool = torch.empty(shape, dtype=torch.bfloat16, device=dev)
        for l in range(self.layers):
            self.kpool[l].normal_(generator=g)
            self.vpool[l].normal_(generator=g)
        self.pool = mux.Pool(self.layers, pages, self.Hkv, self.d, synth.free_list_seed(cfg), self.kpool, self.vpool)
        from synth import indptr
        pi, pd = self.pool.page_tables(self.pf_spec.pages_needed())
        self.pf_batch = mux.Batch(indptr(self.pf_spec.n), self.pf_spec.L, pi, pd)
        di, dd = self.pool.page_tables(self.dc_spec.pages_needed())
        self.dc_batch = mux.Batch(indptr(self.dc_spec.n), self.dc_spec.L, di, dd)
        self.page_hash = int(np.bitwise_xor.reduce(np.array(pd + pi, dtype=np.int64) * 2654435761 % (1 << 31)))
        Tp, Bd = self.pf_spec.total_new, self.dc_spec.num_seqs

        def rnd(*s):
            return torch.randn(*s, generator=g, device=dev).to(torch.bfloat16)
        self.pf_q, self.pf_k, self.pf_v = rnd(Tp, self.Hq, self.d), rnd(Tp, self.Hkv, self.d), rnd(Tp, self.Hkv, self.d)
        self.dc_q, self.dc_k, self.dc_v = rnd(Bd, self.Hq, self.d), rnd(Bd, self.Hkv, self.d), rnd(Bd, self.Hkv, self.d)
        self.pf_o = torch.empty((Tp, self.Hq, self.d), dtype=torch.bfloat16, device=dev)
        self.dc_o = torch.empty((Bd, self.Hq, self.d), dtype=torch.bfloat16, device=dev)
        # a7: this rank's rows of W_o (N(0, 1/(Hq d)), one matrix reused by every layer) and outputs
        self.hidden = S.hidden
        w_o = (torch.randn((self.Hq * self.d, self.hidden), generator=g, device=dev) /
               math.sqrt(S.Hq * self.d)).to(torch.bfloat16)
        self.w_o = mux.mux_outproj_pack_w(w_o)  # weight prep (once, untimed): tile-packed layout
        self.pf_y = torch.empty((Tp, self.hidden), dtype=torch.bfloat16, device=dev)
        self.dc_y = torch.empty((Bd, self.hidden), dtype=torch.bfloat16, device=dev)
        self.hooks = {}
        self.scale = 1.0 / math.sqrt(self.d)
        self.ws = None

    def sides(self, part_sms_dec: int, iters: int):
        mux = self.mux
        import torch
        ns = mux.mux_decode_num_splits(self.dc_spec.num_seqs, self.Hkv, max(self.dc_spec.L), part_sms_dec,
                                       self.dc_spec.L, self.d)
        wsb = mux.mux_decode_workspace_bytes(self.dc_spec.num_seqs, self.Hq, self.d, ns)
        if self.ws is None or self.ws.numel() < wsb:
            self.ws = torch.empty(max(16, wsb), dtype=torch.uint8, device="cuda")
        pf = mux.make_side(self.pf_batch, self.Hq, self.pf_q, self.pf_o, k_new=self.pf_k, v_new=self.pf_v,
                           scale=self.scale, layer0=0, num_layers=self.layers, append=True,
                           w_o=self.w_o, y=self.pf_y, hook=self.hooks.get(1))
        dc = mux.make_side(self.dc_batch, self.Hq, self.dc_q, self.dc_o, k_new=self.dc_k, v_new=self.dc_v,
                           scale=self.scale, layer0=0, num_layers=self.layers * iters, append=True,
                           num_splits=ns, ws=self.ws, w_o=self.w_o, y=self.dc_y, hook=self.hooks.get(0))
        return pf, dc, ns

    def set_allreduce_hooks(self, comms):
        """Per-layer all-reduce of this buffer set's y on each side's own stream (a7, R23)."""
        self.hooks = {0: lambda side, layer, stream: comms[0].all_reduce_(self.dc_y, stream),
                      1: lambda side, layer, stream: comms[1].all_reduce_(self.pf_y, stream)}

    def outproj_flops_layer(self, side):
        return 2.0 * side.total_new * self.Hq * self.d * self.hidden

    # algorithmic work per layer
    def prefill_flops_layer(self):
        return sum(4 * self.d * self.Hq * (n * r + n * (n + 1) / 2) for r, n in zip(self.pf_spec.r, self.pf_spec.n))

    def decode_bytes_layer(self):
        return (sum(self.dc_spec.L) * self.Hkv * self.d * 4 + 2 * self.dc_spec.num_seqs * self.Hq * self.d * 2
                + 4 * sum(self.dc_spec.pages_needed()))

    def append_bytes_layer(self, side):
        return 2 * 2 * side.total_new * self.Hkv * self.d * 2  # read + write of K and V rows


def probe_read_bw(mux, part, wl, split, sms, nbytes=2 << 30, reps=3):
    """BW_read(k) in GB/s: mux_stream_read over `nbytes` of the K pool on split `split`'s decode
    stream (-1: the whole GPU on torch's current stream), one CTA per SM of the partition."""
    import torch
    st = torch.cuda.ExternalStream(part.query(split)[2]) if split >= 0 else torch.cuda.current_stream()
    src = wl.kpool.view(-1)
    nb = min(nbytes, src.numel() * src.element_size())
    torch.cuda.synchronize()
    mux.mux_stream_read(src, sms, st, nb)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        got = mux.mux_stream_read(src, sms, st, nb)
    b.record(st)
    torch.cuda.synchronize()
    return got * reps / (a.elapsed_time(b) * 1e-3) / 1e9


def probe_read_bw_contended(mux, part, wl, split, sms, pf_side, nbytes=2 << 30, reps=6):
    """BW_read(k) with the prefill side running: the same probe on split `split`'s decode stream
    while mux_run_layer runs the step's prefill side (32 layers, ~30 ms) on the prefill partition,
    i.e. the decode partition's read bandwidth under the mux step's HBM/L2/power contention."""
    import torch
    st = torch.cuda.ExternalStream(part.query(split)[2])
    src = wl.kpool.view(-1)
    nb = min(nbytes, src.numel() * src.element_size())
    torch.cuda.synchronize()
    mux.mux_run_layer(part, split, wl.pool, pf_side, None)     # asynchronous: prefill partition busy
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mux.mux_stream_read(src, sms, st, nb)                       # warm, inside the prefill window
    a.record(st)
    for _ in range(reps):
        got = mux.mux_stream_read(src, sms, st, nb)
    b.record(st)
    torch.cuda.synchronize()
    return got * reps / (a.elapsed_time(b) * 1e-3) / 1e9


def time_kernel_alone(mux, part, wl, split, which, reps=5):
    """Average duration (s) of ONE attention launch (prefill6 / decode kernel of layer 0) on split
    `split`'s own partition stream, nothing else running, CUDA events on that stream."""
    import torch
    _, _, sd, sp = part.query(split)
    raw = sp if which == "pf" else sd
    st = torch.cuda.ExternalStream(raw)
    if which == "pf":
        run = lambda: mux.mux_prefill_attn(wl.pool, 0, wl.pf_batch, wl.Hq, wl.pf_q, wl.pf_o, None,  # noqa: E731
                                           scale=wl.scale, stream=raw)
    else:
        dsms = part.query(split)[0]
        ns = mux.mux_decode_num_splits(wl.dc_spec.num_seqs, wl.Hkv, max(wl.dc_spec.L), dsms, wl.dc_spec.L, wl.d)
        ws = torch.empty(max(16, mux.mux_decode_workspace_bytes(wl.dc_spec.num_seqs, wl.Hq, wl.d, ns)),
                         dtype=torch.uint8, device="cuda")
        run = lambda: mux.mux_decode_attn(wl.pool, 0, wl.dc_batch, wl.Hq, wl.dc_q, wl.dc_o, None,  # noqa: E731
                                          scale=wl.scale, num_splits=ns, ws=ws, stream=raw)
    torch.cuda.synchronize()
    run()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        run()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def time_side(mux, part, split, wl, which, iters, reps=3):
    """Isolated time (s) of one side on `split` (the other side NULL)."""
    import torch
    pf, dc, _ = wl.sides(part.query(split)[0], iters)
    st = torch.cuda.current_stream()
    for _ in range(2):
        mux.mux_run_layer(part, split, wl.pool, pf if which == "pf" else None, dc if which == "dc" else None)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        mux.mux_run_layer(part, split, wl.pool, pf if which == "pf" else None, dc if which == "dc" else None)
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


# ----------------------------------------------------------------------------- reference arm (oracle)
def run_reference(args, rank, world):
    """--impl reference: the CPU oracle, as it stands, on the host cores.  Each step is the
    bounded sample of cpu_baseline_sample (a few decode sequences + sampled prefill rows of the
    same workload, one layer), extrapolated to the full step in the same metric.  Rank 0 only."""
    if rank != 0:
        return
    vals, last = [], None
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        last = cpu_baseline_sample(args.config)
        if step >= args.warmup:
            vals.append((last["value"], time.perf_counter() - t0))
    import synth
    c = synth.get_config(args.config)
    value = float(np.median([v for v, _ in vals]))
    toks = c.prefill.total_new + c.decode.num_seqs
    line = {"metric": METRIC, "value": value, "unit": "tok/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": toks / value * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": c.name, "layers": c.shapes.n_layers_model,
                                            "decode_iters_per_step": 1},
            "cpu_baseline": {"value": value, "unit": "tok/s", "cores": last["cores"], "kind": "oracle",
                             "sample": last["sample"]},
            "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "sample_wall_s_per_step": float(np.median([t for _, t in vals]))}
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(config: int):
    """The oracle on a bounded sample (~10-30 s) of the workload, scaled to model tok/s."""
    import oracle
    import synth
    from synth import SideSpec, indptr
    from oracle.alloc import OraclePagePool, build_page_tables
    c = synth.get_config(config)
    S = c.shapes
    nd = 16                                   # sample: 16 decode sequences + 128 prefill rows (~10 s)
    dspec = SideSpec(c.decode.r[:nd], c.decode.n[:nd])
    dside = synth.make_side(config, S, dspec, decode=True)
    pool = OraclePagePool(sum(dspec.pages_needed()) + 1, 1)
    ind, ids = build_page_tables(pool, dspec.pages_needed())
    k, v = oracle.empty_pool(len(ids) + 1, S.Hkv, S.d, poison=False)
    oracle.append(k, v, np.concatenate(dside.k_rows), np.concatenate(dside.v_rows), indptr(dspec.L),
                  np.array(dspec.L, np.int32), np.array(ind, np.int32), np.array(ids, np.int32))
    t0 = time.perf_counter()
    oracle.attention(dside.q, k, v, indptr(dspec.n), np.array(dspec.L, np.int32), np.array(ind, np.int32),
                     np.array(ids, np.int32), 1 / math.sqrt(S.d))
    t_dec_tok = (time.perf_counter() - t0) / nd
    pspec = c.prefill
    pside = synth.make_side(config, S, pspec, decode=False)
    pool = OraclePagePool(sum(pspec.pages_needed()) + 1, 1)
    ind, ids = build_page_tables(pool, pspec.pages_needed())
    k, v = oracle.empty_pool(len(ids) + 1, S.Hkv, S.d, poison=False)
    oracle.append(k, v, np.concatenate(pside.k_rows), np.concatenate(pside.v_rows), indptr(pspec.L),
                  np.array(pspec.L, np.int32), np.array(ind, np.int32), np.array(ids, np.int32))
    rows = synth.sample_rows(pspec.total_new, 128)
    t0 = time.perf_counter()
    oracle.attention(pside.q, k, v, indptr(pspec.n), np.array(pspec.L, np.int32), np.array(ind, np.int32),
                     np.array(ids, np.int32), 1 / math.sqrt(S.d), rows=rows)
    t_pf = time.perf_counter() - t0
    # a causal row's cost is proportional to the keys it attends: extrapolate by keys, not rows
    key_of = np.concatenate([r + 1 + np.arange(n) for r, n in zip(pspec.r, pspec.n)])
    t_pf_all = t_pf * float(key_of.sum()) / float(key_of[rows].sum())
    t_dec_all = nd * t_dec_tok * sum(c.decode.L) / sum(dspec.L)          # decode cost ~ context
    t_layer = t_dec_all + t_pf_all
    value = (pspec.total_new + c.decode.num_seqs) / (t_layer * S.n_layers_model)
    return {"value": value, "unit": "tok/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{nd} decode seqs @ctx {c.decode.L[0]} + {len(rows)} sampled prefill rows (all heads, 1 layer), "
                      f"extrapolated by attended keys to {c.decode.num_seqs} decodes + {pspec.total_new} prefill rows "
                      f"x {S.n_layers_model} layers"}


# ----------------------------------------------------------------------------- main arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mux", choices=["mux", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--layers", type=int, default=0, help="pool layers (default: the model's N_T)")
    ap.add_argument("--split", type=int, default=-2, help="split index; -2 = sweep and pick the best")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--granularity", type=int, default=8, help="decode SM step of the split sweep")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2504_14489_b200 as mux
    mux.lib()
    peaks, peaks_src = load_peaks()

    wl = Workload(args.config, rank, world, layers=args.layers or None)
    comms = []
    if world > 1:
        # one NCCL communicator per side; each layer's out-proj partial sums are all-reduced on
        # the side's own (green-context) stream from the mux_run_layer hook
        from paper_2504_14489_b200 import nccl
        comms = [nccl.Comm(rank, world), nccl.Comm(rank, world)]
        wl.set_allreduce_hooks(comms)
    if world > 1:  # identical page tables on every rank (integer-exact check)
        h = torch.tensor([wl.page_hash], device="cuda")
        hs = [torch.zeros_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        assert all(int(x) == wl.page_hash for x in hs), "page tables differ across ranks"

    total_sms = mux.mux_device_sm_count(local)
    # decode SM counts in steps of --granularity (the paper's 16 on A100/H100, set by
    # its cluster kernels; these kernels use no clusters, and green contexts split in 8s)
    configs = mux.mux_partition_configs(total_sms, args.granularity, 12)
    part = mux.Partition(local, configs)
    # ---- calibration (untimed): isolated side times per split, N_PL balance, predicted mux rate
    sweep = []
    full_pf = time_side(mux, part, -1, wl, "pf", 1)
    full_dc = time_side(mux, part, -1, wl, "dc", 1)
    splits = range(len(configs)) if args.split == -2 else [args.split]
    for i in splits:
        dsms, psms, _, _ = part.query(i)
        t_dc = time_side(mux, part, i, wl, "dc", 1)          # one decode iteration (N_T layers)
        t_pf = time_side(mux, part, i, wl, "pf", 1)          # the whole prefill (N_T layers)
        # decode iterations per whole prefill = N_T / N_PL from the isolated times; both
        # neighbours of the ratio, and one fewer (contention slows the decode side more than the
        # prefill side in the mux window), are measured below and the fastest kept
        r = t_pf / t_dc
        for iters in sorted({max(1, math.floor(r) - 1), max(1, math.floor(r)), max(1, math.ceil(r))}):
            sweep.append({"split": i, "dec_sms": dsms, "pf_sms": psms, "t_dc_iso_ms": t_dc * 1e3,
                          "t_pf_iso_ms": t_pf * 1e3, "iters": iters})

    def measure_mux(entry, reps=3):
        i, iters = entry["split"], entry["iters"]
        pf, dc, ns = wl.sides(entry["dec_sms"], iters)
        times = torch.zeros(4, dtype=torch.int64, device="cuda")
        for _ in range(2):
            mux.mux_run_layer(part, i, wl.pool, pf, dc, times)
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            mux.mux_run_layer(part, i, wl.pool, pf, dc, times)
        b.record(st)
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / reps * 1e-3
        tt = times.cpu().numpy()
        toks = wl.pf_spec.total_new + wl.dc_spec.num_seqs * iters
        entry.update({"t_mux_ms": t * 1e3, "tok_s": toks / t,
                      "dec_side_ms": (tt[1] - tt[0]) * 1e-6, "pf_side_ms": (tt[3] - tt[2]) * 1e-6,
                      "slowdown_dec": (tt[1] - tt[0]) * 1e-9 / (entry["t_dc_iso_ms"] * 1e-3 * iters),
                      "slowdown_pf": (tt[3] - tt[2]) * 1e-9 / (entry["t_pf_iso_ms"] * 1e-3),
                      "num_splits": ns})
        return entry

    for e in sweep:
        measure_mux(e)
    best = max(sweep, key=lambda e: e["tok_s"])
    if world > 1:  # every rank must run the same split: rank 0 decides
        t = torch.tensor([sweep.index(best)], device="cuda")
        dist.broadcast(t, 0)
        best = sweep[int(t.item())]
    i, iters = best["split"], best["iters"]
    pf, dc, ns = wl.sides(best["dec_sms"], iters)
    times = torch.zeros(4, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()

    # ---- timed region: K steps (inputs resident in HBM; pool per layer >> L2)
    for _ in range(args.warmup):
        mux.mux_run_layer(part, i, wl.pool, pf, dc, times)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    side_ms = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        a.record(st)
        step_ev = []
        for _ in range(args.steps):
            mux.mux_run_layer(part, i, wl.pool, pf, dc, times)
            step_ev.append(torch.cuda.Event(enable_timing=True))
            step_ev[-1].record(st)
        b.record(st)
        torch.cuda.synchronize()
    tt = times.cpu().numpy()
    t_step = a.elapsed_time(b) / args.steps * 1e-3
    step_ms = [a.elapsed_time(step_ev[0])] + [step_ev[k - 1].elapsed_time(step_ev[k]) for k in range(1, len(step_ev))]
    if world > 1:
        tm = torch.tensor([t_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        t_step = float(tm.item())
        dist.barrier()
    toks = wl.pf_spec.total_new + wl.dc_spec.num_seqs * iters
    value = toks / t_step  # tokens are whole-model tokens (all N_T layers); aggregate over ranks (head shards)

    # ---- e2e through the public API: every step copies its inputs (new-token Q/K/V) from pinned
    # host memory and its outputs (y of both sides) back.  Double-buffered like a server: step
    # k+1's H2D and step k's D2H run on a copy stream while step k computes.
    import copy as _copy
    names_in = ("pf_q", "pf_k", "pf_v", "dc_q", "dc_k", "dc_v")
    pin = {k: getattr(wl, k).cpu().pin_memory() for k in names_in}
    wl2 = _copy.copy(wl)                                   # second I/O buffer set, same pool / batches / W_o
    for k in names_in + ("pf_o", "dc_o", "pf_y", "dc_y"):
        setattr(wl2, k, torch.empty_like(getattr(wl, k)))
    wl2.ws = None
    if comms:
        wl2.set_allreduce_hooks(comms)
    sets = [wl, wl2]
    sides2 = [(pf, dc), wl2.sides(best["dec_sms"], iters)[:2]]
    outs = [[torch.empty(w.pf_y.shape, dtype=w.pf_y.dtype).pin_memory(),
             torch.empty(w.dc_y.shape, dtype=w.dc_y.dtype).pin_memory()] for w in sets]
    h2d = sum(t.numel() * t.element_size() for t in pin.values())
    d2h = sum(t.numel() * t.element_size() for t in outs[0])
    cs = torch.cuda.Stream()
    ev_in = [torch.cuda.Event(), torch.cuda.Event()]
    ev_done = [torch.cuda.Event(), torch.cuda.Event()]
    ev_out = [torch.cuda.Event(), torch.cuda.Event()]

    def h2d_into(k):
        with torch.cuda.stream(cs):
            cs.wait_event(ev_out[k])                         # set k's last outputs are back on the host
            for n, t in pin.items():
                getattr(sets[k], n).copy_(t, non_blocking=True)
            ev_in[k].record(cs)

    def e2e_run(steps):
        cs.wait_stream(st)
        h2d_into(0)
        for step in range(steps):
            c = step % 2
            if step + 1 < steps:
                h2d_into(1 - c)                              # prefetch the next step's inputs
            st.wait_event(ev_in[c])
            mux.mux_run_layer(part, i, wl.pool, sides2[c][0], sides2[c][1], times)
            ev_done[c].record(st)
            with torch.cuda.stream(cs):
                cs.wait_event(ev_done[c])
                outs[c][0].copy_(sets[c].pf_y, non_blocking=True)
                outs[c][1].copy_(sets[c].dc_y, non_blocking=True)
                ev_out[c].record(cs)
        st.wait_stream(cs)

    for e in ev_out:
        e.record(cs)
    e2e_run(2)
    torch.cuda.synchronize()
    a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a2.record(st)
    e2e_run(args.steps)
    b2.record(st)
    torch.cuda.synchronize()
    t_e2e = a2.elapsed_time(b2) / args.steps * 1e-3
    if world > 1:
        tm = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        t_e2e = float(tm.item())

    # ---- rooflines (achieved = algorithmic work per launch / average launch duration)
    pf_side_s = (tt[3] - tt[2]) * 1e-9
    dc_side_s = (tt[1] - tt[0]) * 1e-9
    # a side's per-layer window holds append + attention + out-proj (+ all-reduce): the prefill
    # roofline counts both tcgen05 kernels' FLOPs over the whole window (a lower bound for each)
    pf_launch_s = pf_side_s / wl.layers
    dc_launch_s = dc_side_s / (wl.layers * iters)
    pf_tflops = (wl.prefill_flops_layer() + wl.outproj_flops_layer(wl.pf_spec)) / pf_launch_s / 1e12
    dc_gbs = wl.decode_bytes_layer() / dc_launch_s / 1e9
    tc_peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    traffic = {}
    try:
        with open(os.path.join(ROOT, "profiles", "r01s3_traffic.json")) as f:
            traffic = json.load(f)
    except Exception:
        pass
    pf_share = best["pf_sms"] / total_sms
    dc_share = best["dec_sms"] / total_sms
    # SURVEY §8(d) denominator (3): BW_read(k_d), a read-only 32 KiB bulk-copy stream (mux_stream_read)
    # on the SAME decode partition, measured here (untimed region), alone and next to the prefill side
    bw_part, bw_full = probe_read_bw(mux, part, wl, i, best["dec_sms"]), probe_read_bw(mux, part, wl, -1, total_sms)
    bw_part_mux = probe_read_bw_contended(mux, part, wl, i, best["dec_sms"], pf)
    # the dominant kernels alone on their own partitions (CUDA events on the partition stream)
    t_pf_k = time_kernel_alone(mux, part, wl, i, "pf")
    t_dc_k = time_kernel_alone(mux, part, wl, i, "dc")
    roofline = {"bound": "tensor", "kernel": "prefill side per layer: prefill6_kernel + outproj2_kernel (tcgen05)",
                "achieved": pf_tflops,
                "peak": tc_peak, "unit": "TFLOP/s", "frac": pf_tflops / tc_peak,
                "frac_of_sm_share": pf_tflops / (tc_peak * pf_share), "peak_src": f"{peaks_src} bf16_tflops_sustained",
                "traffic": (traffic.get("prefill6_kernel") or traffic.get("prefill_kernel") or {}).get("bytes"),
                "traffic_kernel": "prefill6_kernel" if "prefill6_kernel" in traffic else "prefill_kernel",
                "kernel_alone": {"kernel": "prefill6_kernel", "sms": best["pf_sms"], "launch_us": t_pf_k * 1e6,
                                 "achieved": wl.prefill_flops_layer() / t_pf_k / 1e12,
                                 "peak_burst_share": peaks["bf16_tflops"] * pf_share,
                                 "frac_of_burst_share": wl.prefill_flops_layer() / t_pf_k / 1e12
                                 / (peaks["bf16_tflops"] * pf_share),
                                 "frac_of_sustained_share": wl.prefill_flops_layer() / t_pf_k / 1e12 / (tc_peak * pf_share),
                                 "note": "5 launches of layer 0 on the prefill partition stream, nothing else running, "
                                         "right after the timed steps (same power-capped clocks); peaks scaled by the "
                                         "partition's SM share"},
                "per_launch": (f"1 layer: causal prefill attention {wl.prefill_flops_layer():.3e} FLOP + o_proj "
                               f"{wl.pf_spec.total_new}x{wl.Hq * wl.d}x{wl.hidden} {wl.outproj_flops_layer(wl.pf_spec):.3e}")}
    roofline_dec = {"bound": "hbm", "kernel": "decode_kernel", "achieved": dc_gbs, "peak": peaks["hbm_gbs"],
                    "unit": "GB/s", "frac": dc_gbs / peaks["hbm_gbs"], "peak_src": f"{peaks_src} hbm_gbs",
                    "sm_share": dc_share, "partition_read_gbs": bw_part, "full_gpu_read_gbs": bw_full,
                    "frac_of_partition_read": dc_gbs / bw_part,
                    # the same decode layer on the same partition with the prefill side idle (sweep)
                    "iso_achieved": wl.decode_bytes_layer() / (best["t_dc_iso_ms"] * 1e-3 / wl.layers) / 1e9,
                    "iso_frac_of_partition_read": wl.decode_bytes_layer() / (best["t_dc_iso_ms"] * 1e-3 / wl.layers)
                    / 1e9 / bw_part,
                    "partition_read_src": f"mux_stream_read on the {best['dec_sms']}-SM decode partition (alone)",
                    "partition_read_gbs_contended": bw_part_mux,
                    "frac_of_partition_read_contended": dc_gbs / bw_part_mux,
                    "partition_read_contended_src": "the same probe while the step's prefill side runs on the "
                                                    "prefill partition (same run, same clocks regime)",
                    "kernel_alone": {"kernel": "decode_kernel (+ combine)", "sms": best["dec_sms"],
                                     "launch_us": t_dc_k * 1e6, "achieved": wl.decode_bytes_layer() / t_dc_k / 1e9,
                                     "frac_of_partition_read": wl.decode_bytes_layer() / t_dc_k / 1e9 / bw_part},
                    "traffic": traffic.get("decode_kernel", {}).get("bytes")}
    launches_per_step = wl.layers * 3 + wl.layers * iters * (3 + (1 if ns > 1 else 0)) + 4
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) bf16 KV pool, Q/K/V; random-init shapes of Llama-3-8B attention)",
        "config": {"workload": wl.cfg.name, "layers": wl.layers, "Hq_per_rank": wl.Hq, "Hkv_per_rank": wl.Hkv,
                   "split": {"dec_sms": best["dec_sms"], "pf_sms": best["pf_sms"]}, "decode_iters_per_step": iters,
                   "decode_num_splits": ns, "parallelism": f"kv-head shard x{world}" if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (1.1 GB of KV per layer, 32 layers rotate)"},
        "roofline": roofline, "roofline_decode": roofline_dec,
        "e2e": {"value": toks / t_e2e, "unit": "tok/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches_per_step * args.steps,
        "step_ms_p10_p50_p90": [float(np.percentile(step_ms, q)) for q in (10, 50, 90)],
        "clocks": clocks,
        "iso_full_gpu_ms": {"prefill_32_layers": full_pf * 1e3, "decode_iter_32_layers": full_dc * 1e3},
        "time_sliced_tok_s": (wl.pf_spec.total_new + wl.dc_spec.num_seqs * iters) / (full_pf + iters * full_dc),
        "sweep": sweep,
        "partition_mem_bytes": part.memory_bytes(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_sample(args.config)
        except Exception as e:  # reported, never silently replaced
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    part.close()
    for c in comms:
        c.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
