"""bench.py — multiplexed prefill+decode attention throughput on B200 (BASELINE.json metric).

Workload (N=1): BASELINE config 2 = Llama-3-8B attention shapes (Hq=32, Hkv=8, d=128,
N_T=32 layers): one 8192-token prefill (r=0) co-running with a decode batch of 64
sequences at context 4096, on disjoint green-context SM partitions (SM-split sweep over
the 8 configs of the 16-SM rule).

A STEP is one multiplexed window through the whole hot path (all §8(a) rows):
  decode side : D decode layers of the batch, each = mux_append_kv (the current token) +
                split-KV decode attention (+ combine) + out-projection partial GEMM (+ NCCL
                all-reduce of it, enqueued by libmux on the side's stream, when N > 1); a decode
                iteration is N_T layers and step k continues at layer (k * D) mod N_T, so the
                two sides balance at LAYER granularity (the N_PL idea of P:666), not in whole
                iterations;
  prefill side: the prefill through all N_T layers, layer by layer, each layer =
                mux_append_kv (the new K/V rows) + tcgen05 prefill attention + out-projection
                (+ all-reduce on the prefill communicator when N > 1),
both enqueued by ONE mux_run_layer call (decode first) on the chosen SM split.  D is
picked from the isolated per-layer times of each split (and measured around that balance point,
since contention slows the decode side more), so neither partition idles (bubble ratio reported).

metric value = model-equivalent attention tok/s = (prefill tokens + B * D / N_T) / step time
(each prefill token passes all N_T layers; D layers of a decode batch of B are B * D / N_T
model tokens).  e2e = the same through the public API with the step's inputs (new-token Q/K/V,
one layer's worth, reused by every layer: the QKV projections are outside this hot path) copied
from pinned host memory and the last layer's outputs copied back inside the timed region.
roofline / roofline_decode: the dominant kernels' launches INSIDE the timed steps, timed by CUDA
events libmux records on the launching partition stream (mux_side.attn_events).

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
        self.vpool = torch.empty(shape, dtype=torch.float16, device=dev)   # the V cache is fp16 (R25)
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
        self.ar = {}
        self.ar_peers = {}
        self.scale = 1.0 / math.sqrt(self.d)
        self.ws = None

    def sides(self, part_sms_dec: int, dc_layers: int, dc_layer0: int = 0, pf_events=None, dc_events=None):
        """The step's two mux_sides: the prefill through all N_T layers, and `dc_layers` decode layers
        starting at pool layer dc_layer0 (a decode iteration is N_T layers; a step may end inside one
        and the next step continues it, so the two sides balance at layer granularity)."""
        mux = self.mux
        import torch
        ns = mux.mux_decode_num_splits(self.dc_spec.num_seqs, self.Hkv, max(self.dc_spec.L), part_sms_dec,
                                       self.dc_spec.L, self.d)
        wsb = mux.mux_decode_workspace_bytes(self.dc_spec.num_seqs, self.Hq, self.d, ns)
        if self.ws is None or self.ws.numel() < wsb:
            self.ws = torch.empty(max(16, wsb), dtype=torch.uint8, device="cuda")
        pf = mux.make_side(self.pf_batch, self.Hq, self.pf_q, self.pf_o, k_new=self.pf_k, v_new=self.pf_v,
                           scale=self.scale, layer0=0, num_layers=self.layers, append=True,
                           w_o=self.w_o, y=self.pf_y, allreduce=self.ar.get(1), ar_peers=self.ar_peers.get(1),
                           attn_events=pf_events)
        dc = mux.make_side(self.dc_batch, self.Hq, self.dc_q, self.dc_o, k_new=self.dc_k, v_new=self.dc_v,
                           scale=self.scale, layer0=dc_layer0 % self.layers, num_layers=dc_layers, append=True,
                           num_splits=ns, ws=self.ws, w_o=self.w_o, y=self.dc_y, allreduce=self.ar.get(0),
                           ar_peers=self.ar_peers.get(0),
                           attn_events=dc_events)
        return pf, dc, ns

    def set_allreduce(self, comms):
        """Per-layer all-reduce of each side's out-projection partial sums (a7, R23), enqueued by
        libmux from C on the side's own stream through one NCCL communicator per side."""
        self.ar = {0: comms[0].c_allreduce(), 1: comms[1].c_allreduce()}

    def set_fused_allreduce(self, rank: int, world: int):
        """f4: each layer's out-projection AND its all-reduce as ONE kernel over peer memory
        (mux_side.ar_peers, CUDA IPC buffers exchanged over torch.distributed); y lives in the
        IPC-shared buffer the other ranks store their reduced tiles into."""
        from paper_2504_14489_b200 import nccl
        self.peer_sets = [nccl.PeerSet(rank, world, self.dc_y.shape[0], self.hidden),
                          nccl.PeerSet(rank, world, self.pf_y.shape[0], self.hidden)]
        self.dc_y, self.pf_y = self.peer_sets[0].y, self.peer_sets[1].y
        self.ar_peers = {0: self.peer_sets[0].peers(), 1: self.peer_sets[1].peers()}

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


def time_kernel_alone(mux, part, wl, split, which, reps=100, warm=5):
    """Average duration (s) of ONE attention launch (prefill6 / decode kernel of layer 0) on split
    `split`'s own partition stream, nothing else running, CUDA events on that stream around `reps`
    back-to-back launches after `warm` untimed ones; returns (seconds, SM clocks sampled meanwhile)."""
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
                                          scale=wl.scale, num_splits=ns, ws=ws, stream=raw, num_sms=dsms)
    torch.cuda.synchronize()
    for _ in range(warm):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        a.record(st)
        for _ in range(reps):
            run()
        b.record(st)
        torch.cuda.synchronize()
    c = clk.summary()
    return a.elapsed_time(b) / reps * 1e-3, {"sm_mhz": c.get("sm_mhz"), "reasons": c.get("reasons")}


def time_side(mux, part, split, wl, which, dc_layers, reps=3):
    """Isolated time (s) of one side on `split` (the other side NULL)."""
    import torch
    pf, dc, _ = wl.sides(part.query(split)[0], dc_layers)
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


# ----------------------------------------------------------------------------- measurement helpers
def time_tc_share(mux, part, wl, split, pf_sms, reps=5):
    """TC(k_p): a dense bf16 GEMM (libmux's tcgen05 out-projection GEMM, T=8192 x
    K=Hq*d x N=hidden, sized for the partition's SMs) timed with CUDA events on the prefill
    partition's own stream, nothing else running.  Returns TFLOP/s."""
    import torch
    raw = part.query(split)[3] if split >= 0 else torch.cuda.current_stream().cuda_stream
    st = torch.cuda.ExternalStream(raw)
    T = 8192
    x = torch.randn((T, wl.Hq * wl.d), device="cuda").to(torch.bfloat16)
    y = torch.empty((T, wl.hidden), dtype=torch.bfloat16, device="cuda")
    torch.cuda.synchronize()
    for _ in range(2):
        mux.mux_outproj(x, wl.w_o, y, stream=raw, num_sms=pf_sms)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        mux.mux_outproj(x, wl.w_o, y, stream=raw, num_sms=pf_sms)
    b.record(st)
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / reps * 1e-3
    return 2.0 * T * wl.Hq * wl.d * wl.hidden / t / 1e12


def time_qkv_fused(mux, wl, reps=5):
    """f4: the fused QKV projection + RoPE + KV append of the step's prefill rows (T x hidden x
    (Hq + 2 Hkv) d, Llama-3 RoPE), alone on the whole GPU, CUDA events.  Not part of the step (the
    metric is the attention hot path); returns (launch seconds, FLOP per launch)."""
    import torch
    T, hidden = wl.pf_spec.total_new, wl.hidden
    N = (wl.Hq + 2 * wl.Hkv) * wl.d
    x = torch.randn((T, hidden), device="cuda").to(torch.bfloat16)
    w = mux.mux_outproj_pack_w((torch.randn((hidden, N), device="cuda") / math.sqrt(hidden)).to(torch.bfloat16))
    rope = mux.mux_rope_table(max(wl.pf_spec.L) + 1, wl.d, 500000.0)
    q_out = torch.empty((T, wl.Hq, wl.d), dtype=torch.bfloat16, device="cuda")
    run = lambda: mux.mux_qkv_rope_append(wl.pool, 0, wl.pf_batch, wl.Hq, x, w, rope, q_out)  # noqa: E731
    run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        run()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3, 2.0 * T * hidden * N


def time_ffn(mux, wl, inter=14336, reps=3):
    """f4: the layer's SwiGLU FFN (Llama-3-8B width: inter 14336) on the step's prefill rows, alone
    on the whole GPU, CUDA events.  Returns (seconds per call, FLOP per call)."""
    import torch
    T, hidden = wl.pf_spec.total_new, wl.hidden
    x = torch.randn((T, hidden), device="cuda").to(torch.bfloat16)
    w1 = (torch.randn((hidden, inter), device="cuda") / math.sqrt(hidden)).to(torch.bfloat16)
    w3 = (torch.randn((hidden, inter), device="cuda") / math.sqrt(hidden)).to(torch.bfloat16)
    w13 = mux.mux_ffn_pack_w13(w1, w3)
    w2 = mux.mux_outproj_pack_w((torch.randn((inter, hidden), device="cuda") / math.sqrt(inter)).to(torch.bfloat16))
    del w1, w3
    h = torch.empty((T, inter), dtype=torch.bfloat16, device="cuda")
    y = torch.empty((T, hidden), dtype=torch.bfloat16, device="cuda")
    mux.mux_ffn_swiglu(x, w13, w2, h, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        mux.mux_ffn_swiglu(x, w13, w2, h, y)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3, 6.0 * T * hidden * inter


def model_step(mux, part, wl, NT, tbt_slo_ms, total_sms, inter=14336, reps=3):
    """f4: the FULL transformer layer on both sides (fused QKV projection + RoPE + KV append ->
    attention -> out-projection -> SwiGLU FFN, Llama-3-8B widths; norms and residual adds, which are
    elementwise, not modelled), multiplexed like the attention step: a few decode-SM splits, D
    decode layers balancing the isolated side times, the fastest split meeting the TBT SLO.
    Reports model tok/s (the same token accounting as `value`)."""
    import torch
    T, B, hidden = wl.pf_spec.total_new, wl.dc_spec.num_seqs, wl.hidden
    N = (wl.Hq + 2 * wl.Hkv) * wl.d
    dev = "cuda"
    w_qkv = mux.mux_outproj_pack_w((torch.randn((hidden, N), device=dev) / math.sqrt(hidden)).to(torch.bfloat16))
    w1 = (torch.randn((hidden, inter), device=dev) / math.sqrt(hidden)).to(torch.bfloat16)
    w3 = (torch.randn((hidden, inter), device=dev) / math.sqrt(hidden)).to(torch.bfloat16)
    w13 = mux.mux_ffn_pack_w13(w1, w3)
    del w1, w3
    w2 = mux.mux_outproj_pack_w((torch.randn((inter, hidden), device=dev) / math.sqrt(inter)).to(torch.bfloat16))
    rope = mux.mux_rope_table(max(max(wl.pf_spec.L), max(wl.dc_spec.L)) + 1, wl.d, 500000.0)
    bufs = {k: (torch.randn((n, hidden), device=dev).to(torch.bfloat16), torch.empty((n, inter), dtype=torch.bfloat16, device=dev),
                torch.empty((n, hidden), dtype=torch.bfloat16, device=dev)) for k, n in (("pf", T), ("dc", B))}

    def sides(dsms, D, l0=0):
        pf, dc, _ = wl.sides(dsms, D, l0)
        x, h, y = bufs["pf"]
        pf = mux.make_side(wl.pf_batch, wl.Hq, wl.pf_q, wl.pf_o, scale=wl.scale, layer0=0, num_layers=NT, w_o=wl.w_o,
                           y=wl.pf_y, allreduce=wl.ar.get(1), ar_peers=wl.ar_peers.get(1), qkv=(x, w_qkv, rope),
                           ffn=(w13, w2, h, y))
        x, h, y = bufs["dc"]
        ns = mux.mux_decode_num_splits(B, wl.Hkv, max(wl.dc_spec.L), dsms, wl.dc_spec.L, wl.d)
        dc = mux.make_side(wl.dc_batch, wl.Hq, wl.dc_q, wl.dc_o, scale=wl.scale, layer0=l0 % NT, num_layers=D,
                           num_splits=ns, ws=wl.ws, w_o=wl.w_o, y=wl.dc_y, allreduce=wl.ar.get(0),
                           ar_peers=wl.ar_peers.get(0), qkv=(x, w_qkv, rope), ffn=(w13, w2, h, y))
        return pf, dc

    def timed(i, pf, dc, n=reps):
        st = torch.cuda.current_stream()
        times = torch.zeros(4, dtype=torch.int64, device=dev)
        mux.mux_run_layer(part, i, wl.pool, pf, dc, times)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(n):
            mux.mux_run_layer(part, i, wl.pool, pf, dc, times)
        b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n * 1e-3

    # the same work time-sliced on the whole GPU: prefill of all N_T layers, then the decode layers
    pf, dc = sides(total_sms, NT)
    t_pf_full, t_dc_full = timed(-1, pf, None, 2), timed(-1, None, dc, 2)
    res = []
    for i in range(part.n):
        dsms = part.query(i)[0]
        if dsms not in (16, 32, 48, 64):
            continue
        pf, dc = sides(dsms, NT)
        t_pf, t_dc = timed(i, pf, None, 2), timed(i, None, dc, 2)
        D = max(1, int(round(NT * t_pf / t_dc)))
        pf, dc = sides(dsms, D)
        t = timed(i, pf, dc, max(reps, 5))
        toks = T + B * D / NT
        res.append({"dec_sms": dsms, "dc_layers": D, "t_ms": t * 1e3, "tbt_ms": t * 1e3 * NT / D,
                    "tok_s": toks / t, "time_sliced_tok_s": toks / (t_pf_full + t_dc_full * D / NT),
                    "t_pf_iso_ms": t_pf * 1e3, "t_dc_iter_iso_ms": t_dc * 1e3})
    ok = [r for r in res if r["tbt_ms"] <= tbt_slo_ms] or res
    best = max(ok, key=lambda r: r["tok_s"])
    return {"value": best["tok_s"], "unit": "model tok/s", "split": {"dec_sms": best["dec_sms"],
            "pf_sms": total_sms - best["dec_sms"]}, "decode_layers_per_step": best["dc_layers"],
            "tbt_ms": best["tbt_ms"], "time_sliced_tok_s": best["time_sliced_tok_s"], "sweep": res,
            "full_gpu_ms": {"prefill_all_layers": t_pf_full * 1e3, "decode_iter_all_layers": t_dc_full * 1e3},
            "layer": "fused QKV + RoPE + KV append, attention, out-projection, SwiGLU FFN (inter 14336)",
            "note": "full-layer work per step; not the headline (the metric is the attention hot path)"}


def host_cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_1thread():
    """The oracle on ONE thread (OMP_NUM_THREADS=1, run in a subprocess): the whole cfg1 step (one
    layer) and the whole cfg2 decode side of one layer (64 x 4096), as model tok/s."""
    import oracle
    import synth
    from synth import indptr
    from oracle.alloc import OraclePagePool, build_page_tables
    out = {"threads": oracle.num_threads()}

    def side_time(cfg, spec, decode):
        c = synth.get_config(cfg)
        S = c.shapes
        sd = synth.make_side(cfg, S, spec, decode=decode)
        pool = OraclePagePool(sum(spec.pages_needed()) + 1, 1)
        ind, ids = build_page_tables(pool, spec.pages_needed())
        k, v = oracle.empty_pool(len(ids) + 1, S.Hkv, S.d, poison=False)
        oracle.append(k, v, np.concatenate(sd.k_rows), np.concatenate(sd.v_rows), indptr(spec.L),
                      np.array(spec.L, np.int32), np.array(ind, np.int32), np.array(ids, np.int32))
        t0 = time.perf_counter()
        oracle.attention(sd.q, k, v, indptr(spec.n), np.array(spec.L, np.int32), np.array(ind, np.int32),
                         np.array(ids, np.int32), 1 / math.sqrt(S.d))
        return time.perf_counter() - t0

    c1 = synth.get_config(1)
    t1 = side_time(1, c1.prefill, False) + side_time(1, c1.decode, True)
    out["cfg1_step_s"] = t1
    out["cfg1_tok_s"] = (c1.prefill.total_new + c1.decode.num_seqs) / t1
    c2 = synth.get_config(2)
    t2 = side_time(2, c2.decode, True)
    out["cfg2_decode_layer_s"] = t2
    out["cfg2_decode_tok_s"] = c2.decode.num_seqs / (t2 * c2.shapes.n_layers_model)
    return out


def bubble_stats(tt):
    """R21: idle share of each side's partition over the timed steps, from the
    %globaltimer stamps [steps][dec_start, dec_end, pf_start, pf_end]: per step (1 - side busy /
    step window) and over the whole region (1 - sum of side busy / first start .. last end)."""
    tt = np.asarray(tt, dtype=np.float64)
    w0 = np.minimum(tt[:, 0], tt[:, 2])
    w1 = np.maximum(tt[:, 1], tt[:, 3])
    dec, pf = tt[:, 1] - tt[:, 0], tt[:, 3] - tt[:, 2]
    step_dec = float(np.mean(1 - dec / (w1 - w0)))
    step_pf = float(np.mean(1 - pf / (w1 - w0)))
    span = w1.max() - w0.min()
    reg_dec = float(1 - dec.sum() / span)
    reg_pf = float(1 - pf.sum() / span)
    return {"bubble_ratio": (reg_dec + reg_pf) / 2, "bubble_ratio_dec": reg_dec, "bubble_ratio_pf": reg_pf,
            "per_step_dec": step_dec, "per_step_pf": step_pf,
            "def": "idle share of each side's partition between the first and last stamp of the timed "
                   "steps (P:1019-1022), averaged over the two sides; per_step_* = within each step's window"}


# ----------------------------------------------------------------------------- main arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mux", choices=["mux", "reference"])
    ap.add_argument("--config", type=int, default=0, help="BASELINE config (default: 2 at N=1, 4 at N>1)")
    ap.add_argument("--layers", type=int, default=0, help="pool layers (default: the model's N_T)")
    ap.add_argument("--split", type=int, default=-2, help="split index; -2 = sweep and pick the best")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--granularity", type=int, default=8, help="decode SM step of the split sweep")
    ap.add_argument("--tbt-slo-ms", type=float, default=0.0,
                    help="decode TBT SLO the chosen split must meet (default: P:734, 50 ms for Llama3-8B "
                         "shapes, 100 ms for Llama3-70B)")
    ap.add_argument("--no-model-step", action="store_true", help="skip the full-layer (f4) step")
    ap.add_argument("--ar", default=None, choices=["nccl", "fused"],
                    help="out-projection all-reduce: the fused GEMM + all-reduce kernel over CUDA-IPC peer "
                         "memory (f4; default at N>1, also runs at N=1), or an NCCL call per layer (a7)")
    ap.add_argument("--oracle-1thread", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.oracle_1thread:
        print(json.dumps(oracle_1thread()))
        return

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if not args.config:
        # N=1: BASELINE's single-B200 SM-split sweep config; N>1: its KV-head-sharded 70B config
        args.config = 2 if world == 1 else 4
    if not args.tbt_slo_ms:
        args.tbt_slo_ms = 100.0 if args.config == 4 else 50.0
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # communicator init lines (nranks) stay visible
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2504_14489_b200 as mux
    mux.lib()
    peaks, peaks_src = load_peaks()

    wl = Workload(args.config, rank, world, layers=args.layers or None)
    NT = wl.layers
    comms = []
    ar_note = None
    if args.ar is None:
        args.ar = "fused" if world > 1 else "nccl"
    if args.ar == "fused":
        try:
            wl.set_fused_allreduce(rank, world)
        except Exception as e:   # e.g. no CUDA IPC / peer access: every rank falls back together (PeerSet
            if world == 1:       # agrees on failures collectively) to the NCCL path, and says so
                raise
            ar_note = f"fused all-reduce unavailable ({type(e).__name__}: {e}); NCCL used"
            args.ar = "nccl"
            wl.ar_peers = {}
    if world > 1:
        if args.ar == "nccl":
            # one NCCL communicator per side; libmux enqueues each layer's all-reduce of the out-proj
            # partial sums from C on the side's own (green-context) stream (mux_side.ar_fn / ar_comm)
            from paper_2504_14489_b200 import nccl
            comms = [nccl.Comm(rank, world), nccl.Comm(rank, world)]
            wl.set_allreduce(comms)
        h = torch.tensor([wl.page_hash], device="cuda")   # identical page tables on every rank
        hs = [torch.zeros_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        assert all(int(x) == wl.page_hash for x in hs), "page tables differ across ranks"

    total_sms = mux.mux_device_sm_count(local)
    # decode SM counts in steps of --granularity (the paper's 16 on A100/H100, set by
    # its cluster kernels; these kernels use no clusters, and green contexts split in 8s)
    configs = mux.mux_partition_configs(total_sms, args.granularity, 12)
    part = mux.Partition(local, configs)
    Bd = wl.dc_spec.num_seqs

    def step_tokens(dc_layers):
        # model-equivalent tokens: every prefill token passes all N_T layers; a decode token needs
        # N_T layers, so dc_layers decode layers of a batch of Bd are Bd * dc_layers / N_T tokens
        return wl.pf_spec.total_new + Bd * dc_layers / NT

    # ---- calibration (untimed): isolated side times per split, layer-granular balance (N_PL idea,
    # decode layers per whole prefill so both partitions stay busy), measured mux rate
    sweep = []
    full_pf = time_side(mux, part, -1, wl, "pf", NT)
    full_dc = time_side(mux, part, -1, wl, "dc", NT)
    splits = range(len(configs)) if args.split == -2 else [args.split]
    for i in splits:
        dsms, psms, _, _ = part.query(i)
        t_dc = time_side(mux, part, i, wl, "dc", NT)          # one decode iteration (N_T layers)
        t_pf = time_side(mux, part, i, wl, "pf", NT)          # the whole prefill (N_T layers)
        r = t_pf / (t_dc / NT)                                 # decode layers per prefill window
        # contention slows the decode side more than the prefill side: candidates below r too
        for f in (0.7, 0.8, 0.9, 1.0):
            sweep.append({"split": i, "dec_sms": dsms, "pf_sms": psms, "t_dc_iso_ms": t_dc * 1e3,
                          "t_pf_iso_ms": t_pf * 1e3, "dc_layers": max(1, int(round(r * f)))})

    def measure_mux(entry, reps=3):
        i, D = entry["split"], entry["dc_layers"]
        pf, dc, ns = wl.sides(entry["dec_sms"], D)
        times = torch.zeros(4, dtype=torch.int64, device="cuda")
        for _ in range(2):
            mux.mux_run_layer(part, i, wl.pool, pf, dc, times)
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        evs[0].record(st)
        for r_ in range(reps):
            mux.mux_run_layer(part, i, wl.pool, pf, dc, times)
            evs[r_ + 1].record(st)
        torch.cuda.synchronize()
        # median window: one power-cap clock dip in a rep must not decide the split
        t = float(np.median([evs[r_].elapsed_time(evs[r_ + 1]) for r_ in range(reps)])) * 1e-3
        tt = times.cpu().numpy()
        entry.update({"t_mux_ms": t * 1e3, "tok_s": step_tokens(D) / t, "tbt_ms": t * 1e3 * NT / D,
                      "dec_side_ms": (tt[1] - tt[0]) * 1e-6, "pf_side_ms": (tt[3] - tt[2]) * 1e-6,
                      "slowdown_dec": (tt[1] - tt[0]) * 1e-9 / (entry["t_dc_iso_ms"] * 1e-3 * D / NT),
                      "slowdown_pf": (tt[3] - tt[2]) * 1e-9 / (entry["t_pf_iso_ms"] * 1e-3),
                      "num_splits": ns})
        return entry

    if world > 1:
        # every rank must issue the same collectives (a decode layer's all-reduce per D): the candidate
        # decode-layer counts come from rank 0's isolated timings
        dl = torch.tensor([e["dc_layers"] for e in sweep], dtype=torch.int64, device="cuda")
        dist.broadcast(dl, 0)
        for e, v in zip(sweep, dl.tolist()):
            e["dc_layers"] = int(v)
    seen = set()
    for e in list(sweep):
        key = (e["split"], e["dc_layers"])
        if key in seen:
            sweep.remove(e)
            continue
        seen.add(key)
        measure_mux(e)
    def select(cands):
        # the paper's serving objective is goodput under SLOs: the split must keep a decode token's
        # time between tokens (an iteration = N_T layers = N_T / D steps) within the TBT SLO
        # (3 % margin: the timed steps run a little slower than the calibration's three)
        ok = ([e for e in cands if e["tbt_ms"] <= 0.97 * args.tbt_slo_ms] or
              [e for e in cands if e["tbt_ms"] <= args.tbt_slo_ms] or cands)
        # bubble-less: only splits whose two sides are busy for all but <= 5 % of the window
        # on average (the idle share of the shorter side, halved); the fastest of those
        for e in cands:
            e["bubble_pred"] = 0.5 * abs(e["dec_side_ms"] - e["pf_side_ms"]) / max(e["dec_side_ms"], e["pf_side_ms"])
        ok = [e for e in ok if e["bubble_pred"] <= 0.05] or ok
        top = max(ok, key=lambda e: e["tok_s"])
        # among candidates within 1 % of the best rate, the most balanced sides
        near = [e for e in ok if e["tok_s"] >= 0.99 * top["tok_s"]]
        return min(near, key=lambda e: abs(e["dec_side_ms"] - e["pf_side_ms"]) / max(e["dec_side_ms"], e["pf_side_ms"]))

    best = select(sweep)
    # refinement on the chosen split: every decode-layer count between the coarse candidates
    # (0.7 r ... r), each re-measured over 7 windows (median); rank 0's list on every rank
    r_best = best["t_pf_iso_ms"] / (best["t_dc_iso_ms"] / NT)
    fine = list(range(max(1, int(round(0.7 * r_best))), int(round(r_best)) + 1))[:16]
    if world > 1:
        ft = torch.full((17,), -1, dtype=torch.int64, device="cuda")
        ft[0] = sweep.index(best)
        ft[1:1 + len(fine)] = torch.tensor(fine, dtype=torch.int64)
        dist.broadcast(ft, 0)
        best = sweep[int(ft[0].item())]
        fine = [int(v) for v in ft[1:].tolist() if v >= 0]
    refined = []
    for Dn in fine:
        e = {k_: best[k_] for k_ in ("split", "dec_sms", "pf_sms", "t_dc_iso_ms", "t_pf_iso_ms")}
        e["dc_layers"] = Dn
        refined.append(measure_mux(e, reps=7))
    sweep = [e for e in sweep if e["split"] != best["split"]] + refined
    best = select(sweep)
    if world > 1:  # every rank must run the same split: rank 0 decides
        t = torch.tensor([sweep.index(best)], device="cuda")
        dist.broadcast(t, 0)
        best = sweep[int(t.item())]
    i, D = best["split"], best["dc_layers"]
    st = torch.cuda.current_stream()
    K = args.steps

    # ---- timed region: K steps (inputs resident in HBM; the pool per layer is >> L2 except cfg1,
    # which flushes L2 between steps).  Step k's decode side continues at layer (k * D) mod N_T.
    # CUDA events around every attention launch, recorded by libmux on the side's own stream.
    ev_pf = [mux.EventSet(2 * NT) for _ in range(K)]
    ev_dc = [mux.EventSet(2 * D) for _ in range(K)]
    step_sides = [wl.sides(best["dec_sms"], D, (k * D) % NT, ev_pf[k], ev_dc[k]) for k in range(K)]
    ns = step_sides[0][2]
    warm_sides = [wl.sides(best["dec_sms"], D, (k * D) % NT) for k in range(args.warmup)]
    times = torch.zeros((K, 4), dtype=torch.int64, device="cuda")
    wtimes = torch.zeros(4, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if args.config == 1 else None
    for k in range(args.warmup):
        mux.mux_run_layer(part, i, wl.pool, warm_sides[k][0], warm_sides[k][1], wtimes)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sa = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    sb = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        a.record(st)
        for k in range(K):
            if flush is not None:
                flush.zero_()                       # evict L2 (126 MB) before the step (cfg1 only)
            sa[k].record(st)
            mux.mux_run_layer(part, i, wl.pool, step_sides[k][0], step_sides[k][1], times[k])
            sb[k].record(st)
        b.record(st)
        torch.cuda.synchronize()
    tt = times.cpu().numpy()
    step_ms = [sa[k].elapsed_time(sb[k]) for k in range(K)]
    t_step = float(np.mean(step_ms)) * 1e-3 if flush is not None else a.elapsed_time(b) / K * 1e-3
    pf_attn_ms = np.concatenate([e.durations_ms(NT) for e in ev_pf])
    dc_attn_ms = np.concatenate([e.durations_ms(D) for e in ev_dc])
    bub = bubble_stats(tt)
    hot = None
    if flush is not None:   # cfg1 also hot (no flush; per-step events like the flushed loop)
        for k in range(K):
            sa[k].record(st)
            mux.mux_run_layer(part, i, wl.pool, step_sides[k][0], step_sides[k][1], times[k])
            sb[k].record(st)
        torch.cuda.synchronize()
        hot = step_tokens(D) / (float(np.mean([sa[k].elapsed_time(sb[k]) for k in range(K)])) * 1e-3)
    if world > 1:
        tm = torch.tensor([t_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        t_step = float(tm.item())
        dist.barrier()
    value = step_tokens(D) / t_step   # aggregate over ranks (each rank holds a head shard of the same tokens)

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
    if args.ar == "fused":
        wl2.set_fused_allreduce(rank, world)                # its own peer-shared y / staging
    sets = [wl, wl2]
    e2e_sides = {}

    def e2e_side(c, step):
        key = (c, (step * D) % NT)
        if key not in e2e_sides:
            e2e_sides[key] = sets[c].sides(best["dec_sms"], D, key[1])[:2]
        return e2e_sides[key]

    outs = [[torch.empty(w.pf_y.shape, dtype=w.pf_y.dtype).pin_memory(),
             torch.empty(w.dc_y.shape, dtype=w.dc_y.dtype).pin_memory()] for w in sets]
    h2d = sum(t.numel() * t.element_size() for t in pin.values())
    d2h = sum(t.numel() * t.element_size() for t in outs[0])
    cs = torch.cuda.Stream()                                 # H2D copy stream
    cso = torch.cuda.Stream()                                # D2H copy stream: the two directions run on
    ev_in = [torch.cuda.Event(), torch.cuda.Event()]        # separate copy engines (PCIe is full duplex)
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
            pfs, dcs = e2e_side(c, step)
            mux.mux_run_layer(part, i, wl.pool, pfs, dcs, wtimes)
            ev_done[c].record(st)
            with torch.cuda.stream(cso):
                cso.wait_event(ev_done[c])
                outs[c][0].copy_(sets[c].pf_y, non_blocking=True)
                outs[c][1].copy_(sets[c].dc_y, non_blocking=True)
                ev_out[c].record(cso)
        st.wait_stream(cs)
        st.wait_stream(cso)

    for e in ev_out:
        e.record(cso)
    e2e_run(2)
    torch.cuda.synchronize()
    a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a2.record(st)
    e2e_run(K)
    b2.record(st)
    torch.cuda.synchronize()
    t_e2e = a2.elapsed_time(b2) / K * 1e-3
    if world > 1:
        tm = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        t_e2e = float(tm.item())

    # ---- rooflines of the dominant kernels, measured in the timed region (CUDA events on the
    # launching partition stream; achieved = algorithmic work per launch / mean launch duration)
    pf_share = best["pf_sms"] / total_sms
    dc_share = best["dec_sms"] / total_sms
    pf_launch_s = float(np.mean(pf_attn_ms)) * 1e-3
    dc_launch_s = float(np.mean(dc_attn_ms)) * 1e-3
    pf_tflops = wl.prefill_flops_layer() / pf_launch_s / 1e12
    dc_gbs = wl.decode_bytes_layer() / dc_launch_s / 1e9
    burst, sustained = peaks["bf16_tflops"], peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    traffic_files = []
    for tf in ("r02o_traffic.json", "r02z_traffic.json", "r02q_traffic.json", "r02_traffic.json", "r01s3_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", tf)) as f:
                traffic_files.append((tf, json.load(f)))
        except Exception:
            pass

    def traffic_of(kernel):
        """(DRAM bytes per launch, file) from the newest ncu --set full summary that has `kernel`."""
        for tf, t in traffic_files:
            if kernel in t:
                return t[kernel].get("bytes"), tf
        return None, None
    # SURVEY §8(d) decode denominators: BW_read(k_d) = read-only 32 KiB bulk-copy stream on the SAME
    # decode partition, alone and while the step's prefill side runs (contended: the primary one)
    bw_part, bw_full = probe_read_bw(mux, part, wl, i, best["dec_sms"]), probe_read_bw(mux, part, wl, -1, total_sms)
    bw_part_mux = probe_read_bw_contended(mux, part, wl, i, best["dec_sms"], step_sides[0][0])
    tc_kp = time_tc_share(mux, part, wl, i, best["pf_sms"])
    t_pf_k, clk_pf_k = time_kernel_alone(mux, part, wl, i, "pf")
    qkv = None
    if wl.d == 128 and wl.Hq % 2 == 0 and wl.Hkv % 2 == 0:
        t_qkv, f_qkv = time_qkv_fused(mux, wl)
        qkv = {"kernel": "outproj2_kernel<QKV> (tcgen05 CTA pairs, RoPE + pool-slot epilogue)",
               "shape": f"{wl.pf_spec.total_new}x{wl.hidden}x{(wl.Hq + 2 * wl.Hkv) * wl.d}", "launch_us": t_qkv * 1e6,
               "achieved": f_qkv / t_qkv / 1e12, "unit": "TFLOP/s", "peak": burst,
               "frac": f_qkv / t_qkv / 1e12 / burst, "peak_src": f"{peaks_src} bf16_tflops (burst), whole GPU",
               "note": "f4 first part, timed alone after the steps; not in the step (attention-path metric)"}
    ffn = None
    if args.config in (2, 3, 5):   # Llama-3-8B widths
        t_ffn, f_ffn = time_ffn(mux, wl)
        ffn = {"kernel": "outproj2_kernel<SwiGLU> gate/up + outproj2_kernel down (tcgen05 CTA pairs)",
               "shape": f"T {wl.pf_spec.total_new}, hidden {wl.hidden}, inter 14336", "call_us": t_ffn * 1e6,
               "achieved": f_ffn / t_ffn / 1e12, "unit": "TFLOP/s", "peak": burst,
               "frac": f_ffn / t_ffn / 1e12 / burst, "note": "f4 second part, timed alone after the steps"}
    t_dc_k, clk_dc_k = time_kernel_alone(mux, part, wl, i, "dc")
    peak_pf = burst * pf_share
    # which prefill kernel the library launches (prefill.cu launch_prefill): the persistent loop when the
    # batch's K and V fit in 64 MiB of L2, else one CTA pair per work item
    pf_persistent = sum(wl.pf_spec.L) * wl.Hkv * 4.0 * wl.d <= 64.0 * (1 << 20)
    pf_kernel = "prefill6p_kernel" if pf_persistent else "prefill6_kernel"
    roofline = {"bound": "tensor",
                "kernel": pf_kernel + (" (tcgen05 causal prefill attention, persistent over the partition's SMs, "
                                       if pf_persistent else " (tcgen05 causal prefill attention, ") + "1 launch per layer)",
                "achieved": pf_tflops, "peak": peak_pf, "unit": "TFLOP/s", "frac": pf_tflops / peak_pf,
                "traffic": traffic_of(pf_kernel)[0], "traffic_src": traffic_of(pf_kernel)[1],
                "launches": int(len(pf_attn_ms)), "launch_us_mean": pf_launch_s * 1e6,
                "launch_us_p10_p90": [float(np.percentile(pf_attn_ms, q)) * 1e3 for q in (10, 90)],
                "per_launch_flop": wl.prefill_flops_layer(),
                "peak_src": f"{peaks_src} bf16_tflops (burst) {burst} x prefill SM share {best['pf_sms']}/{total_sms}",
                "frac_of_sustained_share": pf_tflops / (sustained * pf_share),
                "tc_kp_tflops": tc_kp, "frac_of_tc_kp": pf_tflops / tc_kp,
                "tc_kp_src": f"libmux tcgen05 GEMM 8192x{wl.Hq * wl.d}x{wl.hidden} on the {best['pf_sms']}-SM prefill "
                             "green context, CUDA events, alone",
                "vendor_peak_share": 2250.0 * pf_share, "frac_of_vendor_share": pf_tflops / (2250.0 * pf_share),
                "alone_launch_us": t_pf_k * 1e6, "alone_frac": wl.prefill_flops_layer() / t_pf_k / 1e12 / peak_pf,
                "alone_clocks": clk_pf_k,
                "window": f"mean over the {len(pf_attn_ms)} prefill attention launches of the {K} timed steps "
                          "(decode side running beside it)"}
    roofline_dec = {"bound": "hbm", "kernel": "decode_kernel (+ combine_kernel when split)", "achieved": dc_gbs,
                    "peak": bw_part_mux, "unit": "GB/s", "frac": dc_gbs / bw_part_mux,
                    "peak_src": f"BW_read({best['dec_sms']}) measured on the decode partition while the prefill side runs",
                    "traffic": traffic_of("decode_kernel")[0], "traffic_src": traffic_of("decode_kernel")[1],
                    "launches": int(len(dc_attn_ms)), "launch_us_mean": dc_launch_s * 1e6,
                    "per_launch_bytes": wl.decode_bytes_layer(),
                    "partition_read_alone_gbs": bw_part, "frac_of_partition_read_alone": dc_gbs / bw_part,
                    "full_gpu_read_gbs": bw_full, "hbm_copy_gbs": peaks["hbm_gbs"],
                    "frac_of_hbm_copy_share": dc_gbs / (peaks["hbm_gbs"] * dc_share),
                    "vendor_hbm_gbs": 8000.0, "frac_of_vendor_hbm": dc_gbs / 8000.0,
                    "sm_share": dc_share,
                    "iso_achieved": wl.decode_bytes_layer() / (best["t_dc_iso_ms"] * 1e-3 / NT) / 1e9,
                    "alone_launch_us": t_dc_k * 1e6, "alone_frac_of_partition_read": wl.decode_bytes_layer() / t_dc_k
                    / 1e9 / bw_part, "alone_clocks": clk_dc_k}
    model = None
    if args.config in (2, 3, 5) and world == 1 and not args.no_model_step:
        try:
            model = model_step(mux, part, wl, NT, args.tbt_slo_ms, total_sms)
        except Exception as e:   # reported, never silently replaced
            model = {"error": str(e)}
    per_dc_layer = 3 + (1 if ns > 1 else 0)   # append, decode, (combine), out-proj
    launches_per_step = NT * 3 + D * per_dc_layer + 4
    line = {
        "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) bf16 KV pool, Q/K/V; random-init W_o; attention shapes of "
                + ("Llama-3-70B" if args.config == 4 else "Llama-3-8B") + ")",
        "config": {"workload": wl.cfg.name, "layers": NT, "Hq_per_rank": wl.Hq, "Hkv_per_rank": wl.Hkv,
                   "split": {"dec_sms": best["dec_sms"], "pf_sms": best["pf_sms"]},
                   "decode_layers_per_step": D, "decode_iters_per_step": D / NT,
                   "tbt_slo_ms": args.tbt_slo_ms, "tbt_ms": t_step * 1e3 * NT / D,
                   "decode_num_splits": ns, "parallelism": f"kv-head shard x{world}" if world > 1 else "single GPU",
                   "allreduce": ("fused out-proj GEMM + all-reduce kernel (peer memory)" if args.ar == "fused"
                                 else "NCCL all-reduce per layer" if world > 1 else "none (one rank)")
                                + (f"; {ar_note}" if ar_note else ""),
                   "l2": ("L2 flushed (256 MB write) before every timed step" if flush is not None else
                          "inputs larger than L2 (KV pool of every layer >> 126 MB; layers rotate)")},
        "roofline": roofline, "roofline_decode": roofline_dec,
        "bubble": bub, "bubble_ratio": bub["bubble_ratio"],
        "e2e": {"value": step_tokens(D) / t_e2e, "unit": "tok/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches_per_step * K,
        "step_ms_p10_p50_p90": [float(np.percentile(step_ms, q)) for q in (10, 50, 90)],
        "clocks": clk.summary(),
        "iso_full_gpu_ms": {"prefill_all_layers": full_pf * 1e3, "decode_iter_all_layers": full_dc * 1e3},
        "time_sliced_tok_s": step_tokens(D) / (full_pf + full_dc * D / NT),
        "sweep": sweep,
        "partition_mem_bytes": part.memory_bytes(),
        "qkv_fused": qkv, "ffn_swiglu": ffn, "model_step": model,
    }
    if hot is not None:
        line["value_hot"] = hot
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline_sample(args.config)
            cb["host_cpu"] = host_cpu_model()
            try:
                env = dict(os.environ, OMP_NUM_THREADS="1")
                out = subprocess.run([sys.executable, os.path.abspath(__file__), "--oracle-1thread"], env=env,
                                     capture_output=True, text=True, timeout=600).stdout.strip().splitlines()
                cb["oracle_1thread"] = json.loads(out[-1])
            except Exception as e:
                cb["oracle_1thread"] = {"error": str(e)}
            line["cpu_baseline"] = cb
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
