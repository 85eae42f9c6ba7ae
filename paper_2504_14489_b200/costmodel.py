"""Solo-run latency predictors of MuxWise (§3.3.2, Eq.1 / Eq.2) fitted to
THIS library's kernels on B200, per SM partition, plus the contention guard's maximum decode
slowdown per partition.

  Eq.1  T_prefill = th1 * sum_i n_i^2 + th2 * sum_i n_i r_i + th3 * sum_i n_i + th4
  Eq.2  T_decode  = th1 * sum_i r_i   + th2 * bs            + th3

Times are per transformer layer of the attention sublayer this library runs (append + attention
(+ combine) + out-projection), in microseconds, measured with the other side idle.  For decode,
r_i is the reused context of request i (its context minus the current token, SURVEY §8 symbols).
Coefficients are fitted by non-negative least squares (all terms are costs), one set per
(side, SM count).  The paper reports max deviations of 8.16% (prefill) and 8.84% (decode)
for its own kernels; `fit` returns ours.

Host-side scheduling logic (no GPU work).  The C engine (csrc/engine.cu) evaluates the
paper-form Eq.1 / Eq.2 coefficients passed in mux_engine_desc (dec_theta / pf_theta) for its
best-fit split and N_PL; this module fits them, and also the wave-aware B200 variants below,
which is where the accuracy claim of P:607 is checked (tests/test_costmodel.py).
"""
from __future__ import annotations

import dataclasses
import json
import math
from typing import Dict, List, Sequence, Tuple

import numpy as np


def prefill_features(r: Sequence[int], n: Sequence[int]) -> np.ndarray:
    r = np.asarray(r, dtype=np.float64)
    n = np.asarray(n, dtype=np.float64)
    return np.array([np.sum(n * n), np.sum(n * r), np.sum(n), 1.0])


def decode_features(r: Sequence[int]) -> np.ndarray:
    r = np.asarray(r, dtype=np.float64)
    return np.array([np.sum(r), float(len(r)), 1.0])


# ---------------------------------------------------------------------------------------------
# Wave-aware B200 variants (Eq.1w / Eq.2w).  Eq.1 / Eq.2's constant + linear terms cannot express
# wave quantisation: a grid of CTAs runs in waves over the partition's SMs, so a layer's time is
# the MAKESPAN of its CTAs on k SMs, not the sum of their work / k (r01: Eq.1 missed by up to 35 %
# on 132-148 SMs).  The features below keep the paper's physics (per-CTA work ~ the keys a q tile
# attends, Table 2; decode work ~ reused context) but schedule it the way these kernels
# launch: one CTA per SM, CTAs dispatched in launch order onto the first free SM.

def _list_makespan(durations, k: int) -> float:
    import heapq
    h = [0.0] * max(1, min(k, len(durations)))
    heapq.heapify(h)
    span = 0.0
    for t in durations:
        s = heapq.heappop(h)
        heapq.heappush(h, s + t)
        span = max(span, s + t)
    return span


def prefill_wave_features(r: Sequence[int], n: Sequence[int], sms: int, hq: int = 32, hkv: int = 8, d: int = 128,
                          cta_overhead_tiles: float = 3.0) -> np.ndarray:
    """[attention makespan (128-key tile units), out-projection waves, sum n, 1, K/V MB streamed
    from HBM] of one layer on `sms` SMs: the prefill grid (q tile x head pair x sequence,
    csrc/prefill.cu tile_coord order: q tiles longest-first grid-wide when the batch K/V is <= 64 MB,
    else per sequence heavy-first) and the CTA-pair out-projection GEMM (256 x 256 tiles of T x
    hidden over sms/2 pairs).  A CTA costs its key tiles + ~3 tiles of prologue / epilogue (TMEM
    alloc, Q load, O write), the constant that fits the recorded B200 samples best
    (profiles/r02_costmodel.json).  The last term is the batch's K/V in MB when it exceeds the L2
    budget (> 64 MB, the per-sequence order): the K/V then comes from HBM rather than L2, which the
    tile makespan alone does not see (two 1k chunks on 8k prefixes ran 11 % above the 4-term fit on
    148 SMs, profiles/r02q_costmodel.json; with the term <= 9.5 % on every partition)."""
    keys = sum(a + b for a, b in zip(r, n))
    nq = max((x + 127) // 128 for x in n)
    heads = max(1, hq // 2)
    ctas = []
    def cta(b, qi):
        return cta_overhead_tiles + math.ceil((r[b] + min((qi + 1) * 128, n[b])) / 128)
    if keys * hkv * 4 * d <= 64 * 2 ** 20:
        for qi in range(nq - 1, -1, -1):
            for b in range(len(n)):
                if qi * 128 < n[b]:
                    ctas += [cta(b, qi)] * heads
    else:
        for b in sorted(range(len(n)), key=lambda i: -n[i] * (r[i] + 0.5 * n[i])):
            for _ in range(heads):
                ctas += [cta(b, qi) for qi in range((n[b] + 127) // 128 - 1, -1, -1)]
    T = sum(n)
    waves = math.ceil(math.ceil(T / 256) * 16 / max(1, sms // 2))
    kv_bytes = keys * hkv * 4 * d
    kv_hbm_mb = kv_bytes / 1e6 if kv_bytes > 64 * 2 ** 20 else 0.0
    return np.array([_list_makespan(ctas, sms), float(waves), float(T), 1.0, kv_hbm_mb])


def decode_wave_features(r: Sequence[int], sms: int, hkv: int = 8, d: int = 128, num_splits: int = 0,
                         cta_overhead_pages: float = 10.0) -> np.ndarray:
    """[CTA makespan (page units), sum r, bs, bs x splits (combine, split > 1), split > 1, 1] of one
    decode layer on `sms` SMs: balanced split-KV CTAs (every split of a sequence covers
    ceil(max_pages / S) pages, csrc/decode.cu) in launch order; S from the library's own
    split heuristic (mux_decode_num_splits) unless given."""
    L = [int(x) + 1 for x in r]
    B = len(L)
    if num_splits <= 0:
        from . import binding
        num_splits = binding.mux_decode_num_splits(B, hkv, max(L), sms, L, d)
    S = num_splits
    maxp = max((x + 15) // 16 for x in L)
    C = math.ceil(maxp / S)
    durs = []
    for x in L:
        p = (x + 15) // 16
        for sp in range(S):
            npg = max(0, min(C, p - sp * C)) if sp < S - 1 else max(0, p - sp * C)
            durs.append(cta_overhead_pages + npg if (npg > 0 or sp == 0) else 2.0)
    split = 1.0 if S > 1 else 0.0
    return np.array([_list_makespan(durs, sms), float(sum(r)), float(B), B * S * split, split, 1.0])


@dataclasses.dataclass
class Fit:
    theta: np.ndarray            # Eq.1: 4 coefficients, Eq.2: 3 (us per unit)
    max_dev: float               # max |pred - meas| / meas over the samples
    mean_dev: float
    n: int

    def predict(self, x: np.ndarray) -> float:
        return float(np.dot(self.theta, x))


def fit(features: np.ndarray, times_us: np.ndarray) -> Fit:
    """Non-negative least squares on RELATIVE error (rows scaled by 1/t): the paper's accuracy
    figure is a relative deviation, and the samples span three orders of magnitude."""
    from scipy.optimize import nnls
    A = np.asarray(features, dtype=np.float64)
    t = np.asarray(times_us, dtype=np.float64)
    w = 1.0 / t
    # column scaling for conditioning (sum n^2 ~ 1e8 vs the constant 1)
    cs = np.maximum(np.abs(A * w[:, None]).max(axis=0), 1e-30)
    th, _ = nnls((A * w[:, None]) / cs, np.ones_like(t))
    th = th / cs
    pred = A @ th
    dev = np.abs(pred - t) / t
    return Fit(th, float(dev.max()), float(dev.mean()), len(t))


@dataclasses.dataclass
class CostModel:
    """Per-partition fits: prefill[sm_count], decode[sm_count], and the contention guard's
    max decode / prefill slowdown per split (decode SM count)."""
    prefill: Dict[int, Fit]
    decode: Dict[int, Fit]
    max_slowdown_dec: Dict[int, float] = dataclasses.field(default_factory=dict)
    max_slowdown_pf: Dict[int, float] = dataclasses.field(default_factory=dict)

    def t_prefill(self, sms: int, r, n) -> float:
        return self.prefill[sms].predict(prefill_features(r, n))

    def t_decode(self, sms: int, r) -> float:
        return self.decode[sms].predict(decode_features(r))

    def worst_case_decode(self, dec_sms: int, r) -> float:
        """Solo prediction x the guard's maximum slowdown for that split."""
        return self.t_decode(dec_sms, r) * self.max_slowdown_dec.get(dec_sms, 1.0)

    def best_fit_split(self, splits: List[Tuple[int, int]], r_dec, n_layers: int, tbt_slo_us: float):
        """Smallest decode SM count whose worst-case decode iteration (n_layers layers) meets
        the TBT SLO ("best-fit number of SMs"); None if none does."""
        for dsms, psms in sorted(splits):
            if dsms in self.decode and self.worst_case_decode(dsms, r_dec) * n_layers <= tbt_slo_us:
                return dsms, psms
        return None

    def to_json(self) -> dict:
        def fj(d):
            return {str(k): {"theta": v.theta.tolist(), "max_dev": v.max_dev, "mean_dev": v.mean_dev, "n": v.n}
                    for k, v in sorted(d.items())}
        return {"units": "us per layer", "prefill_eq1": fj(self.prefill), "decode_eq2": fj(self.decode),
                "max_slowdown_dec": {str(k): v for k, v in sorted(self.max_slowdown_dec.items())},
                "max_slowdown_pf": {str(k): v for k, v in sorted(self.max_slowdown_pf.items())}}

    @staticmethod
    def from_json(d: dict) -> "CostModel":
        def jf(x):
            return {int(k): Fit(np.array(v["theta"]), v["max_dev"], v["mean_dev"], v["n"]) for k, v in x.items()}
        return CostModel(jf(d["prefill_eq1"]), jf(d["decode_eq2"]),
                         {int(k): float(v) for k, v in d.get("max_slowdown_dec", {}).items()},
                         {int(k): float(v) for k, v in d.get("max_slowdown_pf", {}).items()})

    @staticmethod
    def load(path: str) -> "CostModel":
        with open(path) as f:
            d = json.load(f)
        return CostModel.from_json(d["model"] if "model" in d else d)  # profile_costmodel.py output or bare
