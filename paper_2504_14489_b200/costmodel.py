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

Host-side scheduling logic (no GPU work): evaluated by the C engine through
`mux_cost_predict` with the same coefficients; this module fits and checks them.
"""
from __future__ import annotations

import dataclasses
import json
from typing import Dict, List, Sequence, Tuple

import numpy as np


def prefill_features(r: Sequence[int], n: Sequence[int]) -> np.ndarray:
    r = np.asarray(r, dtype=np.float64)
    n = np.asarray(n, dtype=np.float64)
    return np.array([np.sum(n * n), np.sum(n * r), np.sum(n), 1.0])


def decode_features(r: Sequence[int]) -> np.ndarray:
    r = np.asarray(r, dtype=np.float64)
    return np.array([np.sum(r), float(len(r)), 1.0])


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
