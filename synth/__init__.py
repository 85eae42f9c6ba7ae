"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no slot mapping, no attention, no
softmax, no page allocation): it only draws random numbers and lengths and rounds
fp32 samples to bf16 bit patterns, so that the CUDA path (paper_2504_14489_b200)
and the CPU oracle (oracle/) consume byte-identical inputs.

Recipe:
  * base seed 2504_14489, per-tensor stream seed = BASE + 1000*cfg + tensor_id,
    numpy PCG64;
  * Q, K, V ~ N(0, 1) fp32 -> bf16 round-to-nearest-even (BASELINE.json "same
    generated bf16 inputs");  optional "outlier" variant scales 1% of K rows by 8;
  * W_o ~ N(0, 1/(Hq*d)) -> bf16;
  * lengths: the BASELINE.json configs 1-5 (Table 1, shapes the
    chat / multi-turn / long-context mixes; P:571-574 gives the symbols r, n, L).
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np

BASE_SEED = 2504_14489
PAGE_SIZE = 16

# tensor ids of the per-tensor seed streams
T_Q_PF, T_K_PF, T_V_PF, T_Q_DC, T_K_DC, T_V_DC, T_WO, T_LENS, T_FREELIST = range(9)


def rng(cfg: int, tensor_id: int, salt: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(BASE_SEED + 1000 * cfg + tensor_id + 100_000 * salt))


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit pattern, round-to-nearest-even (NaN kept quiet)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    out = ((u + rounding) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        out[nan] = 0x7FC0
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


BF16_NAN = np.uint16(0x7FC0)


def bf16_normal(g: np.random.Generator, shape, std: float = 1.0) -> np.ndarray:
    return f32_to_bf16_bits(g.standard_normal(size=shape, dtype=np.float32) * np.float32(std))


@dataclasses.dataclass
class Shapes:
    Hq: int
    Hkv: int
    d: int
    n_layers_model: int      # N_T used to normalise token*layer/s to model tok/s
    hidden: int = 0          # out-proj width (0 = not used)

    @property
    def g(self) -> int:
        return self.Hq // self.Hkv


@dataclasses.dataclass
class SideSpec:
    """One side of a mux step.  For prefill, seq b has r_b cached + n_b new tokens.
    For decode, seq b has context c_b (including the current token): r_b = c_b - 1, n_b = 1."""
    r: List[int]
    n: List[int]

    @property
    def L(self) -> List[int]:
        return [a + b for a, b in zip(self.r, self.n)]

    @property
    def num_seqs(self) -> int:
        return len(self.n)

    @property
    def total_new(self) -> int:
        return int(sum(self.n))

    def pages_needed(self) -> List[int]:
        return [(l + PAGE_SIZE - 1) // PAGE_SIZE for l in self.L]


@dataclasses.dataclass
class Config:
    cfg: int
    name: str
    shapes: Shapes
    prefill: SideSpec
    decode: SideSpec


def _cfg3_lengths(salt: int = 0, reuse_ratio: float = 0.9):
    g = rng(3, T_LENS, salt)
    n = [int(x) for x in g.integers(512, 2048 + 1, size=4)]
    # "90% prefix-cache hit": r = 9n (reading R14); 0.6 variant: r = 1.5n
    r = [int(round(x * reuse_ratio / (1.0 - reuse_ratio))) for x in n]
    c = [int(x) for x in g.integers(2048, 8192 + 1, size=128)]
    return r, n, c


def get_config(cfg: int, reuse_ratio: float = 0.9) -> Config:
    """BASELINE.json configs 1..5 as concrete shapes."""
    if cfg == 1:
        return Config(1, "cfg1: 1 layer, 4q/1kv, d64, r=64 n=128 prefill + 4 decodes @256",
                      Shapes(4, 1, 64, 1, hidden=256), SideSpec([64], [128]), SideSpec([255] * 4, [1] * 4))
    if cfg == 2:
        return Config(2, "cfg2: Llama-3-8B attention (32q/8kv d128): 8k prefill + decode 64@4k",
                      Shapes(32, 8, 128, 32, hidden=4096), SideSpec([0], [8192]), SideSpec([4095] * 64, [1] * 64))
    if cfg == 3:
        r, n, c = _cfg3_lengths(reuse_ratio=reuse_ratio)
        return Config(3, "cfg3: multi-turn chat mix, 90% prefix hit, 4 prefills n~U[512,2048] + decode 128@U[2k,8k]",
                      Shapes(32, 8, 128, 32, hidden=4096), SideSpec(r, n), SideSpec([x - 1 for x in c], [1] * len(c)))
    if cfg == 4:
        return Config(4, "cfg4: Llama-3-70B attention (64q/8kv d128, hidden 8192): 8k prefill + decode 64@4k",
                      Shapes(64, 8, 128, 80, hidden=8192), SideSpec([0], [8192]), SideSpec([4095] * 64, [1] * 64))
    if cfg == 5:
        return Config(5, "cfg5: long context: 32k prefill + decode 256@2k",
                      Shapes(32, 8, 128, 32, hidden=4096), SideSpec([0], [32768]), SideSpec([2047] * 256, [1] * 256))
    raise ValueError(cfg)


@dataclasses.dataclass
class SideData:
    """Raw (un-paged) rows for one side.  k_rows/v_rows[b] hold ALL L_b positions of
    sequence b ([L_b, Hkv, d] bf16 bits): positions < r_b are the cached prefix, the
    rest are the new tokens' K/V.  q[Σn, Hq, d] holds the new tokens' queries."""
    spec: SideSpec
    q: np.ndarray
    k_rows: List[np.ndarray]
    v_rows: List[np.ndarray]

    def k_new(self) -> np.ndarray:
        return np.concatenate([k[r:] for k, r in zip(self.k_rows, self.spec.r)], axis=0)

    def v_new(self) -> np.ndarray:
        return np.concatenate([v[r:] for v, r in zip(self.v_rows, self.spec.r)], axis=0)

    def k_cached(self) -> np.ndarray:
        return np.concatenate([k[:r] for k, r in zip(self.k_rows, self.spec.r)], axis=0)

    def v_cached(self) -> np.ndarray:
        return np.concatenate([v[:r] for v, r in zip(self.v_rows, self.spec.r)], axis=0)


def make_side(cfg: int, shapes: Shapes, spec: SideSpec, decode: bool, outliers: bool = False,
              salt: int = 0) -> SideData:
    tq, tk, tv = (T_Q_DC, T_K_DC, T_V_DC) if decode else (T_Q_PF, T_K_PF, T_V_PF)
    gq, gk, gv = rng(cfg, tq, salt), rng(cfg, tk, salt), rng(cfg, tv, salt)
    q = bf16_normal(gq, (spec.total_new, shapes.Hq, shapes.d))
    ks, vs = [], []
    for L in spec.L:
        kf = gk.standard_normal(size=(L, shapes.Hkv, shapes.d), dtype=np.float32)
        if outliers:
            sel = gk.random(L) < 0.01
            kf[sel] *= np.float32(8.0)
        ks.append(f32_to_bf16_bits(kf))
        vs.append(bf16_normal(gv, (L, shapes.Hkv, shapes.d)))
    return SideData(spec, q, ks, vs)


def make_wo(cfg: int, shapes: Shapes) -> np.ndarray:
    """W_o [Hq*d, hidden] ~ N(0, 1/(Hq*d)) in bf16 bits."""
    g = rng(cfg, T_WO)
    return bf16_normal(g, (shapes.Hq * shapes.d, shapes.hidden), std=1.0 / np.sqrt(shapes.Hq * shapes.d))


def free_list_seed(cfg: int, salt: int = 0) -> int:
    return int(rng(cfg, T_FREELIST, salt).integers(0, 2**63 - 1))


def indptr(counts) -> np.ndarray:
    out = np.zeros(len(counts) + 1, dtype=np.int32)
    out[1:] = np.cumsum(np.asarray(counts, dtype=np.int64))
    return out


def small_random_spec(g: np.random.Generator, num_seqs: int, max_r: int, max_n: int,
                      min_n: int = 1) -> SideSpec:
    r = [int(x) for x in g.integers(0, max_r + 1, size=num_seqs)]
    n = [int(x) for x in g.integers(min_n, max_n + 1, size=num_seqs)]
    return SideSpec(r, n)


def sample_rows(total: int, k: int, tile: int = 128, extra: Optional[List[int]] = None) -> np.ndarray:
    """Rows used for sampled parity / sampled oracle timing: first, last, tile boundaries,
    then uniform spread; sorted, unique (SURVEY.md §8(d) 'Sampled oracle')."""
    rows = {0, total - 1}
    for t in range(0, total, tile):
        rows.update({t, min(total - 1, t + tile - 1)})
        if len(rows) >= k // 2:
            break
    if extra:
        rows.update(int(x) for x in extra)
    spread = np.linspace(0, total - 1, num=max(2, k - len(rows))).astype(np.int64)
    rows.update(int(x) for x in spread)
    return np.array(sorted(r for r in rows if 0 <= r < total), dtype=np.int32)


def sample_rows_tiles(total: int, k: int, tile: int = 128) -> np.ndarray:
    """Parity sample of about k rows spread over ALL q tiles (the late, heavy tiles of
    a causal prefill must be sampled as densely as the early ones): first and last row; the first
    and last row of the last 4 tiles and of evenly spaced tiles across the whole range; the rest
    uniform.  Sorted, unique."""
    nt = (total + tile - 1) // tile
    rows = {0, total - 1}
    picks = set(range(max(0, nt - 4), nt)) | {int(x) for x in np.linspace(0, nt - 1, num=min(nt, max(1, k // 8)))}
    for t in sorted(picks):
        rows.update({t * tile, min(total - 1, t * tile + tile - 1)})
    extra = max(2, k - len(rows))
    while True:
        spread = np.linspace(0, total - 1, num=min(total, extra)).astype(np.int64)
        got = rows | {int(x) for x in spread}
        if len(got) >= min(k, total) or extra >= total:
            break
        extra += min(k, total) - len(got)
    return np.array(sorted(r for r in got if 0 <= r < total), dtype=np.int32)
