"""Host logic of the multi-GPU path: KV-head sharding.

Rank k of G holds kv heads [k*Hkv/G, (k+1)*Hkv/G) and, by the contiguous GQA map (DESIGN.md
R2), q heads [k*Hq/G, (k+1)*Hq/G); attention needs no communication; the out-projection rows
of W_o that multiply those q heads' outputs give a partial sum of the layer output that one
all-reduce per layer and side completes (P:701-702 tensor parallelism).  Page tables are
replicated and checked identical across ranks through an integer hash.
"""
from __future__ import annotations

from typing import Sequence, Tuple

import numpy as np


def kv_head_range(rank: int, world: int, hkv: int) -> Tuple[int, int]:
    if world < 1 or hkv % world:
        raise ValueError(f"KV-head sharding needs world ({world}) | Hkv ({hkv})")
    per = hkv // world
    return rank * per, (rank + 1) * per


def q_head_range(rank: int, world: int, hq: int, hkv: int) -> Tuple[int, int]:
    a, b = kv_head_range(rank, world, hkv)
    g = hq // hkv
    return a * g, b * g


def wo_row_range(rank: int, world: int, hq: int, hkv: int, d: int) -> Tuple[int, int]:
    """Rows of W_o [Hq*d][hidden] that multiply this rank's q heads."""
    a, b = q_head_range(rank, world, hq, hkv)
    return a * d, b * d


def page_table_hash(page_indptr: Sequence[int], page_ids: Sequence[int]) -> int:
    """Order-sensitive 63-bit FNV-style hash of the CSR page tables (integer, exact)."""
    h = 1469598103934665603
    for x in list(page_indptr) + [-1] + list(page_ids):
        h ^= (int(x) & 0xFFFFFFFF)
        h = (h * 1099511628211) & 0x7FFFFFFFFFFFFFFF
    return h


def shard_rows(a: np.ndarray, rank: int, world: int, axis: int, total: int) -> np.ndarray:
    per = total // world
    sl = [slice(None)] * a.ndim
    sl[axis] = slice(rank * per, (rank + 1) * per)
    return a[tuple(sl)]
