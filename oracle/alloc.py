"""ORACLE — TEST INFRASTRUCTURE ONLY.  Page allocator + page-table oracle.

The paper fixes only that K/V live in one paged pool shared by both phases and by all
requests ("a single KV cache pool", P:1111 PagedAttention).  It is
silent on the allocation policy, so DESIGN.md reading R18 fixes a deterministic one,
which this file states in plain Python and the C++ library implements independently:

  * the free list starts as a permutation of [0, num_pages) drawn by Fisher-Yates with
    a splitmix64 counter generator seeded by `seed` (i from n-1 down to 1:
    j = next() mod (i+1); swap(a[i], a[j]));
  * alloc(n): fewer than n free -> POOL_EXHAUSTED with no effect; else pop n ids from the
    front in order, refcount = 1;
  * share(ids): refcount += 1 for each (prefix pages reused across requests);
  * free(ids): refcount -= 1; a page reaching 0 is appended to the tail (FIFO).

Pins (tests/test_oracle_pins.py): closed-form splitmix64 test vector, permutation
property, all-or-nothing, FIFO reuse order, brute-force refcount bookkeeping.
"""
from __future__ import annotations

from collections import deque
from typing import List

MASK64 = (1 << 64) - 1


class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)


def seeded_permutation(n: int, seed: int) -> List[int]:
    a = list(range(n))
    g = SplitMix64(seed)
    for i in range(n - 1, 0, -1):
        j = g.next() % (i + 1)
        a[i], a[j] = a[j], a[i]
    return a


class PoolExhausted(Exception):
    pass


class SharedPageWrite(Exception):
    pass


class OraclePagePool:
    def __init__(self, num_pages: int, seed: int):
        self.num_pages = num_pages
        self.free = deque(seeded_permutation(num_pages, seed))
        self.ref = [0] * num_pages

    def alloc(self, n: int) -> List[int]:
        if n < 0:
            raise ValueError(n)
        if n > len(self.free):
            raise PoolExhausted(n)
        out = [self.free.popleft() for _ in range(n)]
        for p in out:
            self.ref[p] = 1
        return out

    def share(self, ids: List[int]) -> None:
        for p in ids:
            if not (0 <= p < self.num_pages) or self.ref[p] < 1:
                raise ValueError(p)
        for p in ids:
            self.ref[p] += 1

    def release(self, ids: List[int]) -> None:
        for p in ids:
            if not (0 <= p < self.num_pages) or self.ref[p] < 1:
                raise ValueError(p)
        for p in ids:
            self.ref[p] -= 1
            if self.ref[p] == 0:
                self.free.append(p)

    def num_free(self) -> int:
        return len(self.free)


def build_page_tables(pool: OraclePagePool, pages_needed: List[int]):
    """Allocate each sequence's pages in order; CSR (indptr, ids) as Python lists."""
    indptr, ids = [0], []
    for n in pages_needed:
        ids.extend(pool.alloc(n))
        indptr.append(len(ids))
    return indptr, ids


def slot_of(page_ids_of_seq: List[int], t: int, page_size: int = 16) -> int:
    """O2 slot mapping: slot(b,t) = pt_b[t div 16] * 16 + t mod 16."""
    return page_ids_of_seq[t // page_size] * page_size + t % page_size
