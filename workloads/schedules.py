"""Seeded tensor tables, group assignments and readiness (mark) schedules.

A schedule is an int32 array mark_cycle[N, T]: rank r marks tensor t ready
after it has completed mark_cycle[r, t] coordination cycles (-1 = never).
This is the input both the oracle (oracle.simulate_step) and the CUDA path
(the test driver calls gr_mark_ready/gr_step in that order) consume.

Recipes (DESIGN.md §4 "input recipe"):
* cfg1 (BASELINE.json configs[0]): N=2, T=8, numel ~ U{1..4096}, G=3 random set
  partition (all groups non-empty), per rank a random permutation of the
  tensors with 0-2 marks per cycle. Seeds: table/groups numpy
  default_rng(seed), rank r's order default_rng(seed*1000003 + r).
* reverse-layer (cfg2/cfg3): FCN tensors released in reverse-layer order,
  one layer (weight+bias) per cycle, optionally jittered per rank.
* cfg4: T tensors, G=T/8 contiguous groups of 8; rank r's order is the
  reverse order rotated by r*T/N ("adversarial skew"); T/16 marks per cycle.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Case:
    N: int
    numel: np.ndarray       # [T] int64
    group_of: np.ndarray    # [T] int32, dense 0..G-1
    mark_cycle: np.ndarray  # [N, T] int32
    seed: int

    @property
    def T(self) -> int:
        return int(self.numel.size)

    @property
    def G(self) -> int:
        return int(self.group_of.max()) + 1


def random_partition(T: int, G: int, rng: np.random.Generator) -> np.ndarray:
    """Uniformly random assignment of T tensors to G non-empty groups."""
    assert 1 <= G <= T
    perm = rng.permutation(T)
    g = np.empty(T, dtype=np.int32)
    g[perm[:G]] = np.arange(G, dtype=np.int32)
    g[perm[G:]] = rng.integers(0, G, size=T - G, dtype=np.int32)
    return g


def random_mark_schedule(N: int, T: int, seed: int, max_per_cycle: int = 2,
                         salt: int = 1000003) -> np.ndarray:
    """Per rank: a random permutation of the tensors, U{0..max_per_cycle} marks per cycle."""
    m = np.empty((N, T), dtype=np.int32)
    for r in range(N):
        rng = np.random.default_rng(seed * salt + r)
        order = rng.permutation(T)
        c = 0
        i = 0
        while i < T:
            k = int(rng.integers(0, max_per_cycle + 1))
            for _ in range(k):
                if i < T:
                    m[r, order[i]] = c
                    i += 1
            c += 1
        del c
    return m


def cfg1_case(seed: int, N: int = 2, T: int = 8, G: int = 3, max_numel: int = 4096) -> Case:
    rng = np.random.default_rng(seed)
    numel = rng.integers(1, max_numel + 1, size=T).astype(np.int64)
    group_of = random_partition(T, G, rng)
    mark = random_mark_schedule(N, T, seed)
    return Case(N, numel, group_of, mark, seed)


def reverse_layer_schedule(n_layers: int, N: int, release_order, layers_per_cycle: int = 1,
                           jitter_seed: int | None = None, max_shift: int = 0) -> np.ndarray:
    """Weight+bias of each layer marked in reverse-layer order, layers_per_cycle per cycle.

    With jitter_seed set, each rank's mark cycle for each layer is delayed by
    U{0..max_shift} cycles (keeping per-rank order monotone)."""
    T = 2 * n_layers
    m = np.empty((N, T), dtype=np.int32)
    for r in range(N):
        rng = np.random.default_rng(jitter_seed * 1000003 + r) if jitter_seed is not None else None
        last = 0
        for k, l in enumerate(release_order):
            c = k // layers_per_cycle
            if rng is not None and max_shift > 0:
                c = max(last, c + int(rng.integers(0, max_shift + 1)))
            last = c
            m[r, 2 * l] = c
            m[r, 2 * l + 1] = c
    return m


def cfg4_case(T: int, N: int, marks_per_cycle: int | None = None) -> Case:
    """Bitvector latency workload: contiguous groups of 8, rotated reverse orders."""
    assert T % 8 == 0
    G = T // 8
    group_of = (np.arange(T) // 8).astype(np.int32)
    per = marks_per_cycle or max(1, T // 16)
    rev = np.arange(T - 1, -1, -1)
    m = np.empty((N, T), dtype=np.int32)
    for r in range(N):
        order = np.roll(rev, -(r * T // N))
        m[r, order] = (np.arange(T) // per).astype(np.int32)
    numel = np.full(T, 256, dtype=np.int64)
    return Case(N, numel, group_of, m, 0)
