"""Pins for the oracle's schedule half (§4.1 steps 1-3, §4.2 grouping).

Each test checks the oracle against something other than itself:
* brute-force set intersection over every tuple of per-rank subsets (V1),
* the closed form rel_cycle(g) = max_{t in g} max_r m_r(t) (V2),
* exactly-once / rank-identical / special cases (V3-V5),
* hand-written SPEC.md worked vectors in tests/golden/spec_vectors.json (V6).
"""
import itertools
import json
import os

import numpy as np
import pytest

from workloads.schedules import random_partition

HERE = os.path.dirname(os.path.abspath(__file__))


def set_partitions(n):
    """All set partitions of range(n) as restricted-growth strings (Bell(n) of them)."""
    def rec(prefix, m):
        if len(prefix) == n:
            yield list(prefix)
            return
        for v in range(m + 2):
            yield from rec(prefix + [v], max(m, v))
    yield from rec([0], 0) if n > 0 else iter([[]])


def test_set_partitions_bell():
    assert [sum(1 for _ in set_partitions(n)) for n in range(1, 7)] == [1, 2, 5, 15, 52, 203]


def bits_of_words(A):
    return {w * 32 + b for w, x in enumerate(A) for b in range(32) if (int(x) >> b) & 1}


def test_words(orc):
    # W = ceil((T+2)/32): 30 tensors fit one word, 31 need two (reading R2)
    assert [orc.words(t) for t in (1, 30, 31, 62, 63, 65536)] == [1, 1, 2, 2, 3, 2049]


def test_bit_positions_group_major(orc):
    # reading R3: group-major, tensor order inside a group, after 2 status bits
    assert list(orc.bit_positions([1, 0, 2, 1, 0])) == [4, 2, 6, 5, 3]
    assert list(orc.bit_positions([0, 1, 2, 3])) == [2, 3, 4, 5]
    with pytest.raises(ValueError):
        orc.bit_positions([0, 2])  # group 1 empty


@pytest.mark.parametrize("N,T", [(1, 6), (2, 6), (3, 6)])
def test_intersection_bruteforce_exhaustive(orc, N, T):
    """V1: for every tuple of per-rank pending subsets, A's payload = set intersection."""
    rng = np.random.default_rng(N * 100 + T)
    group_of = random_partition(T, int(rng.integers(1, T + 1)), rng)
    bit_of = orc.bit_positions(group_of)
    subsets = list(range(1 << T))
    Ls = {}
    for s in subsets:
        pend = np.array([(s >> t) & 1 for t in range(T)], dtype=np.uint8)
        L = orc.populate(bit_of, pend)
        # populate itself: exactly the cache bits of the pending set + status bits
        assert bits_of_words(L) == {0, 1} | {int(bit_of[t]) for t in range(T) if pend[t]}
        Ls[s] = L
    for tup in itertools.product(subsets, repeat=N):
        A = orc.intersect([Ls[s] for s in tup])
        common = set(range(T))
        for s in tup:
            common &= {t for t in range(T) if (s >> t) & 1}
        assert bits_of_words(A) == {0, 1} | {int(bit_of[t]) for t in common}


def test_status_bits_or_semantics(orc):
    """Reading R1: complement coding makes one AND compute the OR of the status flags."""
    bit_of = orc.bit_positions([0, 0, 1])
    pend = np.ones(3, dtype=np.uint8)
    for flags in itertools.product([0, 1], repeat=6):
        Ls = [orc.populate(bit_of, pend, abort=flags[2 * r], shutdown=flags[2 * r + 1]) for r in range(3)]
        A = orc.intersect(Ls)
        any_abort = any(flags[0::2])
        any_shut = any(flags[1::2])
        assert bool(A[0] & 1) == (not any_abort)
        assert bool(A[0] & 2) == (not any_shut)
        assert A[0] >> 2 == 0b111


def closed_form(group_of, m):
    """V2: with monotone readiness, group g is released in cycle max_{t in g} max_r m_r(t)."""
    G = int(np.max(group_of)) + 1
    return [int(max(m[:, t].max() for t in range(len(group_of)) if group_of[t] == g)) for g in range(G)]


def test_release_closed_form_exhaustive_n1(orc):
    """Every set partition of 6 tensors x every mark schedule in {0,1,2}^6 (N=1)."""
    T = 6
    cases = 0
    for part in set_partitions(T):
        g = np.array(part, dtype=np.int32)
        for ms in itertools.product(range(3), repeat=T):
            m = np.array([ms], dtype=np.int32)
            r = orc.simulate_step(1, g, m, max_cycles=8)
            assert r.rc == 0
            assert list(r.rel_cycle) == closed_form(g, m)
            cases += 1
    assert cases == 203 * 729


@pytest.mark.parametrize("N", [2, 3, 4, 8])
def test_release_closed_form_random(orc, N):
    rng = np.random.default_rng(1234 + N)
    for _ in range(1500):
        T = int(rng.integers(1, 41))
        G = int(rng.integers(1, T + 1))
        g = random_partition(T, G, rng)
        m = rng.integers(0, 6, size=(N, T)).astype(np.int32)
        r = orc.simulate_step(N, g, m, max_cycles=12)
        assert r.rc == 0
        assert list(r.rel_cycle) == closed_form(g, m)
        # V3 exactly once, in ascending order, each group once
        flat = [x for c in r.released for x in c]
        assert sorted(flat) == list(range(G))
        for rel in r.released:
            assert rel == sorted(rel)
        # released => marked on all ranks by that cycle
        for c, rel in enumerate(r.released):
            for gg in rel:
                assert all(m[rr, t] <= c for rr in range(N) for t in range(T) if g[t] == gg)


def test_permutation_schedules_n2_closed_form(orc):
    """Permutation readiness (one mark per cycle per rank), N=2, T=5, all 52 partitions."""
    T = 5
    perms = list(itertools.permutations(range(T)))
    rng = np.random.default_rng(5)
    for part in set_partitions(T):
        g = np.array(part, dtype=np.int32)
        for _ in range(40):
            p0 = perms[int(rng.integers(len(perms)))]
            p1 = perms[int(rng.integers(len(perms)))]
            m = np.zeros((2, T), dtype=np.int32)
            m[0, list(p0)] = np.arange(T)
            m[1, list(p1)] = np.arange(T)
            r = orc.simulate_step(2, g, m, max_cycles=T + 2)
            assert list(r.rel_cycle) == closed_form(g, m)


@pytest.mark.parametrize("N,T", [(2, 6), (3, 4)])
def test_permutation_schedules_exhaustive(orc, N, T):
    """V2 exhaustively over permutation readiness (one mark per cycle per rank) for every set
    partition: rank 0 marks in identity order (any schedule is one of these after relabeling the
    tensors, and the closed form and the partition set are invariant under relabeling), every
    other rank in every order — N=2, T=6: 203 x 720 schedules; N=3, T=4: 15 x 24^2."""
    perms = list(itertools.permutations(range(T)))
    cases = 0
    for part in set_partitions(T):
        g = np.array(part, dtype=np.int32)
        for rest in itertools.product(perms, repeat=N - 1):
            m = np.zeros((N, T), dtype=np.int32)
            m[0] = np.arange(T)
            for r, pr in enumerate(rest, start=1):
                m[r, list(pr)] = np.arange(T)
            res = orc.simulate_step(N, g, m, max_cycles=T + 2)
            assert res.rc == 0 and list(res.rel_cycle) == closed_form(g, m), (part, rest)
            cases += 1
    assert cases == len(list(set_partitions(T))) * len(perms) ** (N - 1)


def test_special_cases(orc):
    rng = np.random.default_rng(9)
    T = 12
    m = rng.integers(0, 5, size=(3, T)).astype(np.int32)
    # V5a: G=1 releases once, when the last tensor is globally ready
    r = orc.simulate_step(3, np.zeros(T, np.int32), m, max_cycles=10)
    assert r.rel_cycle[0] == m.max() and sum(len(x) for x in r.released) == 1
    # V5b: singleton groups = ungrouped per-cycle behaviour: tensor t goes at max_r m_r(t)
    r = orc.simulate_step(3, np.arange(T, dtype=np.int32), m, max_cycles=10)
    assert list(r.rel_cycle) == [int(m[:, t].max()) for t in range(T)]
    # V5c: N=1, A == L_0 of the pending set each cycle
    g = random_partition(T, 4, rng)
    m1 = m[:1]
    r = orc.simulate_step(1, g, m1, max_cycles=10)
    bit_of = orc.bit_positions(g)
    released = set()
    for c in range(r.n_cycles):
        pend = np.array([(m1[0, t] <= c) and (g[t] not in released) for t in range(T)], np.uint8)
        assert np.array_equal(r.A[c], orc.populate(bit_of, pend))
        released |= set(r.released[c])


def test_never_marked_hits_cycle_bound(orc):
    # reading R14: a tensor some rank never marks keeps its group pending
    r = orc.simulate_step(2, [0, 1], [[0, 0], [0, -1]], max_cycles=5)
    assert r.rc == 2 and r.n_cycles == 5 and list(r.rel_cycle) == [0, -1]


def test_abort_ends_step(orc):
    status = np.zeros((2, 6), np.uint8)
    status[1, 2] = 1  # rank 1 raises ABORT in cycle 2
    r = orc.simulate_step(2, [0, 1, 2], [[0, 1, 4], [0, 1, 4]], status=status, max_cycles=6)
    assert r.rc == 1 and r.n_cycles == 3 and r.released[2] == []
    assert not (r.A[2][0] & 1) and (r.A[2][0] & 2)


def test_golden_spec_vectors(orc):
    with open(os.path.join(HERE, "golden", "spec_vectors.json")) as f:
        gold = json.load(f)
    for case in gold["schedule_cases"]:
        r = orc.simulate_step(case["N"], case["group_of"], case["mark_cycle"],
                              max_cycles=case["max_cycles"])
        assert r.rc == case["expect_rc"], case["id"]
        assert [list(map(int, a)) for a in r.A] == case["expect_A"], case["id"]
        assert r.released == case["expect_released"], case["id"]
