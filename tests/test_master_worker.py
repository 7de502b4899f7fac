"""NEXT-4: the master-worker coordination baseline of PAPER.md:108-110 / Fig. 3a.

CPU only. The oracle (oracle/master_worker.py) is pinned by (a) SPEC.md's worked examples,
(b) an independent closed form of its response order, (c) the bitvector oracle in C: both
strategies execute exactly the common requests of complete groups, so
the SET executed per cycle must agree cycle by cycle; only the order within a cycle differs
(first submission vs cache bit order, R20). The distributed baseline
(harness/master_worker.py, gloo) is then checked against the oracle on world sizes 2 and 3.
"""
import itertools
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

from oracle.master_worker import Coordinator, DuplicateSubmission, simulate_step
from workloads.schedules import random_mark_schedule, random_partition


# --- (a) SPEC.md worked examples ------------------------------------------------

def test_spec_gather_examples():
    c = Coordinator(2, [0, 1])
    c.gather([[0], []])
    assert c.pending == {0: [0]}
    c = Coordinator(2, [0, 1])
    c.gather([[0, 1], [0, 1]])
    assert c.pending == {0: [0, 1], 1: [0, 1]}
    with pytest.raises(DuplicateSubmission):
        Coordinator(2, [0, 1]).gather([[0, 0], []])


def test_spec_form_and_order_examples():
    c = Coordinator(2, [0, 1])
    c.gather([[0], [0]])
    assert c.form_and_order() == [0] and c.pending == {}
    c = Coordinator(2, [0, 1])
    c.gather([[0], []])
    assert c.form_and_order() == [] and c.pending == {0: [0]}     # S:121 deferred
    c.gather([[], [0]])
    assert c.form_and_order() == [0]                               # ... and executed later
    c = Coordinator(2, [0, 1])
    c.gather([[1, 0], [0, 1]])                                     # T2 submitted first
    assert c.form_and_order() == [1, 0]


def test_message_count_grows_with_world_size():
    """S:127 overhead growth: gathers + broadcasts per cycle = 2N."""
    for N in (2, 4, 8):
        c = Coordinator(N, [0])
        c.gather([[0]] * N)
        c.form_and_order()
        assert c.gathers + c.broadcasts == 2 * N


# --- (b) closed form of the order; brute force over submission permutations ----------------

def _closed_form_order(N, group_of, mark_cycle, order, resp_cycle_keys):
    """First-submission key of tensor t: (first cycle any rank submits t, first such rank,
    that rank's position of t) — R20 written as a sort key instead of a dict insertion order."""
    def key(t):
        c = min(mark_cycle[r][t] for r in range(N) if mark_cycle[r][t] >= 0)
        r = min(r for r in range(N) if mark_cycle[r][t] == c)
        return (c, r, list(order[r]).index(t))
    return sorted(resp_cycle_keys, key=key)


@pytest.mark.parametrize("T", [2, 3])
def test_order_bruteforce_permutations(T):
    """N=2, every pair of submission permutations, all tensors in cycle 0, singleton groups:
    responses follow rank 0's order (S:122-124 brute-force example, generalised)."""
    g = list(range(T))
    mark = [[0] * T, [0] * T]
    for p0 in itertools.permutations(range(T)):
        for p1 in itertools.permutations(range(T)):
            cyc, rc = simulate_step(2, g, mark, order=[p0, p1])
            assert rc == 0 and cyc[0] == list(p0)


def test_order_closed_form_random():
    for seed in range(200):
        rng = np.random.default_rng(seed)
        N = int(rng.integers(2, 6))
        T = int(rng.integers(1, 12))
        G = int(rng.integers(1, T + 1))
        g = random_partition(T, G, rng).tolist()
        mark = random_mark_schedule(N, T, seed, max_per_cycle=3).tolist()
        order = [rng.permutation(T).tolist() for _ in range(N)]
        cyc, rc = simulate_step(N, g, mark, order=order)
        assert rc == 0
        for resp in cyc:
            assert resp == _closed_form_order(N, g, mark, order, resp)


# --- (c) the executed SET per cycle equals the bitvector schedule (independent C oracle) -----

def test_same_schedule_as_bitvector_oracle(orc):
    for seed in range(300):
        rng = np.random.default_rng(10_000 + seed)
        N = int(rng.integers(1, 7))
        T = int(rng.integers(1, 40))
        G = int(rng.integers(1, T + 1))
        g = random_partition(T, G, rng)
        mark = random_mark_schedule(N, T, seed, max_per_cycle=4)
        bv = orc.simulate_step(N, g, mark)
        mw, rc = simulate_step(N, g.tolist(), mark.tolist())
        assert rc == bv.rc == 0
        assert len(mw) == bv.n_cycles
        for c in range(bv.n_cycles):
            groups = sorted({int(g[t]) for t in mw[c]})
            assert groups == bv.released[c], (seed, c)
            # whole groups only
            assert sorted(mw[c]) == sorted(t for t in range(T) if g[t] in groups)


def test_never_submitted_tensor_blocks_its_group():
    mark = [[0, 0, 0], [0, 0, -1]]
    cyc, rc = simulate_step(2, [0, 1, 1], mark, max_cycles=5)
    assert rc == 2 and cyc[0] == [0] and all(c == [] for c in cyc[1:])


# --- the distributed baseline against the oracle (gloo, world 2 and 3) ------------------------

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mw_rank(rank, N, port, cases, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=N)
    from harness.master_worker import MasterWorker
    out = []
    for g, mark, order in cases:
        mw = MasterWorker(rank, N, g)
        cycles = []
        for _ in range(2):  # two training steps through the same coordinator (state resets)
            resp_all, c = [], 0
            while True:
                ids, complete = mw.cycle([t for t in order[rank] if mark[rank][t] == c])
                resp_all.append(ids)
                c += 1
                if complete:
                    break
            cycles.append(resp_all)
        out.append(cycles)
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("N", [2, 3])
def test_distributed_master_worker_matches_oracle(N):
    cases = []
    for seed in range(12):
        rng = np.random.default_rng(500 + seed)
        T = int(rng.integers(1, 30))
        G = int(rng.integers(1, T + 1))
        g = random_partition(T, G, rng).tolist()
        mark = random_mark_schedule(N, T, seed, max_per_cycle=3).tolist()
        order = [rng.permutation(T).tolist() for _ in range(N)]
        cases.append((g, mark, order))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_mw_rank, args=(r, N, port, cases, q)) for r in range(N)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(N))
    for p in ps:
        p.join(60)
    for i, (g, mark, order) in enumerate(cases):
        want, rc = simulate_step(N, g, mark, order=order)
        assert rc == 0
        for r in range(N):
            for step in res[r][i]:
                assert step == want, (i, r)
