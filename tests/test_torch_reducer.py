"""Host logic of the autograd integration (NEXT-3) on CPU: the cycle driver issues the same
sequence of collective calls (gr_step / gr_step_drain) on every rank whatever each rank's
local readiness order, and every group is released exactly once (gloo, world sizes 2 and 3).

The collective calls are stood in for by a gloo all_gather of (call kind, local ready bits):
a cycle releases the groups ready on every rank, a drain releases all
remaining groups; a rank whose call kind differs from a peer's at the same position fails.
"""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

from paper_1909_11150_b200.torch_reducer import contiguous_groups, drive_cycles


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, N, port, seeds, q):
    try:
        q.put((rank, _rank_body(rank, N, port, seeds)))
    except Exception as e:  # a desynchronised peer fails fast (gloo timeout) instead of hanging
        q.put((rank, f"error: {e!r}"))


def _rank_body(rank, N, port, seeds):
    import datetime

    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=N, timeout=datetime.timedelta(seconds=20))
    out = []
    for seed in seeds:
        rng = np.random.default_rng(seed * 31 + rank)
        G = int(np.random.default_rng(seed).integers(1, 9))
        drain_tail = int(np.random.default_rng(seed + 1).integers(0, 3))
        # this rank's backward produces the groups in a (rank-dependent, mostly shared) order;
        # each wait_group lets the device run ahead by a random number of further groups
        order = list(range(G))
        if rng.random() < 0.5 and G > 1:
            i = int(rng.integers(0, G - 1))
            order[i], order[i + 1] = order[i + 1], order[i]
        ready = np.zeros(G, dtype=bool)
        released = np.zeros(G, dtype=bool)
        log = []

        def collective(kind):
            mine = torch.tensor([kind] + [int(x) for x in (ready & ~released)], dtype=torch.int64)
            allv = [torch.zeros_like(mine) for _ in range(N)]
            dist.all_gather(allv, mine)
            kinds = {int(v[0]) for v in allv}
            assert len(kinds) == 1, f"rank {rank}: collective call kinds differ {kinds}"
            if kind == 2:  # drain: every remaining group
                rel = [g for g in range(G) if not released[g]]
            else:
                both = np.all(np.stack([v[1:].numpy() for v in allv]) > 0, axis=0)
                rel = [g for g in range(G) if both[g]]
            for g in rel:
                assert not released[g]
                released[g] = True
            log.append((kind, tuple(rel)))
            return rel, bool(released.all())

        def wait_group(g):
            pos = order.index(g)
            ahead = pos + int(rng.integers(0, 3))
            for h in order[:ahead + 1]:
                ready[h] = True

        def step():
            if rng.random() < 0.3:  # the device made progress meanwhile
                for h in order:
                    if not ready[h]:
                        ready[h] = True
                        break
            return collective(1)

        def drain():
            ready[:] = True
            collective(2)

        n = drive_cycles(step, drain, wait_group, order, G, drain_tail)
        assert released.all(), f"rank {rank} seed {seed}: not every group released"
        out.append((n, log))
    dist.destroy_process_group()
    return out


@pytest.mark.parametrize("N", [2, 3])
def test_cycle_driver_lockstep_gloo(N):
    seeds = list(range(40))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank, args=(r, N, port, seeds, q)) for r in range(N)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(N))
    for p in ps:
        p.join(60)
    for r in range(N):
        assert not isinstance(res[r], str), res[r]
    for i in range(len(seeds)):
        logs = [res[r][i] for r in range(N)]
        assert all(x == logs[0] for x in logs), (i, logs)


def test_contiguous_groups_cover_in_reverse_order():
    numels = [5, 100, 3, 40, 40, 7, 90]
    g = contiguous_groups(numels, 3)
    assert sorted(set(g)) == [0, 1, 2]
    rev = [g[t] for t in reversed(range(len(numels)))]
    assert rev == sorted(rev)  # group ids ascend in backward (reverse registration) order


@pytest.mark.parametrize("numels,n_groups", [([5], 4), ([1, 1], 8), ([10] * 7, 3), ([1, 1000, 1, 1], 2),
                                             ([3, 3, 3, 3, 3, 3, 3, 3], 8)])
def test_contiguous_groups_edge_cases(numels, n_groups):
    """Dense ids 0..G-1 (G <= min(T, n_groups)), every group non-empty and contiguous in the
    backward (reverse registration) order, ids ascending in that order."""
    g = contiguous_groups(numels, n_groups)
    T = len(numels)
    G = len(set(g))
    assert sorted(set(g)) == list(range(G)) and 1 <= G <= min(T, n_groups)
    rev = [g[t] for t in reversed(range(T))]
    assert rev == sorted(rev)
