"""CPU oracle for the master-worker coordination baseline: the
strategy the paper's Bitvector Allreduce replaces.

TEST INFRASTRUCTURE ONLY (same rule as the rest of ``oracle/``): only ``tests/`` may import it.
It shares no code with ``harness/master_worker.py`` (the distributed baseline it checks).

PAPER.md:108 §4.1 — "a single coordinator rank is tasked with gathering *requests* from all
workers, determining common requests across workers, forming *responses* for common requests,
and then broadcasting an ordered list of responses to all workers for execution"; PAPER.md:110 —
at each tic "only common collective operation requests across workers are executed";
PAPER.md:130 Fig. 3a caption (i)-(iv). Requests are sent once, when a tensor becomes pending
(the caching scheme exists because requests "are redundantly communicated to the
coordinator rank" every iteration, not every cycle).

Readings (R20-R21):
- R20 response order: first-submission order at the coordinator (the first rank to submit a key
  fixes its position; within one gather, rank 0's list first, each list in submission order).
  SPEC.md:116-124 (form_and_order) and its design decision "first-arrival order".
- R21 Grouping on top of master-worker: a common request is executed only when
  every request of its group is common; held-back keys keep their first-submission position.
  With singleton groups this is the plain master-worker of Fig. 3a.
"""
from __future__ import annotations


class DuplicateSubmission(Exception):
    """A rank submitted the same key twice in one step."""


class Coordinator:
    """Rank 0's state (SPEC.md:100-103 CoordinatorState)."""

    def __init__(self, N: int, group_of):
        self.N = N
        self.group_of = list(group_of)
        self.group_size = {}
        for g in self.group_of:
            self.group_size[g] = self.group_size.get(g, 0) + 1
        self.pending = {}          # key -> ranks that submitted it; dict order = first submission
        self.common = set()        # keys submitted by all N ranks, not yet executed
        self.gathers = 0           # logical messages (SPEC.md:101 message_counter)
        self.broadcasts = 0

    def gather(self, rank_requests):
        """Fig. 3a (i): requests of every rank, rank order."""
        assert len(rank_requests) == self.N
        for r, reqs in enumerate(rank_requests):
            for key in reqs:
                ranks = self.pending.setdefault(key, [])
                if r in ranks:
                    raise DuplicateSubmission(f"rank {r} submitted {key} twice")
                ranks.append(r)
                # (ii) common request: submitted by every rank
                if len(ranks) == self.N:
                    self.common.add(key)
        self.gathers += self.N

    def form_and_order(self):
        """Fig. 3a (iii)-(iv): responses for common requests whose group is complete, in
        first-submission order; executed keys leave ``pending``."""
        done_in_group = {}
        for key in self.common:
            g = self.group_of[key]
            done_in_group[g] = done_in_group.get(g, 0) + 1
        out = [key for key in self.pending
               if key in self.common and done_in_group[self.group_of[key]] == self.group_size[self.group_of[key]]]
        for key in out:
            del self.pending[key]
            self.common.discard(key)
        self.broadcasts += self.N
        return out


def simulate_step(N: int, group_of, mark_cycle, order=None, max_cycles: int = 1000):
    """One training step of N simulated ranks under master-worker coordination.

    mark_cycle[r][t] = cycles rank r completes before submitting t (-1: never);
    order[r] = the sequence in which rank r submits its tensors (default: ascending id).
    Returns (responses per cycle as ordered tensor lists, rc) with rc 0 = every tensor executed,
    2 = cycle bound hit."""
    T = len(group_of)
    co = Coordinator(N, group_of)
    seq = [list(order[r]) if order is not None else list(range(T)) for r in range(N)]
    executed = 0
    cycles = []
    for c in range(max_cycles):
        reqs = [[t for t in seq[r] if mark_cycle[r][t] == c] for r in range(N)]
        co.gather(reqs)
        resp = co.form_and_order()
        cycles.append(resp)
        executed += len(resp)
        if executed == T:
            return cycles, 0
    return cycles, 2
