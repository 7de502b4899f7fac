"""The ordering argument of xfer_kernel's work queue, checked on a model.

Each rank's CTAs take triples k = 0, 1, ... from a per-rank counter; triple k holds PACK(k)
(two-shot: non-owned chunks), RS(k - L1) (owned chunks: needs every peer's PACK of that chunk)
and AG(k - L2) (non-owned chunks: needs the owner's RS), processed in that order, a CTA blocking
on a missing flag. The claim: whatever subset of CTAs is resident (down to one per rank) and
however the ranks' CTAs interleave, every step completes, because every dependency points to an
earlier triple in every rank's queue (lags 0 <= L1 < L2). The model also shows the claim fails
without the lag order (L2 < L1: the all-gather of a chunk is queued before its reduce-scatter).
"""
import numpy as np
import pytest


def simulate(N, P, total, L1, L2, seed, max_steps=200000):
    """Returns True when every rank finished its queue, False on deadlock."""
    rng = np.random.default_rng(seed)
    nk = total + max(L1, L2)
    packed = np.zeros((N, total), bool)   # packed[r, c]: rank r's PACK(c) published
    reduced = np.zeros(total, bool)        # reduced[c]: owner's RS(c) published
    counter = [0] * N
    # CTA state: (triple k, phase 0/1/2/3 = next item PACK/RS/AG/take-next) or None when idle
    ctas = [[None] * P for _ in range(N)]
    done_ranks = 0
    for _ in range(max_steps):
        movable = []
        for r in range(N):
            for i in range(P):
                st = ctas[r][i]
                if st is None:
                    if counter[r] < nk:
                        movable.append((r, i))
                    continue
                k, ph = st
                if ph == 1:  # RS(k-L1) on the owner: every peer's PACK
                    c = k - L1
                    if 0 <= c < total and c % N == r and not all(packed[q, c] for q in range(N) if q != r):
                        continue
                if ph == 2:  # AG(k-L2) on a non-owner: the owner's RS
                    c = k - L2
                    if 0 <= c < total and c % N != r and not reduced[c]:
                        continue
                movable.append((r, i))
        if not movable:
            finished = all(counter[r] >= nk and all(s is None for s in ctas[r]) for r in range(N))
            return finished
        r, i = movable[rng.integers(len(movable))]
        st = ctas[r][i]
        if st is None:
            ctas[r][i] = (counter[r], 0)
            counter[r] += 1
            continue
        k, ph = st
        if ph == 0:
            if k < total and k % N != r:
                packed[r, k] = True
        elif ph == 1:
            c = k - L1
            if 0 <= c < total and c % N == r:
                reduced[c] = True
        elif ph == 2:
            pass  # the all-gather only consumes
        ctas[r][i] = None if ph == 2 else (k, ph + 1)
    raise AssertionError("step bound hit")


@pytest.mark.parametrize("N", [2, 4, 8])
def test_queue_never_deadlocks_with_ordered_lags(N):
    rng = np.random.default_rng(N)
    for case in range(60):
        P = int(rng.integers(1, 4))            # resident CTAs per rank, down to one
        total = int(rng.integers(1, 40))
        L1 = int(rng.integers(0, 12))
        L2 = L1 + int(rng.integers(1, 12))
        assert simulate(N, P, total, L1, L2, seed=case), (N, P, total, L1, L2)


def test_queue_with_unordered_lags_can_deadlock():
    """The argument needs L1 < L2: with the all-gather queued before the reduce-scatter of the
    same chunk and one CTA per rank, the model deadlocks."""
    assert not simulate(2, 1, 8, L1=6, L2=0, seed=0)
