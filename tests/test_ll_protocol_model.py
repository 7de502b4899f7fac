"""The bitvector exchange's LL protocol, checked on a model.

Cycle c of every rank writes its words as (tag = c + 1) | word into its own slot of parity
c & 1, then reads every peer's slot of the same parity until the tag matches (the
AND). Each rank runs its cycles in order (one coordination stream), and ranks drift apart
arbitrarily. The claim: a reader always obtains the word the peer wrote FOR THAT cycle — a rank
can be at most one cycle ahead of the slowest peer's reads, so two slots suffice and a word is
never overwritten before every peer has read it. The model interleaves the per-word writes and
reads of N ranks at random and checks every AND against the intersection of the ranks' words;
with a single slot (no parity) the same model finds a lost word.
"""
import numpy as np
import pytest


def run(N, cycles, W, slots, seed):
    rng = np.random.default_rng(seed)
    words = rng.integers(0, 2**32, size=(cycles, N, W), dtype=np.uint64)  # rank r's word w in cycle c
    mem = [[[(0, 0)] * W for _ in range(slots)] for _ in range(N)]     # (tag, word) per rank/slot/w
    # per rank: current cycle, phase ('write' word index or 'read' (peer, word)), partial AND
    state = [{"c": 0, "w": 0, "reads": None, "acc": None} for _ in range(N)]
    results = {}
    while True:
        live = [r for r in range(N) if state[r]["c"] < cycles]
        if not live:
            break
        progressed = False
        for r in rng.permutation(live):
            s = state[r]
            c = s["c"]
            slot = c % slots
            if s["reads"] is None:  # writing phase: one word per move
                mem[r][slot][s["w"]] = (c + 1, int(words[c, r, s["w"]]))
                s["w"] += 1
                if s["w"] == W:
                    s["reads"] = [(q, w) for q in range(N) if q != r for w in range(W)]
                    s["acc"] = [int(x) for x in words[c, r]]
                progressed = True
                break
            if s["reads"]:
                q, w = s["reads"][0]
                tag, val = mem[q][slot][w]
                if tag == c + 1:  # the peer's word for this cycle
                    s["acc"][w] &= val
                    s["reads"].pop(0)
                    progressed = True
                    break
                continue  # stale tag: re-poll later
            results[(r, c)] = s["acc"]
            s.update(c=c + 1, w=0, reads=None, acc=None)
            progressed = True
            break
        if not progressed:
            return None  # stuck: a word the reader needed was overwritten
    for (r, c), acc in results.items():
        want = [int(np.bitwise_and.reduce(words[c, :, w])) for w in range(W)]
        if acc != want:
            return False
    return True


@pytest.mark.parametrize("N", [2, 3, 4, 8])
def test_two_slots_always_deliver_the_cycles_words(N):
    for seed in range(40):
        assert run(N, cycles=12, W=3, slots=2, seed=seed) is True


def test_one_slot_loses_words():
    """Without the parity double buffer a fast rank overwrites a word a slow peer still needs."""
    outcomes = {run(3, cycles=12, W=3, slots=1, seed=s) for s in range(40)}
    assert None in outcomes
