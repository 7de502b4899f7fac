"""The armed-cycle doorbell / acknowledgement protocol (DESIGN.md §2 "Armed cycles", gr.h
gr_step), checked exhaustively on a model.

A resident bitvector kernel serves cycle after cycle. For each sequence number k it polls the
control word of descriptor slot k % 4: the host's doorbell (k, run) makes it accept — it writes
ack = (k << 1) | 1, runs the cycle and goes on to k + 1 — a skip word (k, skip) makes it leave
silently, and its deadline may pass at any time first, when it writes ack = k << 1 and leaves.
Kernels are launched on one stream, so an instance starts only after the previous one left.
The host, per cycle: if armed, ring k and read the ack word until it decides; otherwise launch
the cycle (no kernel involved). Between cycles it may retire the kernel (gr_wait: skip word),
and it arms a new instance when none is armed. The ack word is never reset: it keeps whatever
the last instance wrote.

Claims, over every interleaving of host and kernel moves (breadth-first over the state space):
the host's decision for cycle k is "accepted" exactly when the kernel ran k, "expired" exactly
when it left at k without running it; the host never waits for an ack that cannot come; every
cycle runs exactly once. The decision rule reads the ack as (seq << 1) | accepted and also
accepts an ack already one cycle ahead (the kernel ran k and then expired waiting for k + 1).
With the first version's rule (wait for seq k exactly) the model finds the hang that the 20-min
soak found on the GPU. The model takes the host's reading branch every cycle; the branch that
skips the read (a doorbell rung well inside the kernel's lifetime) rests on the lifetime bound,
a timing argument the model does not cover.
"""
from collections import deque

import pytest

SLOTS = 4


def decide(rule, ack, k):
    """The host's reading of the ack word for cycle k: None (keep polling), or
    (accepted, kernel_gone_after)."""
    if ack is None:
        return None
    seq, acc = ack >> 1, ack & 1
    if seq == k:
        if rule == "no_acc_bit":  # mutation: any ack for k read as accepted
            return (True, False)
        return (bool(acc), not acc)
    if rule in ("ahead", "no_advance") and seq == k + 1 and not acc:
        return (True, True)  # it ran k (it only moves past k by accepting it), then expired at k + 1
    return None


def explore(rule, cycles, allow_retire=True):
    """Breadth-first over all interleavings. Returns (violations, states)."""
    # state: host (c, phase, k, armed), kernel instances (queue of start seqs; head: current seq),
    # ack, ctrl words per slot, per-cycle record (who ran it / what the host decided)
    # phase: 'top' (start of cycle c), 'wait' (rang k, polling ack), 'between' (may retire/arm)
    init = (0, "between0", 0, False, (), None, ((-1, 0),) * SLOTS, ())
    seen = {init}
    q = deque([init])
    bad = []
    while q:
        st = q.popleft()
        c, phase, k, armed, kq, ack, ctrl, rec = st
        nxt = []
        # ---- kernel moves (head instance only: one stream)
        if kq:
            kk = kq[0]
            cs, cv = ctrl[kk % SLOTS]
            if cs == kk and cv == 1:  # rung: accept, run cycle kk
                nxt.append((c, phase, k, armed, (kk + 1,) + kq[1:], (kk << 1) | 1, ctrl, rec + (("ran", kk),)))
            elif cs == kk and cv == 2:  # retired by the host
                nxt.append((c, phase, k, armed, kq[1:], ack, ctrl, rec))
            # the deadline may pass at any time before it sees the doorbell
            nxt.append((c, phase, k, armed, kq[1:], kk << 1, ctrl, rec + (("exp", kk),)))
        # ---- host moves
        if phase == "top":
            if armed:  # ring k
                ctrl2 = list(ctrl)
                ctrl2[k % SLOTS] = (k, 1)
                nxt.append((c, "wait", k, armed, kq, ack, tuple(ctrl2), rec))
            else:  # a normal launch runs the cycle
                nxt.append((c + 1, "between", k, armed, kq, ack, ctrl, rec + (("launch", c),)))
        elif phase == "wait":
            d = decide(rule, ack, k)
            if d is not None:
                accepted, gone = d
                k2 = k if rule == "no_advance" else k + 1  # mutation: the next doorbell reuses k
                if accepted:
                    nxt.append((c + 1, "between", k2, not gone, kq, ack, ctrl, rec + (("hostA", k),)))
                else:  # expired: the cycle is launched as usual
                    nxt.append((c + 1, "between", k, False, kq, ack, ctrl, rec + (("hostE", k), ("launch", c))))
        elif phase.startswith("between"):
            if c == cycles:
                if armed:  # end of run: retire
                    ctrl2 = list(ctrl)
                    ctrl2[k % SLOTS] = (k, 2)
                    nxt.append((c, "end", k, False, kq, ack, tuple(ctrl2), rec))
                else:
                    nxt.append((c, "end", k, False, kq, ack, ctrl, rec))
            else:
                if armed and allow_retire:  # gr_wait / drain / timing retire it
                    ctrl2 = list(ctrl)
                    ctrl2[k % SLOTS] = (k, 2)
                    nxt.append((c, "between", k, False, kq, ack, tuple(ctrl2), rec))
                if not armed:  # arm(): a new instance polls k + 1
                    nxt.append((c, "top", k + 1, True, kq + (k + 1,), ack, ctrl, rec))
                nxt.append((c, "top", k, armed, kq, ack, ctrl, rec))  # or go on as is
        if not nxt:
            if phase != "end" or kq:
                bad.append(("stuck", st))
            else:
                bad.extend(check(rec, cycles, st))
            continue
        for s2 in nxt:
            if s2 not in seen:
                seen.add(s2)
                q.append(s2)
    return bad, len(seen)


def check(rec, cycles, st):
    out = []
    ran = [k for e, k in rec if e == "ran"]
    exp = [k for e, k in rec if e == "exp"]
    hostA = [k for e, k in rec if e == "hostA"]
    hostE = [k for e, k in rec if e == "hostE"]
    launches = [k for e, k in rec if e == "launch"]
    if sorted(hostA) != sorted(ran):  # "accepted" exactly when the kernel ran that sequence number
        out.append(("accepted != ran", st))
    if not set(hostE) <= set(exp):  # "expired" only when the kernel left there without running it
        out.append(("expired not seen by kernel", st))
    if len(ran) + len(launches) != cycles:  # every cycle runs exactly once
        out.append(("cycle count", st))
    return out


@pytest.mark.parametrize("cycles", [1, 2, 3, 4])
def test_armed_protocol_safe(cycles):
    bad, n = explore("ahead", cycles)
    assert n > 10
    assert not bad, bad[:3]


def test_armed_protocol_exact_rule_hangs():
    """Mutation: the first version waited for an ack carrying exactly k; the model finds the
    state where the kernel already ran k and expired on k + 1, and the host waits forever."""
    bad, _ = explore("exact", 2)
    assert any(kind == "stuck" for kind, _ in bad)


@pytest.mark.parametrize("rule,kind", [("no_acc_bit", "accepted != ran"), ("no_advance", "accepted != ran")])
def test_armed_protocol_mutations(rule, kind):
    """Other plausible mistakes the model must catch: reading an expired ack as accepted (a cycle
    lost), or ringing the next cycle under the sequence number just used (the kernel has moved
    on; its later expiry reads as an acceptance)."""
    bad, _ = explore(rule, 3)
    assert any(k == kind for k, _ in bad), sorted({k for k, _ in bad})


def test_armed_protocol_no_retire():
    """Without any retirement between cycles (a tight loop of gr_step), still safe."""
    bad, _ = explore("ahead", 4, allow_retire=False)
    assert not bad, bad[:3]
