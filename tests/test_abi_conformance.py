"""ABI conformance: the same call scripts through the oracle's simulation of the §8(b) contract
(oracle/abi.py: N simulated ranks in one object) and through libgr.so (include/gr.h), compared
call by call — return codes, released lists, the intersected bitvector A_c, step_complete, and
every gradient byte after each step.

CPU (-m "not gpu"): gr_init's argument validation against the oracle's on dry contexts; the
oracle world itself pinned against the pinned step simulator and against the contract's error
rules written out literally. GPU (-m gpu): random scripts with injected errors (duplicate marks,
bad ids, null pointers, marks after the step completed, ABORT / SHUTDOWN raised by one rank,
never-marked tensors) at N = 1 (gr_init) and N = 2, 3, 4 (virtual ranks, gr_init_virtual).
"""
import ctypes

import numpy as np
import pytest

import oracle
from oracle import abi as oabi
from workloads.schedules import random_mark_schedule, random_partition
from workloads.values import tensor_scales, values_np


def _raw_init_code(N, numel, grad_dtype, group_of, G, buffer_dtype, rank=0):
    """gr_init straight through ctypes (dry: device = -1, no CUDA), any T / G / table."""
    from paper_1909_11150_b200 import binding as b
    T = len(numel)
    tab = (b.GrTensor * max(1, T))()
    for t in range(T):
        tab[t].numel = int(numel[t])
        tab[t].grad_dtype = int(grad_dtype[t])
    grp = (ctypes.c_int32 * max(1, T))(*[int(g) for g in group_of])
    ag = b.ALLGATHER_FN(lambda send, recv, n, user: (ctypes.memmove(recv, send, n), 0)[1])
    # a world of N ranks whose allgather returns N copies of this rank's bytes (every rank equal)
    def cb(send, recv, n, user):
        for r in range(N):
            ctypes.memmove(recv + r * n, send, n)
        return 0
    agN = b.ALLGATHER_FN(cb)
    w = b.GrWorld(rank, N, -1, None, buffer_dtype, -1, 0, 0, 0, agN if N > 1 else ag, None)
    ctx = ctypes.c_void_p()
    rc = b.lib.gr_init(ctypes.byref(ctx), ctypes.byref(w), tab, T, ctypes.cast(grp, ctypes.c_void_p), G)
    if rc == 0:
        b.lib.gr_finalize(ctx)
    return rc


def _init_cases():
    rng = np.random.default_rng(5)
    cases = []
    for _ in range(40):  # valid tables
        T = int(rng.integers(1, 40))
        G = int(rng.integers(1, T + 1))
        cases.append((int(rng.integers(1, 9)), rng.integers(1, 1000, T).tolist(), rng.integers(0, 2, T).tolist(),
                      random_partition(T, G, rng).tolist(), G, int(rng.integers(0, 2))))
    base = (2, [5, 6, 7, 8], [0, 0, 1, 0], [0, 1, 1, 2], 3, 1)
    def mod(**kw):
        N, numel, dt, grp, G, bd = base
        d = dict(N=N, numel=list(numel), dt=list(dt), grp=list(grp), G=G, bd=bd)
        d.update(kw)
        return (d["N"], d["numel"], d["dt"], d["grp"], d["G"], d["bd"])
    cases += [base, mod(N=0), mod(N=9), mod(numel=[5, 0, 7, 8]), mod(numel=[5, -3, 7, 8]),
              mod(dt=[0, 2, 0, 0]), mod(grp=[0, 1, 1, 3]), mod(grp=[0, -1, 1, 2]), mod(G=4),
              mod(G=5), mod(G=0), mod(bd=2), mod(bd=-1), mod(grp=[0, 0, 2, 2]),
              (1, [1], [0], [0], 1, 0), (8, [3] * 8, [1] * 8, list(range(8)), 8, 0)]
    return cases


def test_init_validation_matches_oracle():
    """gr_init's GR_EINVAL cases (numel <= 0, bad dtype, group ids not dense /
    groups empty, world size outside 1..8, G > T) agree with the oracle's validate_init."""
    for N, numel, dt, grp, G, bd in _init_cases():
        want = oabi.validate_init(N, numel, dt, grp, G, bd)
        got = _raw_init_code(N, numel, dt, grp, G, bd)
        assert got == want, (N, numel, dt, grp, G, bd, got, want)


def _values(seed, r, t, n, f16):
    s = tensor_scales(seed, 64)
    v = values_np(seed, r, t, np.arange(n), float(s[t % 64]))
    return v.astype(np.float16).astype(np.float32) if f16 else v


def test_oracle_world_matches_step_simulator():
    """The oracle world, driven mark by mark, reproduces orc_simulate_step (pinned by brute
    force and the closed form, tests/test_oracle_schedule.py) cycle for cycle, and writes
    oracle.emulate's values into every rank's arrays exactly once per tensor."""
    for seed in range(30):
        rng = np.random.default_rng(seed)
        N = int(rng.integers(1, 5))
        T = int(rng.integers(1, 12))
        G = int(rng.integers(1, T + 1))
        grp = random_partition(T, G, rng)
        numel = rng.integers(1, 50, T)
        mark = random_mark_schedule(N, T, seed, 2)
        w = oabi.OracleWorld(N, numel, grp, G, oabi.F16)
        arrays = [[_values(seed, r, t, int(numel[t]), False).copy() for t in range(T)] for r in range(N)]
        ref = oracle.simulate_step(N, grp, mark, max_cycles=50)
        for c in range(ref.n_cycles):
            for r in range(N):
                for t in np.nonzero(mark[r] == c)[0]:
                    assert w.mark(r, int(t), arrays[r][t]) == oabi.OK
            res = w.step_all()
            assert all(x[0] == oabi.OK for x in res)
            assert [int(a) for a in res[0][2]] == [int(a) for a in ref.A[c]]
            assert res[0][1] == ref.released[c]
        assert w.step_complete
        for t in range(T):
            want = oracle.emulate([_values(seed, r, t, int(numel[t]), False) for r in range(N)], True, False)
            for r in range(N):
                assert np.array_equal(arrays[r][t].view(np.uint32), want.view(np.uint32))


def test_oracle_world_error_rules():
    """The contract's lifecycle rules, literally (SURVEY.md §8(b) errors
    DuplicateSubmission; SPEC.md:221-222 status bits; readings R13, R15)."""
    w = oabi.OracleWorld(2, [4, 4, 4], [0, 0, 1], 2, oabi.F32)
    a = [[np.ones(4, np.float32) * (r + 1) for _ in range(3)] for r in range(2)]
    assert w.mark(0, 3, a[0][0]) == oabi.EINVAL        # bad id
    assert w.mark(0, -1, a[0][0]) == oabi.EINVAL
    assert w.mark(0, 0, None) == oabi.EINVAL           # null pointer
    assert w.mark(0, 0, a[0][0]) == oabi.OK
    assert w.mark(0, 0, a[0][0]) == oabi.ESTATE        # duplicate in a step
    for t in (1, 2):
        assert w.mark(0, t, a[0][t]) == oabi.OK
    res = w.step_all()                                 # rank 1 marked nothing: nothing released
    assert [x[1] for x in res] == [[], []] and not res[0][3]
    for t in range(3):
        assert w.mark(1, t, a[1][t]) == oabi.OK
    res = w.step_all()
    assert [x[1] for x in res] == [[0, 1], [0, 1]] and res[0][3]
    assert np.all(a[0][0] == 1.5) and np.all(a[1][2] == 1.5)
    assert w.mark(0, 0, a[0][0]) == oabi.ESTATE        # step complete, gr_wait not called
    assert w.step_all()[0][0] == oabi.ESTATE
    assert w.wait_all() == [oabi.OK, oabi.OK]
    assert w.mark(0, 0, a[0][0]) == oabi.OK            # next step
    w.set_status(1, True, False)
    res = w.step_all()
    assert [x[0] for x in res] == [oabi.EABORT, oabi.EABORT] and res[0][1] == []
    assert not (int(res[0][2][0]) & 1)                  # complement-coded ABORT bit cleared
    assert w.mark(0, 1, a[0][1]) == oabi.ESTATE        # sticky
    w2 = oabi.OracleWorld(3, [4], [0], 1, oabi.F16)
    w2.set_status(2, False, True)
    assert [x[0] for x in w2.step_all()] == [oabi.ESHUTDOWN] * 3
    w3 = oabi.OracleWorld(2, [4], [0], 1, oabi.F16)
    w3.set_status(0, True, True)                        # ABORT takes precedence (reading R13)
    assert [x[0] for x in w3.step_all()] == [oabi.EABORT] * 2


# ------------------------------------------------------------------ GPU: scripts on both sides

def make_script(seed, N, T, G, steps=2, inject=True):
    """Random call script: per step, cycles of per-rank marks (random order, 0-3 per cycle) then
    one collective step; injected errors: duplicate marks, bad ids, null pointers, marks after
    the step completed; optionally a status flag raised by one rank (ends the script)."""
    rng = np.random.default_rng(seed)
    ops = []
    status_at = (int(rng.integers(0, steps)), int(rng.integers(0, 3)), int(rng.integers(0, N)),
                 int(rng.integers(0, 2))) if inject and rng.random() < 0.3 else None
    never = int(rng.integers(0, T)) if inject and rng.random() < 0.15 else None
    for s in range(steps):
        orders = [list(rng.permutation(T)) for _ in range(N)]
        if never is not None and s == steps - 1:
            orders[N - 1] = [t for t in orders[N - 1] if t != never]
        c = 0
        while any(orders) and c < 3 * T + 4:
            for r in range(N):
                k = int(rng.integers(0, 4))
                for _ in range(k):
                    if not orders[r]:
                        break
                    t = orders[r].pop(0)
                    ops.append(("mark", r, t, False))
                    if inject and rng.random() < 0.08:
                        ops.append(("mark", r, t, False))                  # duplicate -> ESTATE
                    if inject and rng.random() < 0.05:
                        ops.append(("mark", r, int(rng.choice([-1, T, T + 7])), False))  # bad id
                    if inject and rng.random() < 0.05:
                        ops.append(("mark", r, int(rng.integers(0, T)), True))  # null pointer
            if status_at and status_at[0] == s and status_at[1] == c:
                ops.append(("status", status_at[2], status_at[3] == 0, status_at[3] == 1))
                ops.append(("step",))
                ops.append(("mark", 0, 0, False))                           # sticky -> ESTATE
                return ops
            ops.append(("step",))
            c += 1
        for _ in range(3):
            ops.append(("step",))  # drains the step (ESTATE once complete), or cycles on (never-marked)
        if inject and rng.random() < 0.5:
            ops.append(("mark", int(rng.integers(0, N)), int(rng.integers(0, T)), False))  # after complete
        if never is not None and s == steps - 1:
            return ops
        ops.append(("wait",))
    return ops


def run_oracle(ops, N, numel, grp, G, buf16, grad_f16, seed):
    w = oabi.OracleWorld(N, numel, grp, G, oabi.F16 if buf16 else oabi.F32, [int(x) for x in grad_f16])
    arrays = [[_values(seed + 1000 * k, r, t, int(numel[t]), grad_f16[t]).copy() for t in range(len(numel))]
              for k in range(8) for r in range(N)]
    log, snaps, step_no = [], [], 0
    cur = lambda r: arrays[step_no * N + r]  # noqa: E731 — fresh gradients per step
    for op in ops:
        if op[0] == "mark":
            _, r, t, null = op
            a = None if null else (cur(r)[t] if 0 <= t < len(numel) else np.zeros(1, np.float32))
            log.append(("mark", r, w.mark(r, t, a)))
        elif op[0] == "status":
            w.set_status(op[1], op[2], op[3])
        elif op[0] == "step":
            res = w.step_all()
            log.append(("step", [(x[0], x[1] if x[0] == 0 else None,
                                  [int(v) for v in x[2]] if x[0] == 0 else None, x[3] if x[0] == 0 else None)
                                 for x in res]))
        else:
            w.wait_all()
            snaps.append([[cur(r)[t].copy() for t in range(len(numel))] for r in range(N)])
            step_no += 1
    snaps.append([[cur(r)[t].copy() for t in range(len(numel))] for r in range(N)])
    return log, snaps


def run_gpu(ops, N, numel, grp, buf16, grad_f16, seed, dev):
    import torch

    from paper_1909_11150_b200 import GR_F16, GR_F32, Context, GrError, virtual_world
    from tests.parity_lib import run_ranks
    kw = dict(numel=numel, group_of=grp, grad_f16=grad_f16, buffer_dtype=GR_F16 if buf16 else GR_F32,
              timeout_ms=20000)
    ctxs = virtual_world(world_size=N, device=0, **kw) if N > 1 else [Context(rank=0, world_size=1, device=0, **kw)]
    T = len(numel)

    def tens(k, r, t):
        v = torch.from_numpy(_values(seed + 1000 * k, r, t, int(numel[t]), grad_f16[t]))
        return v.to(dev).half() if grad_f16[t] else v.to(dev)

    grads = [[tens(k, r, t) for t in range(T)] for k in range(8) for r in range(N)]
    torch.cuda.synchronize()
    log, snaps, step_no = [], [], 0
    try:
        for op in ops:
            if op[0] == "mark":
                _, r, t, null = op
                ptr = 0 if null else (grads[step_no * N + r][t].data_ptr() if 0 <= t < T else grads[0][0].data_ptr())
                try:
                    ctxs[r].gr_mark_ready(t, ptr)
                    code = 0
                except GrError as e:
                    code = e.code
                log.append(("mark", r, code))
            elif op[0] == "status":
                ctxs[op[1]].gr_set_status(op[2], op[3])
            elif op[0] == "step":
                def one(r):
                    try:
                        rel, complete, A, _ = ctxs[r].gr_step()
                        return (0, list(rel), [int(v) for v in A], bool(complete))
                    except GrError as e:
                        return (e.code, None, None, None)
                log.append(("step", run_ranks(N, one)))
            else:
                for c in ctxs:
                    c.gr_wait()
                snaps.append([[grads[step_no * N + r][t].float().cpu().numpy() for t in range(T)] for r in range(N)])
                step_no += 1
        for c in ctxs:
            try:
                c.gr_wait()
            except GrError:
                pass
        torch.cuda.synchronize()
        snaps.append([[grads[step_no * N + r][t].float().cpu().numpy() for t in range(T)] for r in range(N)])
    finally:
        for c in ctxs:
            c.gr_finalize()
    return log, snaps


@pytest.mark.gpu
@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_conformance_scripts(N):
    from tests.conftest import gpu_count
    if gpu_count() < 1:
        pytest.skip("no GPU")
    import torch
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    for seed in range(10 if N > 1 else 16):
        rng = np.random.default_rng(seed + 100 * N)
        T = int(rng.integers(1, 10))
        G = int(rng.integers(1, T + 1))
        grp = random_partition(T, G, rng).tolist()
        numel = rng.integers(1, 3000, T).tolist()
        grad_f16 = (rng.random(T) < 0.3).tolist()
        buf16 = bool(seed % 2)
        ops = make_script(seed, N, T, G)
        want_log, want_snaps = run_oracle(ops, N, numel, grp, G, buf16, grad_f16, seed)
        got_log, got_snaps = run_gpu(ops, N, numel, grp, buf16, grad_f16, seed, dev)
        assert len(got_log) == len(want_log)
        for i, (g, w) in enumerate(zip(got_log, want_log)):
            assert g == w, f"N={N} seed {seed} call {i} ({ops_desc(ops, i)}): gpu {g} oracle {w}"
        for k, (gs, ws) in enumerate(zip(got_snaps, want_snaps)):
            for r in range(N):
                for t in range(T):
                    assert np.array_equal(gs[r][t].astype(np.float32).view(np.uint32),
                                          ws[r][t].astype(np.float32).view(np.uint32)), \
                        f"N={N} seed {seed} step {k} rank {r} tensor {t}: values differ"


def ops_desc(ops, i):
    k = -1
    for op in ops:
        if op[0] in ("mark", "step"):
            k += 1
            if k == i:
                return op
    return None
