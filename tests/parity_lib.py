"""GPU-vs-oracle parity checks shared by the -m gpu tests, the torchrun worker
(tests/mp_worker.py) and __graft_entry__.smoke().

The bar:
* schedule: per cycle, the intersected bitvector A_c (status bits included)
  and the released group list are BIT-EXACT against oracle.simulate_step;
* values: every reduced gradient element is bit-exact against
  oracle.emulate (fp32 rank-order sum, x fl32(1/N), buffer/grad rounding —
  readings R7-R9), AND within the north-star tolerance of the fp64 reference
  oracle.reduce_f64: |out-ref| <= 1e-6*max(|ref|, mean_r|g_r|) for fp32
  buffers (reading R10), |out-ref| <= 2^-10*N*max|g| for fp16 (reading R11);
* cross-rank: gradients identical bit for bit on every rank (checked by the
  caller through a hash allgather).
"""
from __future__ import annotations

import hashlib

import numpy as np

import oracle
from harness.replay import make_grads, replay_step
from workloads.values import tensor_scales, values_np


def sample_indices(n: int, seed: int, full_below: int = 1 << 20, k: int = 1 << 16):
    """All indices of small tensors; for large ones the head, the tail and k random ones."""
    if n <= full_below:
        return np.arange(n)
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([np.arange(4096), np.arange(n - 4096, n), rng.integers(0, n, k)]))


def host_inputs(numel, N, seed, t, grad_f16_t: bool, kind: str = "uniform", idx=None):
    s = tensor_scales(seed, len(numel))
    if idx is None:
        idx = np.arange(int(numel[t]))
    gs = []
    for r in range(N):
        v = values_np(seed, r, t, idx, float(s[t]), kind)
        if grad_f16_t:
            v = v.astype(np.float16).astype(np.float32)
        gs.append(v)
    return gs


def check_schedule(log, ref, where=""):
    assert log.n_cycles == ref.n_cycles, f"{where}: cycles gpu={log.n_cycles} oracle={ref.n_cycles}"
    for c in range(ref.n_cycles):
        assert [int(x) for x in log.A[c]] == [int(x) for x in ref.A[c]], \
            f"{where}: cycle {c} A gpu={log.A[c]} oracle={list(ref.A[c])}"
        assert log.released[c] == ref.released[c], \
            f"{where}: cycle {c} released gpu={log.released[c]} oracle={ref.released[c]}"


def check_values(out_np, gs, N, buffer_f16: bool, grad_f16_t: bool, where="", exact: bool = True):
    """exact=False (NVLS: the switch accumulates in its own order) keeps only the north-star
    tolerance; integer payloads are exact in any order and are checked with exact=True."""
    emu = oracle.emulate(gs, buffer_f16, grad_f16_t)
    ref = oracle.reduce_f64(gs)
    out = out_np.astype(np.float32)
    both_nan = np.isnan(out) & np.isnan(emu)  # NaN payloads are not part of the contract
    bad = np.nonzero((out.view(np.uint32) != emu.view(np.uint32)) & ~both_nan)[0]
    if exact:
        assert bad.size == 0, (f"{where}: {bad.size} elements differ from the oracle emulation, first "
                               f"i={bad[0]} gpu={out[bad[0]]!r} emu={emu[bad[0]]!r}")
    o64 = out.astype(np.float64)
    stack = np.stack(gs).astype(np.float64)
    fin = np.all(np.isfinite(stack), axis=0)
    if not np.all(fin):  # IEEE specials propagate: the exact sum's class (inf of its sign, or NaN)
        r_nf, o_nf = ref[~fin], o64[~fin]
        assert np.array_equal(np.isnan(o_nf), np.isnan(r_nf)), f"{where}: NaN not propagated"
        keep = ~np.isnan(r_nf)
        assert np.array_equal(o_nf[keep], r_nf[keep]), f"{where}: Inf not propagated"
        o64, ref, stack = o64[fin], ref[fin], stack[:, fin]
        if o64.size == 0:
            return
    if buffer_f16:
        # reading R11: the north-star bound is relative; a tensor whose values all sit in fp16's
        # subnormal range (|g| < 2^-14) is rounded with an absolute error, so the bound gains the
        # subnormal quantum 2^-24 (input + output rounding, 2^-25 each)
        tol = 2.0 ** -10 * N * float(np.max(np.abs(stack))) + 2.0 ** -24
        assert np.all(np.abs(o64 - ref) <= tol), f"{where}: fp16 tolerance violated"
    else:
        bound = 1e-6 * np.maximum(np.abs(ref), np.mean(np.abs(stack), axis=0))
        if grad_f16_t:  # fp16 gradient storage adds one output rounding (half an fp16 ulp)
            bound = bound + np.abs(ref) * 2.0 ** -11 + 2.0 ** -25
        assert np.all(np.abs(o64 - ref) <= bound), f"{where}: fp32 tolerance violated"


def run_case_on_rank(ctx, case, r, seed, device, buffer_f16: bool, grad_f16=None, kind="uniform",
                     max_cycles=None, async_stream=None, exact: bool = True, before_step=None):
    """Replay `case` on rank r through the C ABI and check it against the oracle.
    Returns (log, sha256 of all output gradients) for the cross-rank comparison."""
    import torch

    T = case.T
    if max_cycles is None:
        max_cycles = int(np.max(case.mark_cycle)) + 2
    grads = make_grads(case.numel, r, seed, device, grad_f16, kind)
    torch.cuda.synchronize(device)
    log = replay_step(ctx, case.mark_cycle[r], [g.data_ptr() for g in grads], max_cycles,
                      async_stream=async_stream, before_step=before_step)
    ref = oracle.simulate_step(case.N, case.group_of, case.mark_cycle, max_cycles=max_cycles)
    check_schedule(log, ref, where=f"rank {r} seed {seed}")
    released_groups = {g for rel in ref.released for g in rel}
    h = hashlib.sha256()
    for t in range(T):
        f16 = bool(grad_f16 is not None and grad_f16[t])
        out = grads[t].float().cpu().numpy()
        h.update(out.tobytes())
        if int(case.group_of[t]) not in released_groups:
            continue
        idx = sample_indices(out.size, seed * 7919 + t)
        gs = host_inputs(case.numel, case.N, seed, t, f16, kind, idx)
        check_values(out[idx], gs, case.N, buffer_f16, f16, where=f"rank {r} seed {seed} tensor {t}",
                     exact=exact or kind == "int")
    return log, h.hexdigest()


def check_grad_stats(ctx, case, seed, buffer_f16: bool, grad_f16=None, kind="uniform", exact: bool = True,
                     where=""):
    """NEXT-2 epilogue: per-tensor sum of squares of the reduced gradient against the fp64 sum of
    squares of the oracle's emulated values (relative 1e-6: the kernels sum fp32 squares of 8
    values before the fp64 accumulation), and the non-finite flag (False for finite inputs)."""
    sumsq, nonfinite = ctx.gr_grad_stats()
    assert not nonfinite, f"{where}: non-finite flag set on finite inputs"
    for t in range(case.T):
        f16 = bool(grad_f16 is not None and grad_f16[t])
        gs = host_inputs(case.numel, case.N, seed, t, f16, kind)
        emu = oracle.emulate(gs, buffer_f16, f16).astype(np.float64)
        want = float(np.sum(emu * emu))
        tol = 1e-6 * want + 1e-30
        if not exact:  # NVLS: values within the north-star tolerance, so compare loosely
            tol = 2.0 ** -9 * want + 1e-30
        assert abs(sumsq[t] - want) <= tol, f"{where}: tensor {t} sumsq gpu={sumsq[t]!r} oracle={want!r}"
    return sumsq


def run_drain_case_on_rank(ctx, case, r, seed, device, buffer_f16: bool, drain_after: int, async_stream=None):
    """gr_step_drain: the first `drain_after` cycles follow the oracle's schedule exactly; the
    drain cycle then releases every remaining group, so every tensor ends up reduced — values
    bit-exact against the oracle's emulation (they do not depend on the schedule, R5)."""
    import torch

    grads = make_grads(case.numel, r, seed, device)
    torch.cuda.synchronize(device)
    log = replay_step(ctx, case.mark_cycle[r], [g.data_ptr() for g in grads], 1000,
                      async_stream=async_stream, drain_after=drain_after)
    ref = oracle.simulate_step(case.N, case.group_of, case.mark_cycle, max_cycles=1000)
    k = len(log.released)
    assert log.released == ref.released[:k], f"rank {r} seed {seed}: pre-drain schedule {log.released} != {ref.released[:k]}"
    h = hashlib.sha256()
    for t in range(case.T):
        out = grads[t].float().cpu().numpy()
        h.update(out.tobytes())
        idx = sample_indices(out.size, seed * 7919 + t)
        gs = host_inputs(case.numel, case.N, seed, t, False, "uniform", idx)
        check_values(out[idx], gs, case.N, buffer_f16, False, where=f"rank {r} seed {seed} tensor {t} (drain)")
    return log, h.hexdigest()


def run_ranks(N: int, fn, timeout: float = 600.0):
    """Run fn(r) for r in 0..N-1 concurrently, one thread per virtual rank (gr_init_virtual:
    the ranks' collective calls must overlap, as N processes' would). Re-raises the first
    failure with its rank; returns the per-rank results."""
    import threading
    import traceback

    res, errs = [None] * N, [None] * N

    def body(r):
        try:
            res[r] = fn(r)
        except BaseException as e:  # noqa: BLE001 — reported below with the rank
            errs[r] = (e, traceback.format_exc())

    ths = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(N)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout)
    if any(t.is_alive() for t in ths):
        raise TimeoutError(f"virtual ranks still running after {timeout} s")
    for r, e in enumerate(errs):
        if e is not None:
            raise AssertionError(f"virtual rank {r}: {e[0]!r}\n{e[1]}")
    return res


def run_virtual_case(case, seed, device, buffer_f16: bool, grad_f16=None, kind="uniform", max_cycles=None,
                     exact: bool = True, async_streams=None, before_step=None, stats: bool = False,
                     drain_after=None, **world_kw):
    """One case on N = case.N virtual ranks of `device` (gr_init_virtual): every rank replays its
    schedule through the C ABI in its own thread and is checked against the oracle exactly as a
    process of a real N-GPU run is (run_case_on_rank / run_drain_case_on_rank); then the
    replicas must be bitwise identical. Returns the per-rank contexts' stats and logs."""
    from paper_1909_11150_b200 import GR_F16, GR_F32, virtual_world

    N = case.N
    ctxs = virtual_world(world_size=N, device=device.index or 0, numel=case.numel, group_of=case.group_of,
                         grad_f16=grad_f16, buffer_dtype=GR_F16 if buffer_f16 else GR_F32, **world_kw)
    try:
        if stats:
            for c in ctxs:
                c.gr_enable_grad_stats(True)

        def one(r):
            s = async_streams[r] if async_streams else None
            if drain_after is not None:
                log, h = run_drain_case_on_rank(ctxs[r], case, r, seed, device, buffer_f16, drain_after,
                                                async_stream=s)
            else:
                log, h = run_case_on_rank(ctxs[r], case, r, seed, device, buffer_f16, grad_f16, kind,
                                          max_cycles=max_cycles, async_stream=s, exact=exact,
                                          before_step=before_step[r] if before_step else None)
            ss = check_grad_stats(ctxs[r], case, seed, buffer_f16, grad_f16, kind, exact=exact,
                                  where=f"rank {r} seed {seed}") if stats else None
            return log, h, ss, ctxs[r].stats(), ctxs[r].query_int(5)

        out = run_ranks(N, one)
        hs = [o[1] for o in out]
        assert len(set(hs)) == 1, f"seed {seed}: outputs differ across virtual ranks"
        if stats:
            for o in out[1:]:  # fp64 atomics: equal up to summation order
                for a, b in zip(out[0][2], o[2]):
                    assert abs(a - b) <= 1e-12 * max(abs(a), abs(b)) + 1e-300, "statistics differ across ranks"
        return out
    finally:
        for c in ctxs:
            c.gr_finalize()
