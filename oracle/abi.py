"""The §8(b) call contract (gr_init / gr_mark_ready / gr_step / gr_wait / gr_set_status) as a
plain, slow simulation of N ranks in one Python object — the oracle side of the ABI conformance
suite (tests/test_abi_conformance.py runs the same call scripts here and through libgr.so).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Shares no code, table or constant with the
product path: the status codes below are restated from SURVEY.md §8(b), not imported.

Every cycle is computed with the pinned primitives of gr_oracle.c, in the paper's order:
populate (§4.1 step 1) -> intersect (step 2) -> release
(PAPER.md:116 step 3 + PAPER.md:137 §4.2 Grouping); the values of a released group are
oracle.emulate over every rank's gradient (readings R7-R9) written into every rank's array in
place. The lifecycle / error rules are the contract's (SURVEY.md §8(b) "errors"
DuplicateSubmission -> GR_ESTATE, SPEC.md:221-222 ABORT/SHUTDOWN status -> GR_EABORT /
GR_ESHUTDOWN, readings R12-R15), each written as its own plain check below.
"""
from __future__ import annotations

import numpy as np

from . import bit_positions, emulate, intersect, populate, release, words

# status codes
OK, EINVAL, ESTATE, EMISMATCH, ECUDA, ETIMEOUT, EABORT, ESHUTDOWN, ENOMEM = 0, -1, -2, -3, -4, -5, -6, -7, -8
F32, F16 = 0, 1
MAX_RANKS = 8  # one NVSwitch domain


def validate_init(N: int, numel, grad_dtype, group_of, G: int, buffer_dtype: int) -> int:
    """gr_init's argument checks (SURVEY.md §8(b) GR_EINVAL: bad id, numel <= 0, group ids not
    dense or empty), in argument order."""
    T = len(numel)
    if not (1 <= N <= MAX_RANKS):
        return EINVAL
    if T <= 0 or G <= 0 or G > T:
        return EINVAL
    if buffer_dtype not in (F32, F16):
        return EINVAL
    members = [0] * G
    for t in range(T):
        if int(numel[t]) <= 0 or int(grad_dtype[t]) not in (F32, F16):
            return EINVAL
        g = int(group_of[t])
        if g < 0 or g >= G:
            return EINVAL
        members[g] += 1
    if any(m == 0 for m in members):
        return EINVAL
    return OK


class OracleWorld:
    """N simulated ranks sharing one table (a globally consistent cache)."""

    def __init__(self, N: int, numel, group_of, G: int, buffer_dtype: int = F16, grad_dtype=None):
        self.grad_dtype = [F32] * len(numel) if grad_dtype is None else [int(x) for x in grad_dtype]
        rc = validate_init(N, numel, self.grad_dtype, group_of, G, buffer_dtype)
        if rc:
            raise ValueError(rc)
        self.N, self.T, self.G = N, len(numel), G
        self.numel = [int(x) for x in numel]
        self.group_of = np.asarray(group_of, dtype=np.int32)
        self.buffer_f16 = buffer_dtype == F16
        self.bit_of = bit_positions(self.group_of)   # response cache, built once
        self.W = words(self.T)
        self.cycle = 0
        self.step = 0
        self.sticky = [0] * N                # per rank: sticky error code (0 = none)
        self.abort = [False] * N             # status flags raised by gr_set_status
        self.shutdown = [False] * N
        self._new_step()

    def _new_step(self):
        self.marked = np.zeros((self.N, self.T), dtype=np.uint8)
        self.arrays = [[None] * self.T for _ in range(self.N)]  # per rank: the caller's gradient
        self.group_released = np.zeros(self.G, dtype=np.uint8)
        self.step_complete = False

    # ---- gr_mark_ready (LOCAL): §4.1 step 1's pending request
    def mark(self, r: int, t: int, array) -> int:
        if self.sticky[r]:
            return ESTATE                      # any call after a sticky error
        if t < 0 or t >= self.T:
            return EINVAL                      # bad id
        if array is None:
            return EINVAL                      # null pointer
        if self.step_complete:
            return ESTATE                      # mark after the step completed, before gr_wait (R15)
        if self.marked[r, t]:
            return ESTATE                      # duplicate mark in a step (R15)
        self.marked[r, t] = 1
        self.arrays[r][t] = array
        return OK

    # ---- gr_set_status (LOCAL): reserved status bits (reading R1)
    def set_status(self, r: int, abort: bool, shutdown: bool) -> int:
        self.abort[r], self.shutdown[r] = bool(abort), bool(shutdown)
        return OK

    # ---- gr_step (COLLECTIVE): one cycle for every rank at once (reading R12)
    def step_all(self):
        """Returns per rank (code, released list, A or None, step_complete)."""
        out = [None] * self.N
        live = [r for r in range(self.N) if not self.sticky[r]]
        for r in range(self.N):
            if self.sticky[r]:
                out[r] = (ESTATE, [], None, False)
            elif self.step_complete:
                out[r] = (ESTATE, [], None, False)  # step complete: gr_wait first
        if any(o is not None for o in out):
            return out
        # step 1: each rank's local bitvector = its pending requests (marked and not released,
        # reading R4) plus its complement-coded status bits (reading R1)
        released_t = self.group_released[self.group_of].astype(bool)
        Ls = [populate(self.bit_of, (self.marked[r].astype(bool) & ~released_t).astype(np.uint8),
                       self.abort[r], self.shutdown[r]) for r in live]
        A = intersect(Ls)                      # step 2: bitwise AND over ranks
        self.cycle += 1
        if not (A[0] & 1):                     # some rank raised ABORT: nothing released (R13)
            for r in range(self.N):
                self.sticky[r] = EABORT
            return [(EABORT, [], A.copy(), False) for _ in range(self.N)]
        if not (A[0] & 2):                     # some rank raised SHUTDOWN (R13)
            for r in range(self.N):
                self.sticky[r] = ESHUTDOWN
            return [(ESHUTDOWN, [], A.copy(), False) for _ in range(self.N)]
        rel = release(self.group_of, self.bit_of, A, self.group_released)  # step 3 + §4.2
        for g in rel:                          # values of the released groups, every rank
            for t in np.nonzero(self.group_of == g)[0]:
                gs = [np.asarray(self.arrays[r][t], dtype=np.float32).reshape(-1) for r in range(self.N)]
                y = emulate(gs, self.buffer_f16, self.grad_dtype[t] == F16)
                for r in range(self.N):
                    a = self.arrays[r][t]
                    a[...] = y.reshape(a.shape).astype(a.dtype)
        self.step_complete = bool(np.all(self.group_released))
        return [(OK, list(rel), A.copy(), self.step_complete) for _ in range(self.N)]

    # ---- gr_wait (LOCAL): if the step is complete, start the next (marks cleared)
    def wait(self, r: int) -> int:
        return OK

    def wait_all(self):
        if self.step_complete:
            self.step += 1
            self._new_step()
        return [OK] * self.N
