"""CPU oracle for arXiv 1909.11150 §4.1-4.2 (Bitvector Allreduce + Grouping) and
the reduced gradient values — ctypes wrapper over ``oracle/gr_oracle.c``.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package. It shares no code with the product path (``include/gr.h``,
``paper_1909_11150_b200/``) and the product path never imports it.

Every function follows a passage of PAPER.md, cited in ``gr_oracle.h``; the
readings of silent passages (R1..R14) are listed in DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

STATUS_BITS = 2  # PAPER.md:130 "an initial set of bits ... reserved" (reading R1)


def lib():
    global _LIB
    if _LIB is None:
        path = _build.build()
        L = ctypes.CDLL(path)
        i32, i64, p = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
        L.orc_words.argtypes = [i32]
        L.orc_words.restype = i32
        L.orc_bit_positions.argtypes = [i32, p, i32, p]
        L.orc_bit_positions.restype = ctypes.c_int
        L.orc_populate.argtypes = [i32, i32, p, p, ctypes.c_int, ctypes.c_int, p]
        L.orc_populate.restype = None
        L.orc_intersect.argtypes = [i32, i32, p, p]
        L.orc_intersect.restype = None
        L.orc_release.argtypes = [i32, i32, p, p, p, p, p]
        L.orc_release.restype = i32
        L.orc_simulate_step.argtypes = [i32, i32, i32, p, p, p, i32, p, p, p, p, p]
        L.orc_simulate_step.restype = ctypes.c_int
        L.orc_reduce_f64.argtypes = [i32, i64, p, p]
        L.orc_reduce_f64.restype = None
        L.orc_emulate.argtypes = [i32, i64, p, ctypes.c_int, ctypes.c_int, p]
        L.orc_emulate.restype = None
        L.orc_round_f16.argtypes = [ctypes.c_float]
        L.orc_round_f16.restype = ctypes.c_float
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def words(T: int) -> int:
    """W = ceil((T+2)/32) u32 words (reading R2)."""
    return int(lib().orc_words(T))


def bit_positions(group_of) -> np.ndarray:
    """Cache bit of each tensor, group-major (reading R3)."""
    g = np.ascontiguousarray(group_of, dtype=np.int32)
    G = int(g.max()) + 1 if g.size else 0
    out = np.zeros(g.size, dtype=np.int32)
    if lib().orc_bit_positions(g.size, _ptr(g), G, _ptr(out)) != 0:
        raise ValueError("group_of must be dense 0..G-1 with non-empty groups")
    return out


def populate(bit_of, pending, abort=False, shutdown=False) -> np.ndarray:
    """§4.1 step 1."""
    b = np.ascontiguousarray(bit_of, dtype=np.int32)
    pe = np.ascontiguousarray(pending, dtype=np.uint8)
    W = words(b.size)
    L = np.zeros(W, dtype=np.uint32)
    lib().orc_populate(b.size, W, _ptr(b), _ptr(pe), int(abort), int(shutdown), _ptr(L))
    return L


def intersect(Ls) -> np.ndarray:
    """§4.1 step 2: bitwise AND over ranks."""
    L = np.ascontiguousarray(np.stack(Ls), dtype=np.uint32)
    N, W = L.shape
    A = np.zeros(W, dtype=np.uint32)
    lib().orc_intersect(N, W, _ptr(L), _ptr(A))
    return A


def release(group_of, bit_of, A, group_released):
    """§4.1 step 3 + §4.2 rule. Mutates group_released."""
    g = np.ascontiguousarray(group_of, dtype=np.int32)
    b = np.ascontiguousarray(bit_of, dtype=np.int32)
    A = np.ascontiguousarray(A, dtype=np.uint32)
    assert group_released.dtype == np.uint8 and group_released.flags.c_contiguous
    G = group_released.size
    out = np.zeros(G, dtype=np.int32)
    n = lib().orc_release(g.size, G, _ptr(g), _ptr(b), _ptr(A), _ptr(group_released), _ptr(out))
    return [int(x) for x in out[:n]]


@dataclass
class StepResult:
    rc: int                      # 0 complete, 1 status-bit abort, 2 cycle bound hit
    A: np.ndarray                # [n_cycles, W] uint32 intersected bitvectors
    released: list               # per cycle: list of group ids (ascending)
    rel_cycle: np.ndarray        # [G] cycle of release, -1 if never
    n_cycles: int


def simulate_step(N: int, group_of, mark_cycle, status=None, max_cycles: int = 1000) -> StepResult:
    """One training step of N simulated ranks.

    mark_cycle[r, t] = cycles rank r completes before marking tensor t (-1: never)."""
    g = np.ascontiguousarray(group_of, dtype=np.int32)
    T = g.size
    G = int(g.max()) + 1
    m = np.ascontiguousarray(mark_cycle, dtype=np.int32).reshape(N, T)
    W = words(T)
    A = np.zeros((max_cycles, W), dtype=np.uint32)
    nrel = np.zeros(max_cycles, dtype=np.int32)
    rel = np.zeros((max_cycles, G), dtype=np.int32)
    relc = np.zeros(G, dtype=np.int32)
    nc = ctypes.c_int32(0)
    st_ptr = None
    if status is not None:
        st = np.ascontiguousarray(status, dtype=np.uint8).reshape(N, max_cycles)
        st_ptr = _ptr(st)
    rc = lib().orc_simulate_step(N, T, G, _ptr(g), _ptr(m), st_ptr, max_cycles, _ptr(A),
                                 _ptr(nrel), _ptr(rel), _ptr(relc), ctypes.byref(nc))
    if rc < 0:
        raise ValueError("bad input to orc_simulate_step")
    n = nc.value
    return StepResult(rc, A[:n].copy(), [[int(x) for x in rel[c, :nrel[c]]] for c in range(n)],
                      relc, n)


def _ptr_array(gs):
    arrs = [np.ascontiguousarray(x, dtype=np.float32) for x in gs]
    ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    return arrs, ptrs


def reduce_f64(gs) -> np.ndarray:
    """Reference value (1/N)·Σ_r g_r in fp64 (reading R7)."""
    arrs, ptrs = _ptr_array(gs)
    n = arrs[0].size
    ref = np.zeros(n, dtype=np.float64)
    lib().orc_reduce_f64(len(arrs), n, ptrs, _ptr(ref))
    return ref


def emulate(gs, buffer_f16: bool, grad_f16: bool) -> np.ndarray:
    """Exact arithmetic of readings R7-R9 (fp32 rank-order sum, ×fl32(1/N))."""
    arrs, ptrs = _ptr_array(gs)
    n = arrs[0].size
    out = np.zeros(n, dtype=np.float32)
    lib().orc_emulate(len(arrs), n, ptrs, int(buffer_f16), int(grad_f16), _ptr(out))
    return out


def round_f16(x: float) -> float:
    return float(lib().orc_round_f16(x))
