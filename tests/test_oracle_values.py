"""Pins for the oracle's value half (readings R7-R11 in DESIGN.md §3).

* reduce_f64 against exact rational arithmetic (fractions.Fraction),
* the fp16 cast against numpy's IEEE binary16 conversion (a library routine),
* emulate's special cases: N=1 identity / plain fp16 cast, N=2 single
  rounding == fl32 of the exact mean, integer payloads exact for every order,
* the north-star tolerances (1e-6 relative for fp32, 2^-10*N*max|g| for fp16)
  hold for the emulated arithmetic against the fp64 reference,
* SPEC.md worked value vectors (tests/golden/spec_vectors.json).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from workloads.values import grad_values

HERE = os.path.dirname(os.path.abspath(__file__))


def test_round_f16_matches_numpy(orc):
    rng = np.random.default_rng(0)
    xs = np.concatenate([
        (rng.standard_normal(20000) * np.exp2(rng.uniform(-30, 18, 20000))).astype(np.float32),
        np.array([0.0, -0.0, 65504.0, 65519.996, 65520.0, -65520.0, 1e30, np.inf, -np.inf,
                  2.0 ** -24, 2.0 ** -25, 3 * 2.0 ** -26, 2.0 ** -14, 1.0 + 2.0 ** -11,
                  1.0 + 3 * 2.0 ** -11, 2049.0, 2051.0], dtype=np.float32),
    ])
    ours = np.array([orc.round_f16(float(x)) for x in xs], dtype=np.float32)
    ref = xs.astype(np.float16).astype(np.float32)
    assert np.array_equal(ours.view(np.uint32), ref.view(np.uint32))
    assert np.isnan(orc.round_f16(float("nan")))


@pytest.mark.parametrize("N", [1, 2, 3, 5, 8])
def test_reduce_f64_vs_exact_rationals(orc, N):
    rng = np.random.default_rng(N)
    gs = [(rng.standard_normal(300) * np.exp2(rng.uniform(-20, 20, 300))).astype(np.float32)
          for _ in range(N)]
    ref = orc.reduce_f64(gs)
    for i in range(300):
        exact = sum(Fraction(float(g[i])) for g in gs) / N
        scale = sum(abs(Fraction(float(g[i]))) for g in gs) / N
        assert abs(Fraction(float(ref[i])) - exact) <= scale * Fraction(N + 1, 2 ** 53)


def test_golden_value_vectors(orc):
    with open(os.path.join(HERE, "golden", "spec_vectors.json")) as f:
        gold = json.load(f)
    for case in gold["value_cases"]:
        gs = [np.array(x, dtype=np.float32) for x in case["g"]]
        want = np.array(case["expect_mean"], dtype=np.float32)
        assert np.array_equal(orc.reduce_f64(gs).astype(np.float32), want), case["id"]
        assert np.array_equal(orc.emulate(gs, False, False), want), case["id"]


def test_emulate_n1_identity_and_cast(orc):
    rng = np.random.default_rng(1)
    g = (rng.standard_normal(5000) * np.exp2(rng.uniform(-20, 15, 5000))).astype(np.float32)
    # V7: N=1, fp32 buffer: out == g bit for bit
    assert np.array_equal(orc.emulate([g], False, False).view(np.uint32), g.view(np.uint32))
    # V7: N=1, fp16 buffer: out == fl32(fl16(g)) (numpy's cast)
    want = g.astype(np.float16).astype(np.float32)
    assert np.array_equal(orc.emulate([g], True, False).view(np.uint32), want.view(np.uint32))
    assert np.array_equal(orc.emulate([g], True, True).view(np.uint32), want.view(np.uint32))


def test_emulate_n2_single_rounding(orc):
    """V8: at N=2 the fp64 sum of two floats is exact, so emu32 == fl32(exact mean)."""
    rng = np.random.default_rng(2)
    gs = [(rng.standard_normal(20000) * np.exp2(rng.uniform(-20, 20, 20000))).astype(np.float32)
          for _ in range(2)]
    emu = orc.emulate(gs, False, False)
    ref = orc.reduce_f64(gs).astype(np.float32)
    assert np.array_equal(emu.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("N", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("buf16,grad16", [(False, False), (True, False), (False, True), (True, True)])
def test_emulate_integer_payloads_exact(orc, N, buf16, grad16):
    """V9: |g| <= 16 integers: every partial sum is exact, so out == exact mean
    whenever the mean is representable (always for N in {1,2,4,8})."""
    gs = [grad_values([4096], N, seed=N, kind="int")[r][0] for r in range(N)]
    out = orc.emulate(gs, buf16, grad16)
    exact = [sum(Fraction(int(g[i])) for g in gs) / N for i in range(4096)]
    if N in (1, 2, 4, 8):
        assert all(Fraction(float(out[i])) == exact[i] for i in range(4096))
    # permutation of ranks does not change the result on integer payloads
    out_rev = orc.emulate(gs[::-1], buf16, grad16)
    assert np.array_equal(out, out_rev)


@pytest.mark.parametrize("N", [2, 4, 8])
def test_emulated_arithmetic_within_north_star_tolerance(orc, N):
    """The exact emulation of readings R7-R9 satisfies the north star's bounds (R10, R11)."""
    numel = [3000, 7, 1, 4096]
    gv = grad_values(numel, N, seed=11 + N)
    for t in range(len(numel)):
        gs = [gv[r][t] for r in range(N)]
        ref = orc.reduce_f64(gs)
        mean_abs = np.mean(np.abs(np.stack(gs).astype(np.float64)), axis=0)
        e32 = orc.emulate(gs, False, False).astype(np.float64)
        assert np.all(np.abs(e32 - ref) <= 1e-6 * np.maximum(np.abs(ref), mean_abs))
        maxg = float(np.max(np.abs(np.stack(gs))))
        e16 = orc.emulate(gs, True, False).astype(np.float64)
        assert np.all(np.abs(e16 - ref) <= 2.0 ** -10 * N * maxg)
        # the derived bound (input RN + output RN) is N times tighter
        assert np.all(np.abs(e16 - ref) <= 2.0 ** -10 * maxg)


# ---- hand-derived pins of emulate at N >= 3 and at the reading-R8 boundary -----------------

def _golden_emulate_cases():
    with open(os.path.join(HERE, "golden", "emulate_vectors.json")) as f:
        return json.load(f)["cases"]


def _f32(xs):
    return np.array([float(x) for x in xs], dtype=np.float32)


def _check_golden(emulate, case):
    gs = [_f32(g) for g in case["g"]]
    assert len(gs) == case["N"]
    out = emulate(gs, case["buffer_f16"], case["grad_f16"])
    want = _f32(case["expect"])
    nan = np.isnan(want)
    return bool(np.array_equal(np.isnan(out), nan) and
                np.array_equal(out[~nan].view(np.uint32), want[~nan].view(np.uint32)))


@pytest.mark.parametrize("case", _golden_emulate_cases(), ids=lambda c: c["id"])
def test_emulate_hand_derived_goldens(orc, case):
    """tests/golden/emulate_vectors.json: rank-order fp32 sums at N = 3 and 8, x fl32(1/N),
    the per-rank fp16 pack, scaling before the fp16 store (R8), fp16 subnormals, IEEE specials,
    cancellation — each value worked by hand from the arithmetic (bit-exact, sign of zero too)."""
    assert _check_golden(orc.emulate, case), case["id"]


# Each mutation is a plausible mistake in orc_emulate; the goldens above must catch every one
# (so the oracle's value arithmetic is pinned by something other than itself).
_MUTATIONS = {
    "fp64_accumulation": [("float acc = 0.0f;", "double acc = 0.0;")],
    "scale_after_fp16_store": [("float y = acc * inv_n;\n        if (buffer_f16) y = orc_round_f16(y);",
                                "float y = acc;\n        if (buffer_f16) y = orc_round_f16(y);\n        y = y * inv_n;")],
    "divide_by_n": [("float y = acc * inv_n;", "float y = acc / (float)N;")],
    "no_pack_rounding": [("float x = buffer_f16 ? orc_round_f16(g[r][i]) : g[r][i];", "float x = g[r][i];")],
    "reverse_rank_order": [("float x = buffer_f16 ? orc_round_f16(g[r][i]) : g[r][i];",
                            "float x = buffer_f16 ? orc_round_f16(g[N - 1 - r][i]) : g[N - 1 - r][i];")],
    "no_grad_cast": [("if (grad_f16) y = orc_round_f16(y);", "")],
}


@pytest.mark.parametrize("mutation", sorted(_MUTATIONS))
def test_goldens_catch_mutated_emulate(tmp_path, mutation):
    """Mutation check of the pins: orc_emulate rebuilt with one plausible mistake (fp64
    accumulation, scaling after the fp16 store, division by N, no per-rank fp16 pack, reversed
    rank order, no final gradient cast) fails at least one hand-derived golden."""
    import ctypes
    import subprocess
    src = open(os.path.join(os.path.dirname(HERE), "oracle", "gr_oracle.c")).read()
    for old, new in _MUTATIONS[mutation]:
        assert src.count(old) == 1, f"mutation {mutation}: pattern not found once"
        src = src.replace(old, new)
    c = tmp_path / "mut.c"
    c.write_text(src)
    so = tmp_path / "libmut.so"
    subprocess.run(["gcc", "-std=c11", "-O1", "-fno-fast-math", "-ffp-contract=off", "-shared", "-fPIC",
                    "-I", os.path.join(os.path.dirname(HERE), "oracle"), str(c), "-o", str(so)], check=True)
    L = ctypes.CDLL(str(so))
    L.orc_emulate.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                              ctypes.c_void_p]
    L.orc_emulate.restype = None

    def emulate(gs, b16, g16):
        arrs = [np.ascontiguousarray(g, dtype=np.float32) for g in gs]
        ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        out = np.zeros(arrs[0].size, dtype=np.float32)
        L.orc_emulate(len(arrs), arrs[0].size, ctypes.cast(ptrs, ctypes.c_void_p), int(b16), int(g16),
                      out.ctypes.data_as(ctypes.c_void_p))
        return out

    failed = [c["id"] for c in _golden_emulate_cases() if not _check_golden(emulate, c)]
    assert failed, f"no golden catches the mutation {mutation}"
