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
