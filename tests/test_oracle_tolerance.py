"""Pins of the L9 checker every GPU parity assertion goes through (oracle.tolerance_ok) and of
the unfloored relative-error report (oracle.rel_err_unfloored).

Ledger L9 (BASELINE.json "max relative error 1e-3 per element", undefined at y ~ 0):
    |y16 - y*| <= 1e-3 * max(|y*|, 2^-12 * A_j, 2^-14)
Every case below is constructed by hand so that the error sits 1 % above or below the bound
of exactly one branch; a sign, exponent or branch slip in tolerance_ok flips one of them."""

import numpy as np
import pytest

from oracle import rel_err_unfloored, tolerance_ok


def _pair_at(y16_val, rel):
    """y* such that |fp16(y16_val) - y*| = rel * |y*| (y* between 0 and y16)."""
    y = float(np.float16(y16_val))
    return y / (1.0 + rel)


@pytest.mark.parametrize("y16_val", [1.0, -3.5, 1234.0, 0.0625, -60000.0])
def test_relative_branch_accepts_099_rejects_101(y16_val):
    y16 = np.array([y16_val, y16_val], dtype=np.float16)
    y64 = np.array([_pair_at(y16_val, 0.99e-3), _pair_at(y16_val, 1.01e-3)])
    A = np.zeros(2)  # floors inactive: 2^-12 * 0 and 2^-14 << 1e-3 |y*| here
    ok, err, bound = tolerance_ok(y16, y64, A)
    assert ok.tolist() == [True, False]
    assert np.allclose(err / np.abs(y64), [0.99e-3, 1.01e-3], rtol=1e-9)
    assert np.allclose(bound, 1e-3 * np.abs(y64), rtol=0)


def test_A_floor_engages_only_where_it_dominates():
    # y* = 0 (cancellation): bound = 1e-3 * 2^-12 * A.  y16 = 2^-10 exactly representable.
    y16v = 2.0 ** -10
    A_exact = y16v / (1e-3 * 2.0 ** -12)          # bound == |y16 - 0| exactly
    y16 = np.full(3, y16v, dtype=np.float16)
    y64 = np.zeros(3)
    A = np.array([A_exact * 1.01, A_exact * 0.99, A_exact])
    ok, err, bound = tolerance_ok(y16, y64, A)
    assert ok.tolist() == [True, False, True]     # '<=' at equality
    assert np.allclose(bound, 1e-3 * 2.0 ** -12 * A)
    # the same A does not loosen an output whose |y*| dominates 2^-12 A
    big = 4.0
    ok2, _, b2 = tolerance_ok(np.array([big], np.float16), np.array([_pair_at(big, 1.01e-3)]),
                              np.array([big * 2.0 ** 12 * 0.5]))
    assert not ok2[0] and np.isclose(b2[0], 1e-3 * _pair_at(big, 1.01e-3))


def test_absolute_floor_2pow_minus14():
    # y* = 0 and A = 0: bound = 1e-3 * 2^-14 = 6.10e-8.  fp16 subnormals 2^-24 (5.96e-8) and
    # 2^-23 (1.19e-7) straddle it.
    y16 = np.array([2.0 ** -24, 2.0 ** -23, 0.0], dtype=np.float16)
    ok, err, bound = tolerance_ok(y16, np.zeros(3), np.zeros(3))
    assert ok.tolist() == [True, False, True]
    assert np.allclose(bound, 1e-3 * 2.0 ** -14)


def test_sign_flip_and_fp16_rounding_of_input():
    ok, _, _ = tolerance_ok(np.array([-1.0], np.float16), np.array([1.0]), np.array([1.0]))
    assert not ok[0]
    # y16 is interpreted as fp16: a float64 value is rounded before comparing (1 + 2^-12 -> 1.0)
    ok, err, _ = tolerance_ok(np.array([1.0 + 2.0 ** -12]), np.array([1.0]), np.zeros(1))
    assert ok[0] and err[0] == 0.0


def test_fp16_output_rounding_alone_fits():
    # the L9 note: fp16 RN of an exact y* contributes <= 2^-11 relative (< 1e-3)
    rng = np.random.default_rng(0)
    # magnitudes inside fp16's normal range [2^-14, 65504)
    y64 = rng.choice([-1.0, 1.0], 10000) * np.exp2(rng.uniform(-12, 15, 10000))
    ok, err, _ = tolerance_ok(y64.astype(np.float16), y64, np.abs(y64))
    assert ok.all() and np.max(err / np.abs(y64)) <= 2.0 ** -11 * (1 + 1e-12)


def test_rel_err_unfloored():
    y64 = np.array([10.0, -10.0, 1e-3, 0.0])           # rms = 7.07 -> threshold 0.0707
    y16 = np.array([10.0 * (1 + 2.0 ** -10), -10.0, 5.0, 3.0], dtype=np.float16)
    r, n = rel_err_unfloored(y16, y64)
    assert n == 2                                        # the near-zero outputs are excluded
    assert r == pytest.approx(float(np.float16(10.0 * (1 + 2.0 ** -10))) / 10.0 - 1.0)
    assert rel_err_unfloored(np.zeros(0, np.float16), np.zeros(0)) == (0.0, 0)
