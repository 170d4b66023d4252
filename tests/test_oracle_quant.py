"""Pins for oracle O1-O3 (quantizers) and the fp16 / rounding helpers.  CPU only."""

import itertools

import numpy as np
import pytest

from oracle import (
    dequantize_base,
    dequantize_residual_rows,
    fp16_rne,
    quantize_base,
    quantize_residual,
    residual,
    round_half_away,
)
from synth import gen_weight_fp16


def test_fp16_rne_ties_to_even():
    # 1 + 2^-11 is halfway between 1 and 1 + 2^-10 -> even (1.0); 1 + 3*2^-11 -> 1 + 2^-9
    assert fp16_rne(1 + 2.0 ** -11) == 1.0
    assert fp16_rne(1 + 3 * 2.0 ** -11) == 1 + 2.0 ** -9
    assert fp16_rne(65519.0) == 65504.0
    assert fp16_rne(2.0 ** -25) == 0.0          # halfway to the smallest subnormal -> even (0)
    assert fp16_rne(3 * 2.0 ** -25) == 2.0 ** -23


def test_round_half_away():
    v = np.array([0.5, -0.5, 1.5, -1.5, 2.5, 0.49999999999999994, -2.4999, 0.0])
    assert list(round_half_away(v)) == [1, -1, 2, -2, 3, 0, -2, 0]


@pytest.mark.parametrize("name", ["base_quant_group.txt", "base_quant_group4.txt"])
def test_base_quant_hand_worked(golden, name):
    lines = golden(name)
    bits = int(lines[0].split()[1])
    s_exp = float(lines[1].split()[1])
    z_exp = int(lines[2].split()[1])
    rows = [tuple(p.strip() for p in ln.split(";")) for ln in lines[3:]]
    col = np.zeros(128)
    for i, (v, _, _) in enumerate(rows):
        col[i] = float(v)
    W = col.astype(np.float16)[:, None]
    q, s, z = quantize_base(W, bits)
    assert float(s[0, 0]) == s_exp and int(z[0, 0]) == z_exp
    Wh = dequantize_base(q, s, z)
    for i, (_, qe, we) in enumerate(rows):
        assert int(q[i, 0]) == int(qe), (i, rows[i])
        assert Wh[i, 0] == float(we), (i, rows[i])


def test_base_zero_fixed_point():
    W = np.zeros((256, 8), np.float16)
    for bits in (3, 4):
        q, s, z = quantize_base(W, bits)
        assert np.all(dequantize_base(q, s, z) == 0.0)
        assert np.all(residual(W, dequantize_base(q, s, z)) == 0.0)


@pytest.mark.parametrize("bits", [3, 4])
def test_base_exact_grid_idempotent(bits):
    # integer weights in [0, 2^b-1] with 0 and max present in every group -> s = 1, z = 0, R = 0
    rng = np.random.default_rng(1)
    qmax = (1 << bits) - 1
    W = rng.integers(0, qmax + 1, size=(256, 16)).astype(np.float64)
    W[0::128, :] = 0
    W[1::128, :] = qmax
    W16 = W.astype(np.float16)
    q, s, z = quantize_base(W16, bits)
    assert np.all(s == 1.0) and np.all(z == 0)
    assert np.all(residual(W16, dequantize_base(q, s, z)) == 0.0)
    # scaled grid: W = 0.125 * (k - 3) is also exact (s = 0.125, z = 3)
    W2 = (0.125 * (W - 3)).astype(np.float16)
    q2, s2, z2 = quantize_base(W2, bits)
    Wh2 = dequantize_base(q2, s2, z2)
    assert np.all(Wh2 == W2.astype(np.float64))
    # idempotence: quantize(W_hat) == W_hat when codes span the full range
    q3, s3, z3 = quantize_base(Wh2.astype(np.float16), bits)
    assert np.all(dequantize_base(q3, s3, z3) == Wh2)


@pytest.mark.parametrize("bits", [3, 4])
def test_base_rtn_bound(bits):
    W = gen_weight_fp16(512, 64, seed=7)
    q, s, z = quantize_base(W, bits)
    Wh = dequantize_base(q, s, z)
    R = residual(W, Wh)
    s_rows = np.repeat(s.astype(np.float64), 128, axis=0)
    # RTN: |R| <= s/2 except where the code clipped (only possible at the range ends by <= s)
    qmax = (1 << bits) - 1
    interior = (q > 0) & (q < qmax)
    assert np.all(np.abs(R[interior]) <= s_rows[interior] / 2 + 1e-12)
    assert np.all(np.abs(R) <= s_rows + 1e-12)
    # W_hat lies on the grid s * integer
    assert np.all(np.abs(Wh / s_rows - np.rint(Wh / s_rows)) < 1e-9)
    assert q.max() <= qmax


def test_residual_worked_example(golden):
    lines = dict((ln.split()[0], ln.split()[1:]) for ln in golden("residual_example.txt"))
    s = float(lines["s"][0])
    vals = np.array([float(v) for v in lines["values"]])
    codes_at_s = np.array([int(c) for c in lines["codes_at_s"]])
    mse_at_s = float(lines["mse_at_s"][0])
    assert np.array_equal(np.clip(round_half_away(vals / s), -7, 7), codes_at_s)
    assert abs(np.mean((vals - s * codes_at_s) ** 2) - mse_at_s) < 1e-15
    c, S = quantize_residual(vals[:, None], 4)
    mse = np.mean((vals - float(S[0]) * c[:, 0]) ** 2)
    assert mse <= mse_at_s + 1e-15
    assert np.all(np.abs(c) <= 7)


def _scalar_grid_search(col):
    """Independent scalar-loop restatement of the S:83 grid (brute-force argmin)."""
    m = max(abs(float(v)) for v in col)
    if m == 0:
        return 1.0, [0] * len(col)
    best = None
    for t in range(128):
        g = 0.30 + 0.70 * t / 127.0
        St = float(np.float16(m * g / 7.0))
        if St == 0:
            continue
        cs = []
        e = 0.0
        for v in col:
            r = float(v) / St
            a = abs(r)
            n = int(a) + (1 if a - int(a) >= 0.5 else 0)
            n = min(n, 7)
            c = n if r >= 0 else -n
            cs.append(c)
            e += (float(v) - St * c) ** 2
        if best is None or e <= best[0]:  # ascending t, '<=' -> ties to the larger t
            best = (e, St, cs)
    return best[1], best[2]


def test_residual_grid_bruteforce():
    rng = np.random.default_rng(3)
    R = rng.standard_normal((64, 12)) * rng.lognormal(0, 1, size=12)[None, :] * 1e-3
    R[:, 3] = 0.0
    c, S = quantize_residual(R, 4)
    for j in range(R.shape[1]):
        Sj, cj = _scalar_grid_search(R[:, j])
        assert float(S[j]) == Sj, j
        assert list(c[:, j]) == cj, j
    assert np.all(np.abs(c) <= 7)
    assert float(S[3]) == 1.0 and np.all(c[:, 3] == 0)


def test_residual_beats_naive_scale():
    rng = np.random.default_rng(5)
    for seed in range(5):
        r = np.random.default_rng(seed).standard_normal((4096, 1))
        c, S = quantize_residual(r, 4)
        mse = np.mean((r[:, 0] - float(S[0]) * c[:, 0]) ** 2)
        naive = float(np.float16(np.abs(r).max() / 7))
        cn = np.clip(round_half_away(r[:, 0] / naive), -7, 7)
        assert mse <= np.mean((r[:, 0] - naive * cn) ** 2)
    del rng


def test_residual16_roundtrip_and_rows():
    rng = np.random.default_rng(9)
    R = (rng.standard_normal((32, 16)) * 1e-2).astype(np.float16).astype(np.float64)
    assert np.array_equal(quantize_residual(R, 16).astype(np.float64), R)
    c, S = quantize_residual(R, 4)
    rows = [5, 0, 31]
    D = dequantize_residual_rows(c, S, rows)
    for a, i in enumerate(rows):
        assert np.array_equal(D[a], S.astype(np.float64) * c[i].astype(np.float64))
    assert dequantize_residual_rows(c, S, []).shape == (0, 16)


def test_residual_grid_exhaustive_small():
    # every 3-vector over a small lattice: chosen S is the grid argmin with ties -> larger t
    vals = [-0.3, -0.1, 0.0, 0.05, 0.2, 0.35]
    for trip in itertools.islice(itertools.product(vals, repeat=3), 0, None, 7):
        col = np.array(trip)
        c, S = quantize_residual(col[:, None], 4)
        Sj, cj = _scalar_grid_search(col)
        assert float(S[0]) == Sj and list(c[:, 0]) == cj
