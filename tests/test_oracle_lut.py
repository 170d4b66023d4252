"""Pins of the non-uniform (LUT) base quantizer O1-LUT (the paper's
SqueezeLLM base, P:397 / P:502, ledger L17) and of O5 on LUT weights."""

import numpy as np
import pytest

import oracle
from oracle import decdec_linear_ref, dequantize_lut, quantize_base_lut, residual, tolerance_ok


def _floats(s):
    return [float(t) for t in s.split()]


def test_lut_hand_worked_columns(golden):
    for ln in golden("lut_kmeans.txt"):
        b, vals, lut, codes = (p.strip() for p in ln.split(";"))
        v = np.array(_floats(vals), dtype=np.float16)[:, None]
        q, L = quantize_base_lut(v, int(b))
        assert L[:, 0].astype(np.float64).tolist() == _floats(lut), ln
        assert q[:, 0].tolist() == [int(c) for c in codes.split()], ln


@pytest.mark.parametrize("bits", [3, 4])
def test_lut_exact_when_column_has_2b_equal_runs(bits):
    """2^b distinct fp16 values per column, each 128/2^b... times: the table reproduces them and
    R = W - W_hat = 0, so O5 gives y = W x for every k (numpy matmul of the original W)."""
    n = 1 << bits
    rng = np.random.default_rng(bits)
    d_in, d_out = 128, 24
    W = np.zeros((d_in, d_out), np.float16)
    for j in range(d_out):
        vals = np.sort(rng.choice(np.arange(-200, 200), size=n, replace=False)).astype(np.float64) / 64.0
        col = np.repeat(vals, d_in // n)
        W[:, j] = rng.permutation(col).astype(np.float16)
    q, L = quantize_base_lut(W, bits)
    assert np.array_equal(dequantize_lut(q, L), W.astype(np.float64))
    R = residual(W, dequantize_lut(q, L))
    assert np.all(R == 0)
    x = rng.standard_normal(d_in).astype(np.float16)
    for k in (0, 7, d_in):
        out = decdec_linear_ref(q, None, None, x, k, rc=np.zeros((d_in, d_out), np.int8), rS=np.ones(d_out, np.float16),
                                lut=L)
        Wx = x.astype(np.float64) @ W.astype(np.float64)
        assert np.allclose(out["y64"], Wx, rtol=0, atol=1e-12)


def test_lut_codes_are_nearest_entry_bruteforce():
    rng = np.random.default_rng(3)
    W = (rng.standard_normal((96, 7)) * 0.02).astype(np.float16)
    q, L = quantize_base_lut(W, 3)
    Wd = W.astype(np.float64)
    Ld = L.astype(np.float64)
    for j in range(W.shape[1]):
        for i in range(W.shape[0]):
            d = [abs(Wd[i, j] - Ld[c, j]) for c in range(8)]
            best = min(d)
            assert q[i, j] == d.index(best)  # nearest, lowest code on ties
    assert np.all(np.diff(Ld, axis=0) >= 0)  # quantile init + 1-D Lloyd keep the order


def test_lut_lloyd_mse_non_increasing():
    rng = np.random.default_rng(4)
    W = (rng.standard_normal((256, 5)) * np.exp(rng.standard_normal(5))[None, :]).astype(np.float16)
    prev = None
    for it in (0, 1, 2, 4, 8, 16):
        q, L = quantize_base_lut(W, 3, iters=it)
        # MSE of the (unrounded-then-fp16) table is not strictly monotone because of fp16
        # rounding; compare with a slack of one fp16 ulp of the column scale
        mse = ((dequantize_lut(q, L) - W.astype(np.float64)) ** 2).mean(axis=0)
        if prev is not None:
            assert np.all(mse <= prev * (1 + 1e-3) + 1e-9), it
        prev = mse


def test_lut_beats_uniform_rtn_on_heavy_tails():
    """Sanity (not a theorem): on heavy-tailed columns the k-means table has lower MSE than a
    uniform RTN grid of the same bit width over the whole column."""
    rng = np.random.default_rng(5)
    W = (rng.standard_t(3, size=(512, 6)) * 0.01).astype(np.float16)
    q, L = quantize_base_lut(W, 3)
    mse_lut = ((dequantize_lut(q, L) - W.astype(np.float64)) ** 2).mean()
    qu, su, zu = oracle.quantize_base(W, 3, group=512)
    mse_rtn = ((oracle.dequantize_base(qu, su, zu, group=512) - W.astype(np.float64)) ** 2).mean()
    assert mse_lut < mse_rtn


def test_lut_linear_matches_definition_small():
    """O5 with a LUT: y = sum_i lut[q_ij, j] x_i + sum_{i in S} x_i R_hat_ij, brute force loops."""
    rng = np.random.default_rng(6)
    d_in, d_out, k = 32, 5, 4
    q = rng.integers(0, 8, size=(d_in, d_out)).astype(np.uint8)
    L = np.sort(rng.standard_normal((8, d_out)), axis=0).astype(np.float16)
    rc = rng.integers(-7, 8, size=(d_in, d_out)).astype(np.int8)
    rS = (rng.random(d_out) * 0.01).astype(np.float16)
    x = rng.standard_normal(d_in).astype(np.float16)
    out = decdec_linear_ref(q, None, None, x, k, rc=rc, rS=rS, lut=L)
    sel = set(np.argsort(-np.abs(x.astype(np.float64)), kind="stable")[:k].tolist())
    for j in range(d_out):
        acc = 0.0
        for i in range(d_in):
            acc += float(L[q[i, j], j]) * float(x[i])
            if i in sel:
                acc += float(x[i]) * float(rS[j]) * float(rc[i, j])
        assert abs(acc - out["y64"][j]) <= 1e-12 * max(1.0, abs(acc))
    ok, _, _ = tolerance_ok(out["y16"], out["y64"], out["A"])
    assert ok.all()
