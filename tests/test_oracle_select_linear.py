"""Pins for oracle O4 (exact Top-K), O5 (decdec_linear_ref) and O6 (packing).  CPU only."""

import itertools

import numpy as np
import pytest

import oracle
from oracle import (
    decdec_linear_ref,
    dequantize_base,
    k_from_kchunk,
    quantize_base,
    quantize_residual,
    residual,
    tolerance_ok,
    topk_ref,
)
from synth import gen_activations, gen_perf_layer, gen_special_activations, gen_weight_fp16


# ----------------------------------------------------------------------------- O4
def test_topk_spec_examples(golden):
    for ln in golden("topk_examples.txt"):
        xs, k, exp = (p.strip() for p in ln.split(";"))
        x = np.array([float(v) for v in xs.split()], np.float16)
        idx, vals = topk_ref(x, int(k))
        assert list(idx) == [int(e) for e in exp.split()]
        assert np.array_equal(vals, x[idx])


def _dominates(x16, S):
    """Definition of the selected set: every selected i beats every unselected j."""
    key = (x16.view(np.uint16) & 0x7FFF).astype(int)
    Sset = set(S)
    for i in S:
        for j in range(len(x16)):
            if j in Sset:
                continue
            if not (key[i] > key[j] or (key[i] == key[j] and i < j)):
                return False
    return True


def test_topk_bruteforce_small():
    rng = np.random.default_rng(0)
    for trial in range(60):
        n = int(rng.integers(1, 13))
        pool = [0.0, -0.0, 1.0, -1.0, 2.0, -2.0, 0.5, 3.0, -7.0]
        x = np.array(rng.choice(pool, size=n), np.float16) if trial % 2 else rng.standard_normal(n).astype(np.float16)
        for k in range(0, n + 1):
            winners = [S for S in itertools.combinations(range(n), k) if _dominates(x, S)]
            assert len(winners) == 1, (x, k, winners)   # the definition has a unique solution
            idx, _ = topk_ref(x, k)
            assert tuple(idx) == winners[0]


def test_topk_threshold_property_large():
    x = gen_activations(14336, 1, seed=11, kind="down")[0]
    key = (x.view(np.uint16) & 0x7FFF).astype(int)
    for k in (1, 7, 358, 1433, 14336):
        idx, _ = topk_ref(x, k)
        assert len(idx) == k and np.all(np.diff(idx) > 0)
        sel = np.zeros(len(x), bool)
        sel[idx] = True
        if k < len(x):
            T = key[sel].min()
            assert key[~sel].max() <= T
            # ties at the threshold: selected ones precede unselected ones in index order
            tie_sel = np.nonzero(sel & (key == T))[0]
            tie_un = np.nonzero(~sel & (key == T))[0]
            if len(tie_un):
                assert tie_sel.max() < tie_un.min()


def test_topk_signed_zero_and_ties():
    x = gen_special_activations(64, "zeros")
    idx, _ = topk_ref(x, 10)
    assert list(idx) == list(range(10))                 # +0 and -0 tie -> lowest indices
    x = gen_special_activations(256, "all_equal")
    assert list(topk_ref(x, 17)[0]) == list(range(17))


def test_topk_chunk_mode_paper_example(golden):
    rows = {ln.split()[0]: ln.split()[1:] for ln in golden("paper_accounting.txt")}
    d_in, k, kc = (int(v) for v in rows["chunk_example"])
    x = gen_activations(d_in, 1, seed=5)[0]
    idx, _ = topk_ref(x, kc, chunk=1024)
    assert len(idx) == k
    for c in range(d_in // 1024):
        seg = idx[(idx >= 1024 * c) & (idx < 1024 * (c + 1))]
        assert len(seg) == kc
        assert np.array_equal(seg, topk_ref(x[1024 * c:1024 * (c + 1)], kc)[0] + 1024 * c)
    # short last chunk: d_in = 17920 = 17.5 chunks, quota min(k_chunk, len)
    x = gen_activations(17920, 1, seed=6)[0]
    idx, _ = topk_ref(x, 600, chunk=1024)
    assert len(idx) == 17 * 600 + 512


def test_paper_accounting(golden):
    rows = [ln.split() for ln in golden("paper_accounting.txt")]
    for r in rows:
        if r[0] == "kchunk_fraction_dinp":
            frac, d_in, k = float(r[1]), int(r[2]), int(r[3])
            assert int(frac * d_in) == k   # L3: floor
        if r[0] == "chunk_example":
            assert k_from_kchunk(int(r[3]), int(r[1])) == int(r[2])
        if r[0] == "buffer_bytes":
            assert int(r[1]) * (4 + 2) == int(r[2])


# ----------------------------------------------------------------------------- O5
def _small_layer(bits=3, d_in=512, d_out=64, seed=1):
    W = gen_weight_fp16(d_in, d_out, seed)
    q, s, z = quantize_base(W, bits)
    R = residual(W, dequantize_base(q, s, z))
    rc, rS = quantize_residual(R, 4)
    r16 = quantize_residual(R, 16)
    return W, q, s, z, rc, rS, r16


def test_linear_exact_weights_equal_Wx():
    # R = 0 -> y = W x for every k (independent numpy matmul of the original W)
    rng = np.random.default_rng(2)
    W = (0.125 * (rng.integers(0, 8, size=(256, 48)) - 3)).astype(np.float16)
    W[0::128] = (0.125 * -3)
    W[1::128] = (0.125 * 4)
    q, s, z = quantize_base(W, 3)
    R = residual(W, dequantize_base(q, s, z))
    assert np.all(R == 0)
    rc, rS = quantize_residual(R, 4)
    x = gen_activations(256, 1, seed=3)[0]
    Wx = x.astype(np.float64) @ W.astype(np.float64)
    for k in (0, 5, 256):
        out = decdec_linear_ref(q, s, z, x, k, rc=rc, rS=rS)
        assert np.allclose(out["y64"], Wx, rtol=0, atol=1e-12 * np.abs(Wx).max())


def test_linear_full_fp16_compensation_recovers_Wx():
    W, q, s, z, rc, rS, r16 = _small_layer()
    x = gen_activations(512, 1, seed=4)[0]
    Wx = x.astype(np.float64) @ W.astype(np.float64)
    out = decdec_linear_ref(q, s, z, x, 512, r16=r16)
    A = np.abs(x.astype(np.float64)) @ np.abs(W.astype(np.float64))
    ok, err, bound = tolerance_ok(out["y16"], Wx, A)
    assert ok.all()
    # and k = 0 is strictly the quantized result (differs from W x)
    out0 = decdec_linear_ref(q, s, z, x, 0, r16=r16)
    assert np.array_equal(out0["y64"], out0["ob"]) and not np.allclose(out0["y64"], Wx)


def test_linear_single_channel_and_empty():
    W, q, s, z, rc, rS, r16 = _small_layer()
    i = 37
    x = np.zeros(512, np.float16)
    x[i] = 2.0
    out = decdec_linear_ref(q, s, z, x, 1, rc=rc, rS=rS)
    assert list(out["idx"]) == [i]
    assert np.array_equal(out["odec"], 2.0 * rS.astype(np.float64) * rc[i].astype(np.float64))
    # o_b picks row i of W_hat: catches a transposed operand
    assert np.array_equal(out["ob"], 2.0 * dequantize_base(q, s, z)[i])
    out0 = decdec_linear_ref(q, s, z, x, 0, rc=rc, rS=rS)
    assert np.all(out0["odec"] == 0) and len(out0["idx"]) == 0


def test_linear_linearity_disjoint():
    W, q, s, z, rc, rS, r16 = _small_layer()
    x = gen_activations(512, 1, seed=8)[0]
    full = decdec_linear_ref(q, s, z, x, 40, rc=rc, rS=rS)
    idx = full["idx"]
    # split the selection into two disjoint halves by zeroing x outside each half
    parts = []
    for half in (idx[::2], idx[1::2]):
        xh = np.zeros_like(x)
        xh[half] = x[half]
        o = decdec_linear_ref(q, s, z, xh, len(half), rc=rc, rS=rS)
        assert set(o["idx"]) == set(half)
        parts.append(o["odec"])
    assert np.allclose(parts[0] + parts[1], full["odec"], rtol=1e-13, atol=1e-15)


def test_compensation_usually_helps():
    # statistical (not a pin): error vs W x falls with k in most trials
    W, q, s, z, rc, rS, r16 = _small_layer(d_in=1024, d_out=128, seed=12)
    X = gen_activations(1024, 20, seed=13)
    wins = 0
    for x in X:
        Wx = x.astype(np.float64) @ W.astype(np.float64)
        e0 = np.mean((decdec_linear_ref(q, s, z, x, 0, rc=rc, rS=rS)["y64"] - Wx) ** 2)
        e1 = np.mean((decdec_linear_ref(q, s, z, x, 32, rc=rc, rS=rS)["y64"] - Wx) ** 2)
        wins += e1 < e0
    assert wins >= 18


def test_sorted_beats_random_order():
    # synthetic analogue of fig:cumul_errors: compensating by |x| order beats random order
    W, q, s, z, rc, rS, r16 = _small_layer(d_in=1024, d_out=128, seed=21)
    x = gen_activations(1024, 1, seed=22)[0]
    Wx = x.astype(np.float64) @ W.astype(np.float64)
    base = decdec_linear_ref(q, s, z, x, 0, r16=r16)["y64"]
    R16 = r16.astype(np.float64)
    order_sorted = np.argsort(-np.abs(x.astype(np.float64)), kind="stable")
    order_rand = np.random.default_rng(0).permutation(1024)

    def area(order):
        y = base.copy()
        tot = 0.0
        for i in order[:128]:
            y = y + x[i].astype(np.float64) * R16[i]
            tot += np.mean((y - Wx) ** 2)
        return tot

    assert area(order_sorted) < area(order_rand)


def test_perf_layer_shapes():
    L = gen_perf_layer(1024, 256, 3, seed=1)
    assert L["q"].shape == (1024, 256) and L["q"].max() <= 7
    assert L["s"].shape == (8, 256) and L["z"].min() >= 3 and L["z"].max() <= 4
    assert np.abs(L["rc"]).max() <= 7 and L["rS"].shape == (256,)


# ----------------------------------------------------------------------------- O6
def test_pack_golden_words(golden):
    for ln in golden("pack_words.txt"):
        kind, rest = ln.split(None, 1)
        lhs, rhs = (p.strip() for p in rest.split(";"))
        exp = [int(w, 16) for w in rhs.split()]
        if kind == "w4k":
            q = np.zeros((8, 1), np.uint8)
            q[:, 0] = [int(v) for v in lhs.split()]
            assert [int(w) for w in oracle.pack_w4k_ref(q)[0]] == exp
        elif kind == "w3k":
            q = np.zeros((32, 1), np.uint8)
            for tok in lhs.split():
                c, v = tok.split(":")
                q[int(c), 0] = int(v)
            assert [int(w) for w in oracle.pack_w3k_ref(q)[0]] == exp
        elif kind == "rq":
            c = np.zeros((1, 8), np.int8)
            c[0] = [int(v) for v in lhs.split()]
            assert [int(w) for w in oracle.pack_rq_ref(c)[0]] == exp


@pytest.mark.parametrize("bits", [3, 4])
def test_pack_roundtrip(bits):
    L = gen_perf_layer(256, 64, bits, seed=2)
    if bits == 4:
        words = oracle.pack_w4k_ref(L["q"])
        assert words.shape == (64, 32)
        assert np.array_equal(oracle.unpack_w4k_ref(words, 256), L["q"])
    else:
        words = oracle.pack_w3k_ref(L["q"])
        assert words.shape == (64, 24)
        assert np.array_equal(oracle.unpack_w3k_ref(words, 256), L["q"])
    rq = oracle.pack_rq_ref(L["rc"])
    assert rq.shape == (256, 8)
    assert np.array_equal(oracle.unpack_rq_ref(rq, 64), L["rc"])
    # every bit of the 3-bit layout is used exactly once (3.0 bits/weight)
    if bits == 3:
        full = oracle.pack_w3k_ref(np.full((32, 1), 7, np.uint8))
        assert [int(w) for w in full[0]] == [0xFFFFFFFF] * 3
