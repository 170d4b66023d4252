"""GPU parity: the sm_100a path (through the C ABI) against the float64 oracle.

Bar (BASELINE.json, DESIGN.md ledger L9): selected indices and decoded integer codes
bit-exact; outputs |y - y*| <= 1e-3 * max(|y*|, 2^-12 A_j, 2^-14)."""

import json
import os

import numpy as np
import pytest

import oracle
from oracle import (decdec_linear_ref, dequantize_base, quantize_base, quantize_residual, rel_err_unfloored, residual,
                    tolerance_ok, topk_ref)
from synth import SHAPES, gen_activations, gen_perf_layer, gen_special_activations, gen_weight_fp16, layer_seed

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2412_20185_b200 as dd  # noqa: E402

DEV = "cuda"


def to_dev(x16):
    return torch.from_numpy(np.ascontiguousarray(x16, np.float16)).to(DEV)


def check_close(y_gpu, ref, what=""):
    y = y_gpu.cpu().numpy()
    ok, err, bound = tolerance_ok(y, ref["y64"], ref["A"])
    if not ok.all():
        bad = np.nonzero(~ok)[0][:8]
        raise AssertionError(f"{what}: {int((~ok).sum())} / {len(ok)} outside tolerance; e.g. cols {bad}, "
                             f"y={y[bad]}, y*={ref['y64'][bad]}, err={err[bad]}, bound={bound[bad]}")


# ------------------------------------------------------------------ decode (integer codes)
@pytest.mark.parametrize("bits", [3, 4])
@pytest.mark.parametrize("shape", [(1024, 256), (4096, 512), (14336, 64)])
def test_debug_unpack_bit_exact(bits, shape):
    L = gen_perf_layer(*shape, bits, seed=layer_seed("unpack", bits, *shape), with_residual=False)
    lin = dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], bits)
    q = lin.debug_unpack().cpu().numpy()
    assert np.array_equal(q, L["q"].T)


# ------------------------------------------------------------------ selection (bit-exact)
@pytest.mark.parametrize("d_in", [128, 1024, 4096, 5120, 14336, 17920, 28672])
def test_select_exact(d_in):
    X = gen_activations(d_in, 3, seed=layer_seed("sel", d_in), kind="down" if d_in > 8192 else "qkv")
    for x in X:
        xd = to_dev(x)
        for k in sorted({0, 1, 7, d_in // 64, d_in // 12, d_in // 2, d_in}):
            idx, xs = dd.select(xd, k)
            ridx, rxs = topk_ref(x, k)
            assert np.array_equal(idx.cpu().numpy(), ridx), (d_in, k)
            assert np.array_equal(xs.cpu().numpy().view(np.uint16), rxs.view(np.uint16))


@pytest.mark.parametrize("kind", ["all_equal", "zeros", "ties", "sparse"])
def test_select_ties_and_degenerate(kind):
    for d_in in (1024, 4096, 14336):
        x = gen_special_activations(d_in, kind, seed=d_in)
        for k in (1, 3, 100, d_in // 3, d_in - 1):
            idx, _ = dd.select(to_dev(x), k)
            assert np.array_equal(idx.cpu().numpy(), topk_ref(x, k)[0]), (kind, d_in, k)


@pytest.mark.parametrize("d_in", [1024, 4096, 17920, 28672])
def test_select_chunk_mode(d_in):
    x = gen_activations(d_in, 1, seed=layer_seed("chunk", d_in))[0]
    for kc in (1, 8, 32, 200, 1024):
        idx, xs = dd.select(to_dev(x), kc, chunk=1024)
        ridx, _ = topk_ref(x, kc, chunk=1024)
        assert np.array_equal(idx.cpu().numpy(), ridx), (d_in, kc)


# ------------------------------------------------------------------ config 1 full pipeline
def _config1(bits=3, seed=1):
    d_in, d_out = SHAPES["config1"]["l"]
    W = gen_weight_fp16(d_in, d_out, layer_seed("config1", "W", seed))
    q, s, z = quantize_base(W, bits)
    R = residual(W, dequantize_base(q, s, z))
    rc, rS = quantize_residual(R, 4)
    r16 = quantize_residual(R, 16)
    return W, q, s, z, rc, rS, r16


@pytest.mark.parametrize("bits", [3, 4])
@pytest.mark.parametrize("r_bits", [4, 16])
def test_config1_parity(bits, r_bits):
    W, q, s, z, rc, rS, r16 = _config1(bits)
    lin = (dd.QuantLinear.from_codes(q, s, z, bits, rc=rc, rS=rS) if r_bits == 4
           else dd.QuantLinear.from_codes(q, s, z, bits, r16=r16))
    ws = dd.Workspace(1024, 1024)
    X = gen_activations(1024, 8, seed=layer_seed("config1", "x"))
    for x in X:
        xd = to_dev(x)
        for k in (0, 1, 16, 100, 1024):
            sel = torch.full((max(k, 1),), -1, dtype=torch.int32, device=DEV)
            y = lin(xd, k, sel=sel, workspace=ws)
            ref = decdec_linear_ref(q, s, z, x, k, rc=rc if r_bits == 4 else None, rS=rS if r_bits == 4 else None,
                                    r16=r16 if r_bits == 16 else None)
            if k:
                assert np.array_equal(sel.cpu().numpy(), ref["idx"])
            check_close(y, ref, f"config1 bits={bits} r={r_bits} k={k}")


def test_k0_bit_identical_to_gemv():
    W, q, s, z, rc, rS, r16 = _config1(3)
    lin = dd.QuantLinear.from_codes(q, s, z, 3, rc=rc, rS=rS)
    x = to_dev(gen_activations(1024, 1, seed=5)[0])
    ws = dd.Workspace(64, 1024)
    assert torch.equal(lin(x, 0, workspace=ws), lin.gemv(x))


def test_full_fp16_compensation_recovers_Wx():
    W, q, s, z, rc, rS, r16 = _config1(3)
    lin = dd.QuantLinear.from_codes(q, s, z, 3, r16=r16)
    ws = dd.Workspace(1024, 1024)
    x = gen_activations(1024, 1, seed=6)[0]
    y = lin(to_dev(x), 1024, workspace=ws).cpu().numpy()
    Wx = x.astype(np.float64) @ W.astype(np.float64)
    A = np.abs(x.astype(np.float64)) @ np.abs(W.astype(np.float64))
    # fp16 residual rounding (2^-11 relative per element) adds to the L9 bound here
    err = np.abs(y.astype(np.float64) - Wx)
    assert np.all(err <= 1e-3 * np.maximum(np.abs(Wx), 2.0 ** -12 * A) + 2e-3 * 2.0 ** -11 * A)


# ------------------------------------------------------------------ Llama-3-8B shapes (config 2/3)
# L9 unfloored relative error per case (DESIGN.md ledger L9 "also report"); written to
# $DECDEC_PARITY_REPORT (JSON) at the end of the session when that variable is set.
REPORT = {}


@pytest.fixture(scope="module", autouse=True)
def _write_report():
    yield
    path = os.environ.get("DECDEC_PARITY_REPORT")
    if path and REPORT:
        old = {}
        if os.path.exists(path):
            with open(path) as f:
                old = json.load(f)
        old.update(REPORT)
        with open(path, "w") as f:
            json.dump(old, f, indent=1, sort_keys=True)


def check_full(y_gpu, ref, what):
    """Every output column against the oracle (L9) + the unfloored relative error report."""
    y = y_gpu.cpu().numpy() if hasattr(y_gpu, "cpu") else y_gpu
    ok, err, bound = tolerance_ok(y, ref["y64"], ref["A"])
    r, n = rel_err_unfloored(y, ref["y64"])
    REPORT[what] = {"cols": int(len(ok)), "max_err_over_bound": float(np.max(err / bound)) if len(ok) else 0.0,
                    "rel_err_unfloored": r, "n_unfloored": n}
    if not ok.all():
        bad = np.nonzero(~ok)[0][:8]
        raise AssertionError(f"{what}: {int((~ok).sum())} / {len(ok)} outside tolerance; e.g. cols {bad}, "
                             f"y={y[bad]}, y*={ref['y64'][bad]}, err={err[bad]}, bound={bound[bad]}")


_LAYERS = {}


def perf_layer(model, name, bits, d_r=None, tag=""):
    """Seeded perf layer + its oracle W_hat (cached: dequantized once per layer)."""
    key = (model, name, bits, d_r, tag)
    if key not in _LAYERS:
        _LAYERS.clear()  # keep one layer's W_hat (float64) alive at a time
        d_in, d_out = SHAPES[model][name]
        d = d_out if d_r is None else d_r
        L = gen_perf_layer(d_in, d, bits, seed=layer_seed(model, name, bits, d, tag))
        L["W_hat"] = dequantize_base(L["q"], L["s"], L["z"])
        L["lin"] = dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], bits, rc=L["rc"], rS=L["rS"])
        _LAYERS[key] = L
    return _LAYERS[key]


@pytest.mark.parametrize("bits", [3, 4])
@pytest.mark.parametrize("name", ["qkv", "o", "gu", "d", "k"])
def test_llama_shapes_all_columns(bits, name):
    """Config 2/3 shapes: EVERY output column within L9 at k_chunk 0/8/21/82, selection bit-exact."""
    d_in, d_out = SHAPES["llama3_8b"][name]
    L = perf_layer("llama3_8b", name, bits)
    lin = L["lin"]
    ws = dd.Workspace(oracle.k_from_kchunk(82, d_in), d_out)
    X = gen_activations(d_in, 2, seed=layer_seed("llama3_8b", name, "x"), kind="d" if name == "d" else "qkv")
    for xi, x in enumerate(X):
        xd = to_dev(x)
        for kc in (0, 8, 21, 82):
            k = oracle.k_from_kchunk(kc, d_in)
            sel = torch.empty(max(k, 1), dtype=torch.int32, device=DEV)
            y = lin(xd, k, sel=sel, workspace=ws)
            ref = decdec_linear_ref(L["q"], L["s"], L["z"], x, k, rc=L["rc"], rS=L["rS"], W_hat=L["W_hat"])
            if k:
                assert np.array_equal(sel.cpu().numpy(), ref["idx"])
            check_full(y, ref, f"llama3_8b/{name}/w{bits}/kc{kc}/x{xi}")


# ------------------------------------------------------------------ Phi-3 / Llama-3-70B shards (configs 4/5)
@pytest.mark.parametrize("model,name,P", [("phi3_medium", "qkv", 1), ("phi3_medium", "o", 1), ("phi3_medium", "gu", 1),
                                          ("phi3_medium", "d", 1), ("phi3_medium", "o", 8), ("phi3_medium", "gu", 8),
                                          ("phi3_medium", "d", 8), ("llama3_70b", "qkv", 8), ("llama3_70b", "o", 8),
                                          ("llama3_70b", "d", 8), ("llama3_70b", "gu", 8)])
def test_tp_shard_shapes_all_columns(model, name, P):
    """A rank's output-feature shard (d_out / P columns) at the BASELINE configs
    4/5 shapes (P = 1: the whole Phi-3 layer): selection bit-exact (identical on every rank),
    every output column within L9."""
    d_in, d_out = SHAPES[model][name]
    d_r = d_out // P
    L = perf_layer(model, name, 3, d_r=d_r, tag=P)
    lin = L["lin"]
    ws = dd.Workspace(oracle.k_from_kchunk(82, d_in), d_r)
    x = gen_activations(d_in, 1, seed=layer_seed(model, name, "x"), kind="d" if name == "d" else "qkv")[0]
    xd = to_dev(x)
    for kc in (0, 21, 82):
        k = oracle.k_from_kchunk(kc, d_in)
        sel = torch.empty(max(k, 1), dtype=torch.int32, device=DEV)
        y = lin(xd, k, sel=sel, workspace=ws)
        ref = decdec_linear_ref(L["q"], L["s"], L["z"], x, k, rc=L["rc"], rS=L["rS"], W_hat=L["W_hat"])
        if k:
            assert np.array_equal(sel.cpu().numpy(), ref["idx"])
        check_full(y, ref, f"{model}/{name}/P{P}/kc{kc}")


# ------------------------------------------------------------------ every DEC CTA's selection
def _plan(lin, k):
    return json.loads(lin.plan(k))


@pytest.mark.parametrize("name,kc", [("qkv", 21), ("o", 4), ("gu", 21), ("d", 21), ("d", 82), ("gu", 82)])
def test_every_dec_cta_selection_bit_exact(name, kc):
    """Each DEC CTA computes the exact Top-k itself; the `sel` output shows only
    CTA 0's.  decdec_debug_selections makes EVERY DEC CTA dump its own S / x[S]: each must be
    the oracle's selection (as a set, with x[S] bit-exact) and all must be identical."""
    d_in, d_out = SHAPES["llama3_8b"][name]
    L = perf_layer("llama3_8b", name, 3)
    lin = L["lin"]
    k = oracle.k_from_kchunk(kc, d_in)
    ws = dd.Workspace(k, d_out)
    n_dec = _plan(lin, k)["n_dec"]
    assert n_dec >= 1
    X = gen_activations(d_in, 2, seed=layer_seed("dbgsel", name, kc), kind="d" if name == "d" else "qkv")
    dbg_i = torch.full((n_dec, k), -1, dtype=torch.int32, device=DEV)
    dbg_x = torch.zeros((n_dec, k), dtype=torch.float16, device=DEV)
    dd.decdec_debug_selections(dbg_i.data_ptr(), dbg_x.data_ptr(), k, n_dec)
    try:
        for x in X:
            dbg_i.fill_(-1)
            lin(to_dev(x), k, workspace=ws)
            torch.cuda.synchronize()
            ridx, rxs = topk_ref(x, k)
            I = dbg_i.cpu().numpy()
            XS = dbg_x.cpu().numpy().view(np.uint16)
            for c in range(n_dec):
                order = np.argsort(I[c], kind="stable")
                assert np.array_equal(I[c][order], ridx), (name, kc, c)
                assert np.array_equal(XS[c][order], rxs.view(np.uint16)), (name, kc, c)
                assert np.array_equal(I[c], I[0]) and np.array_equal(XS[c], XS[0]), (name, kc, c)
    finally:
        dd.decdec_debug_selections(0, 0, 0, 0)


# ------------------------------------------------------------------ tuner-chosen DEC CTA counts
@pytest.mark.parametrize("n_dec", [2, 4, 8, 16, 24, 32, 48, 64])
def test_parity_under_dec_cta_override(n_dec):
    """decdec_set_dec_ctas (the tuner's knob, §4.4 n_tb): every plan it can produce
    stays exact -- all columns of o / gu / d at k_chunk 8 and 21."""
    dd.decdec_set_dec_ctas(n_dec)
    try:
        for name in ("o", "gu", "d"):
            d_in, d_out = SHAPES["llama3_8b"][name]
            L = perf_layer("llama3_8b", name, 3)
            lin = L["lin"]
            ws = dd.Workspace(oracle.k_from_kchunk(21, d_in), d_out)
            x = gen_activations(d_in, 1, seed=layer_seed("ndec", name, n_dec), kind="d" if name == "d" else "qkv")[0]
            for kc in (8, 21):
                k = oracle.k_from_kchunk(kc, d_in)
                plan = _plan(lin, k)
                assert 1 <= plan["n_dec"] <= (d_out + 255) // 256  # clamped to the output segments
                sel = torch.empty(k, dtype=torch.int32, device=DEV)
                y = lin(to_dev(x), k, sel=sel, workspace=ws)
                ref = decdec_linear_ref(L["q"], L["s"], L["z"], x, k, rc=L["rc"], rS=L["rS"], W_hat=L["W_hat"])
                assert np.array_equal(sel.cpu().numpy(), ref["idx"])
                check_full(y, ref, f"ndec{n_dec}/{name}/kc{kc}")
    finally:
        dd.decdec_set_dec_ctas(0)


def test_r16_llama_o_shape():
    """r_bits = 16 (Table 3 "FP16") at a Llama-3-8B shape (o, 4096 x 4096), all columns."""
    d_in, d_out = SHAPES["llama3_8b"]["o"]
    L = gen_perf_layer(d_in, d_out, 3, seed=layer_seed("r16", "o"))
    rng = np.random.default_rng(5)
    r16 = (rng.standard_normal((d_in, d_out)) * 0.002).astype(np.float16)
    lin = dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 3, r16=r16)
    W_hat = dequantize_base(L["q"], L["s"], L["z"])
    ws = dd.Workspace(d_in, d_out)
    x = gen_activations(d_in, 1, seed=layer_seed("r16", "x"))[0]
    for kc in (8, 21, 82, 1024):
        k = oracle.k_from_kchunk(kc, d_in)
        sel = torch.empty(k, dtype=torch.int32, device=DEV)
        y = lin(to_dev(x), k, sel=sel, workspace=ws)
        ref = decdec_linear_ref(L["q"], L["s"], L["z"], x, k, r16=r16, W_hat=W_hat)
        assert np.array_equal(sel.cpu().numpy(), ref["idx"])
        check_full(y, ref, f"r16/o/kc{kc}")


# ------------------------------------------------------------------ NEXT-3: non-uniform (LUT) base
@pytest.mark.parametrize("bits", [3, 4])
def test_lut_config1_full_pipeline(bits):
    """SqueezeLLM-style LUT base (ledger L17) with DecDEC compensation: seeded fp16
    W -> oracle k-means tables -> residual R = W - W_hat (O2) -> Q_r (O3) -> the LUT GEMV kernel
    (k = 0) and the fused kernel with the LUT base (k = 16, the compensation of P:204-207):
    every output column within L9, selection bit-exact, codes decoded bit-exact."""
    d_in, d_out = SHAPES["config1"]["l"]
    W = gen_weight_fp16(d_in, d_out, layer_seed("lut", "W", bits))
    q, lut = oracle.quantize_base_lut(W, bits)
    rc, rS = quantize_residual(residual(W, oracle.dequantize_lut(q, lut)), 4)
    lin = dd.QuantLinear.from_lut_codes(q, lut, bits, rc=rc, rS=rS)
    assert np.array_equal(lin.debug_unpack().cpu().numpy(), q.T)
    # k = 0: the fused kernel's LUT GEMV CTAs alone (3-bit tables) or k_gemv16 (4-bit tables)
    assert _plan(lin, 0).get("n_dec", 0) == 0 and (_plan(lin, 0).get("kernel") == "k_gemv") == (bits == 4)
    assert _plan(lin, 16)["n_dec"] >= 1   # k > 0: the fused kernel with DEC CTAs
    ws = dd.Workspace(64, d_out)
    X = gen_activations(d_in, 4, seed=layer_seed("lut", "x", bits))
    for xi, x in enumerate(X):
        y = lin(to_dev(x), 0)
        ref = decdec_linear_ref(q, None, None, x, 0, lut=lut)
        check_full(y, ref, f"lut/config1/b{bits}/x{xi}")
        assert torch.equal(y, lin.gemv(to_dev(x)))
        for k in (16, 64):
            sel = torch.empty(k, dtype=torch.int32, device=DEV)
            y = lin(to_dev(x), k, sel=sel, workspace=ws)
            ref = decdec_linear_ref(q, None, None, x, k, rc=rc, rS=rS, lut=lut)
            assert np.array_equal(sel.cpu().numpy(), ref["idx"])
            check_full(y, ref, f"lut/config1/b{bits}/k{k}/x{xi}")


@pytest.mark.parametrize("bits", [3, 4])
@pytest.mark.parametrize("model,name", [("llama3_8b", "qkv"), ("llama3_8b", "o"), ("llama3_8b", "gu"),
                                        ("llama3_8b", "d"), ("phi3_medium", "o"), ("phi3_medium", "d")])
def test_lut_shapes_all_columns(bits, model, name):
    """LUT base at full Llama-3-8B / Phi-3 shapes, k_chunk 0 (k_gemv16) and 21 (fused kernel with
    the LUT base + compensation): every output column, selection bit-exact."""
    from synth import gen_perf_layer_lut

    d_in, d_out = SHAPES[model][name]
    L = gen_perf_layer_lut(d_in, d_out, bits, seed=layer_seed("lutperf", model, name, bits))
    lin = dd.QuantLinear.from_lut_codes(L["q"], L["lut"], bits, rc=L["rc"], rS=L["rS"])
    W_hat = oracle.dequantize_lut(L["q"], L["lut"])
    x = gen_activations(d_in, 1, seed=layer_seed("lutperf", name, "x"), kind="d" if name == "d" else "qkv")[0]
    ws = dd.Workspace(oracle.k_from_kchunk(21, d_in), d_out)
    for kc in (0, 21):
        k = oracle.k_from_kchunk(kc, d_in)
        sel = torch.empty(max(k, 1), dtype=torch.int32, device=DEV)
        y = lin(to_dev(x), k, sel=sel if k else None, workspace=ws)
        ref = decdec_linear_ref(L["q"], None, None, x, k, rc=L["rc"], rS=L["rS"], W_hat=W_hat)
        if k:
            assert np.array_equal(sel.cpu().numpy(), ref["idx"])
        check_full(y, ref, f"lut/{model}/{name}/b{bits}/kc{kc}")


@pytest.mark.parametrize("kind", ["all_equal", "zeros", "ties", "sparse"])
def test_fused_selection_ties_and_degenerate(kind):
    """The fused layer kernel's own (split-order) selector on tie-heavy / degenerate x: the
    threshold bin then holds thousands of candidates (bitmap path) or all keys are equal."""
    for d_in, d_out in ((4096, 1024), (14336, 512)):
        L = gen_perf_layer(d_in, d_out, 3, seed=layer_seed("fused_ties", d_in))
        lin = dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 3, rc=L["rc"], rS=L["rS"])
        ws = dd.Workspace(d_in // 2, d_out)
        x = gen_special_activations(d_in, kind, seed=d_in + 1)
        for k in (1, 3, 100, d_in // 5):
            sel = torch.empty(k, dtype=torch.int32, device=DEV)
            y = lin(to_dev(x), k, sel=sel, workspace=ws)
            ref = decdec_linear_ref(L["q"], L["s"], L["z"], x, k, rc=L["rc"], rS=L["rS"])
            assert np.array_equal(sel.cpu().numpy(), ref["idx"]), (kind, d_in, k)
            check_close(y, ref, f"fused ties {kind} d_in={d_in} k={k}")


def test_chunk_mode_linear():
    d_in, d_out = 5120, 640   # Phi-3 o shard at P=8; 5 chunks
    L = gen_perf_layer(d_in, d_out, 3, seed=11)
    lin = dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 3, rc=L["rc"], rS=L["rS"])
    ws = dd.Workspace(5 * 64, d_out)
    x = gen_activations(d_in, 1, seed=12)[0]
    y = lin(to_dev(x), 21, chunk=1024, workspace=ws).cpu().numpy()
    ref = decdec_linear_ref(L["q"], L["s"], L["z"], x, 21, chunk=1024, rc=L["rc"], rS=L["rS"])
    assert tolerance_ok(y, ref["y64"], ref["A"])[0].all()


def test_deterministic_repeats():
    d_in, d_out = SHAPES["llama3_8b"]["qkv"]
    L = gen_perf_layer(d_in, d_out, 3, seed=21)
    lin = dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 3, rc=L["rc"], rS=L["rS"])
    ws = dd.Workspace(256, d_out)
    x = to_dev(gen_activations(d_in, 1, seed=22)[0])
    y0 = lin(x, 84, workspace=ws).clone()
    for _ in range(50):
        assert torch.equal(lin(x, 84, workspace=ws), y0)


def test_rejects_unmapped_residual():
    L = gen_perf_layer(1024, 256, 3, seed=3)
    lin = dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 3, rc=L["rc"], rS=L["rS"])
    st = lin.struct
    bad = torch.zeros(1024 * 128, dtype=torch.uint8, device=DEV)   # device memory, not host-mapped
    st.r_rows = bad.data_ptr()
    ws = dd.Workspace(16, 256)
    x = to_dev(gen_activations(1024, 1, seed=1)[0])
    y = torch.empty(256, dtype=torch.float16, device=DEV)
    with pytest.raises(dd.DecdecError) as e:
        dd.decdec_linear(st, x.data_ptr(), 16, 0, y.data_ptr(), 0, ws.ptr, ws.nbytes,
                         torch.cuda.current_stream().cuda_stream)
    assert e.value.status == -3
    with pytest.raises(dd.DecdecError):
        lin(x, 2000, workspace=ws)


def test_stack_graph_matches_per_layer_calls():
    """decdec_stack (one captured CUDA graph) == the same layers called one by one."""
    shapes = [(4096, 1024), (1024, 4096), (4096, 2048)]
    lins, xs = [], []
    for i, (d_in, d_out) in enumerate(shapes):
        L = gen_perf_layer(d_in, d_out, 3, seed=100 + i)
        lins.append(dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 3, rc=L["rc"], rS=L["rS"]))
        xs.append(to_dev(gen_activations(d_in, 1, seed=200 + i)[0]))
    ks = [oracle.k_from_kchunk(21, d_in) for d_in, _ in shapes]
    ws = dd.Workspace(max(ks), 4096)
    ref = [lin(x, k, workspace=ws).clone() for lin, x, k in zip(lins, xs, ks)]
    ys = [torch.empty(d_out, dtype=torch.float16, device=DEV) for _, d_out in shapes]
    st = dd.Stack(lins, ks, xs, ys, ws)
    assert st.kernels == 3
    for _ in range(3):
        st.launch()
    torch.cuda.synchronize()
    for a, b in zip(ys, ref):
        assert torch.equal(a, b)
    st.close()


def test_stack_fitted_grids_match_per_layer_calls():
    """Llama-sized qkv/o layers at k_chunk 21: in the stack graph the o layer's cooperative grid is
    shrunk to fit beside qkv's DEC CTAs (decdec_api.cu stack_create, the time model admits it);
    the rows' arithmetic does not depend on the grid, so y is bit-identical to per-layer calls."""
    shapes = [(4096, 6144), (4096, 4096), (4096, 6144), (4096, 4096)]
    lins, xs = [], []
    for i, (d_in, d_out) in enumerate(shapes):
        L = gen_perf_layer(d_in, d_out, 3, seed=300 + i)
        lins.append(dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 3, rc=L["rc"], rS=L["rS"]))
        xs.append(to_dev(gen_activations(d_in, 1, seed=400 + i)[0]))
    ks = [oracle.k_from_kchunk(21, d_in) for d_in, _ in shapes]
    ws = dd.Workspace(max(ks), 6144)
    ref = [lin(x, k, workspace=ws).clone() for lin, x, k in zip(lins, xs, ks)]
    ys = [torch.empty(d_out, dtype=torch.float16, device=DEV) for _, d_out in shapes]
    st = dd.Stack(lins, ks, xs, ys, ws)
    for _ in range(3):
        st.launch()
    torch.cuda.synchronize()
    for a, b in zip(ys, ref):
        assert torch.equal(a, b)
    st.close()


# ------------------------------------------------------------------ TP entry points (1 rank)
def _comm1():
    assert dd.decdec_nccl_version() > 0, "NCCL could not be loaded by libdecdec"
    return dd.decdec_comm_init(dd.decdec_nccl_unique_id(), 0, 1)


def test_linear_tp_single_rank_matches_linear():
    """decdec_linear_tp on a 1-rank library communicator == decdec_linear (the all-gather of one
    shard is the identity); selection bit-exact against the oracle."""
    d_in, d_out = 4096, 1024
    L = gen_perf_layer(d_in, d_out, 3, seed=7)
    lin = dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 3, rc=L["rc"], rS=L["rS"])
    x = gen_activations(d_in, 1, seed=8)[0]
    k = oracle.k_from_kchunk(21, d_in)
    ws = dd.Workspace(k, d_out)
    comm = _comm1()
    try:
        assert dd.decdec_comm_rank(comm) == 0 and dd.decdec_comm_nranks(comm) == 1
        y_full = torch.empty(d_out, dtype=torch.float16, device=DEV)
        sel = torch.empty(k, dtype=torch.int32, device=DEV)
        dd.decdec_linear_tp(lin.struct, to_dev(x).data_ptr(), k, 0, y_full.data_ptr(), sel.data_ptr(),
                            ws.ptr, ws.nbytes, comm, 0)
        y_ref = lin(to_dev(x), k, workspace=ws)
        torch.cuda.synchronize()
        assert torch.equal(y_full, y_ref)
        ref = decdec_linear_ref(L["q"], L["s"], L["z"], x, k, rc=L["rc"], rS=L["rS"])
        assert np.array_equal(sel.cpu().numpy(), ref["idx"])
        check_close(y_full, ref, "linear_tp")
    finally:
        dd.decdec_comm_destroy(comm)


def test_stack_tp_single_rank_matches_stack():
    shapes = [(4096, 1024), (1024, 4096)]
    lins, xs = [], []
    for i, (d_in, d_out) in enumerate(shapes):
        L = gen_perf_layer(d_in, d_out, 3, seed=300 + i)
        lins.append(dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 3, rc=L["rc"], rS=L["rS"]))
        xs.append(to_dev(gen_activations(d_in, 1, seed=400 + i)[0]))
    ks = [oracle.k_from_kchunk(21, d_in) for d_in, _ in shapes]
    ws = dd.Workspace(max(ks), 4096)
    ref = [lin(x, k, workspace=ws).clone() for lin, x, k in zip(lins, xs, ks)]
    ys = [torch.empty(d_out, dtype=torch.float16, device=DEV) for _, d_out in shapes]
    comm = _comm1()
    try:
        h = dd.decdec_stack_create_tp([l.struct for l in lins], ks, 0, [x.data_ptr() for x in xs],
                                      [y.data_ptr() for y in ys], ws.ptr, ws.nbytes, comm, 0)
        for _ in range(2):
            dd.decdec_stack_launch(h, 0)
        torch.cuda.synchronize()
        for a, b in zip(ys, ref):
            assert torch.equal(a, b)
        dd.decdec_stack_destroy(h)
    finally:
        dd.decdec_comm_destroy(comm)


def test_tp_python_classes_world1():
    """Comm (unique id over a torch PG) + TPLinear + TPStack on a 1-rank group."""
    import socket

    import torch.distributed as dist

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        d_in, d_out = 1024, 2048
        L = gen_perf_layer(d_in, d_out, 4, seed=9)
        lin = dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 4, rc=L["rc"], rS=L["rS"])
        x = to_dev(gen_activations(d_in, 1, seed=10)[0])
        k = oracle.k_from_kchunk(32, d_in)
        ws = dd.Workspace(k, d_out)
        comm = dd.Comm()
        y_ref = lin(x, k, workspace=ws).clone()
        y_tp = dd.TPLinear(lin, comm)(x, k, workspace=ws)
        y_st = torch.empty(d_out, dtype=torch.float16, device=DEV)
        st = dd.TPStack([lin], [k], [x], [y_st], ws, comm)
        st.launch()
        torch.cuda.synchronize()
        assert torch.equal(y_tp, y_ref) and torch.equal(y_st, y_ref)
        st.close()
        comm.close()
    finally:
        dist.destroy_process_group()


def test_validation_error_codes():
    """include/decdec.h error contract: synchronous validation, nothing enqueued, the documented
    status per violated condition."""
    import ctypes

    L = gen_perf_layer(1024, 256, 3, seed=5)
    lin = dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 3, rc=L["rc"], rS=L["rS"])
    ws = dd.Workspace(64, 256)
    x = to_dev(gen_activations(1024, 1, seed=6)[0])
    y = torch.empty(256, dtype=torch.float16, device=DEV)
    s = torch.cuda.current_stream().cuda_stream

    def call(st, k=16, chunk=0, xp=None, yp=None, wsp=None, wsb=None):
        try:
            dd.decdec_linear(st, x.data_ptr() if xp is None else xp, k, chunk, y.data_ptr() if yp is None else yp,
                             0, ws.ptr if wsp is None else wsp, ws.nbytes if wsb is None else wsb, s)
            return 0
        except dd.DecdecError as e:
            return e.status

    def mod(**kw):
        st = dd.decdec_layer()
        ctypes.pointer(st)[0] = lin.struct
        for k, v in kw.items():
            setattr(st, k, v)
        return st

    base = lin.struct
    assert call(base) == 0
    assert call(mod(group_size=64)) == -4          # EUNSUPPORTED
    assert call(mod(w_bits=5)) == -4
    assert call(mod(r_bits=8)) == -4
    assert call(mod(d_in=1000)) == -1              # EINVAL: d_in % 128
    assert call(mod(d_out=100)) == -1              # d_out % 32
    assert call(mod(w_packed=base.w_packed + 4)) == -2   # EALIGN
    assert call(mod(r_scales=None)) == -1
    assert call(base, k=1025) == -1                # k > d_in
    assert call(base, k=-1) == -1
    assert call(base, chunk=1024, k=2000) == -1    # k_chunk > chunk
    assert call(base, xp=0) == -1                  # NULL x
    assert call(base, yp=y.data_ptr() + 2) == -2   # misaligned y
    assert call(base, wsb=16) == -7                # ESPACE
    torch.cuda.synchronize()
    with pytest.raises(dd.DecdecError):
        dd.decdec_linear_tp(base, x.data_ptr(), 16, 0, y.data_ptr(), 0, ws.ptr, ws.nbytes, 0, s)  # NULL comm
    with pytest.raises(dd.DecdecError):
        dd.decdec_set_dec_ctas(65)
    # decdec_select: the selector reads x as 16-B chunks (d_in % 8, 16-B aligned x)
    idx = torch.empty(64, dtype=torch.int32, device=DEV)
    xs = torch.empty(64, dtype=torch.float16, device=DEV)
    for d_in, xp, want in ((1020, x.data_ptr(), -1), (1024, x.data_ptr() + 2, -2), (0, x.data_ptr(), -1)):
        with pytest.raises(dd.DecdecError) as e:
            dd.decdec_select(xp, d_in, 16, 0, idx.data_ptr(), xs.data_ptr(), s)
        assert e.value.status == want
    with pytest.raises(dd.DecdecError) as e:
        dd.decdec_debug_selections(idx.data_ptr(), xs.data_ptr(), 0, 4)
    assert e.value.status == -1


def test_concurrent_streams_no_deadlock():
    """Liveness (include/decdec.h "one workspace per concurrent stream"): three streams issue
    compensated calls back to back; the fused grids are launched cooperatively, so none is ever
    left partially resident while its DEC CTAs wait.  Run in a child process with a timeout so a
    hang fails the test instead of the session."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "concurrency_check.py"), "--iters", "40"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert '"bit_identical_to_serial": true' in r.stdout
