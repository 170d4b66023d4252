"""Seeded synthetic generators (no method arithmetic).  Recipe: DESIGN.md "Input recipe".

Weights   W_ij ~ N(0, 0.02^2) x per-column LogNormal(0, 0.25), cast to fp16.
Acts      x_i = sigma_i * t_i, sigma_i ~ LogNormal(0, 0.5) fixed per layer, t_i ~ Student-t(3)
          per step, plus 8 persistent massive-outlier channels per layer with sigma x 20
          (qkv/o/gu inputs) or x 200 (down input); clamp to +-2^15; fp16.  (S:523 style,
          'outlier-heavy activations shaped like Llama-3 decode', BASELINE.json.)
Perf      stored quantities drawn directly: q ~ U[0, 2^b-1];
layers    z ~ U{3,4} (3-bit) / U{7,8} (4-bit); s = fp16(0.02*sqrt(12)/2^b * LogNormal(0,0.25))
          per group; residual codes ~ U[-7,7]; S_j = fp16(median_g s_gj / 14).
"""

from __future__ import annotations

import hashlib

import numpy as np

# Layer shapes d_in x d_out (W is logically [d_in, d_out], rows = input channels).
SHAPES = {
    "config1": {"l": (1024, 1024)},
    "llama3_8b": {
        "q": (4096, 4096), "k": (4096, 1024), "v": (4096, 1024), "o": (4096, 4096),
        "gate": (4096, 14336), "up": (4096, 14336), "down": (14336, 4096),
        "qkv": (4096, 6144), "gu": (4096, 28672), "d": (14336, 4096),
    },
    "phi3_medium": {"qkv": (5120, 7680), "o": (5120, 5120), "gu": (5120, 35840), "d": (17920, 5120)},
    "llama3_70b": {"qkv": (8192, 10240), "o": (8192, 8192), "gu": (8192, 57344), "d": (28672, 8192)},
}

# Decode-step layer classes per block (the paper's classes qkv, o, gu, d) and blocks.
MODEL_BLOCKS = {"llama3_8b": 32, "phi3_medium": 40, "llama3_70b": 80}


def model_layers(model: str, fused: bool = True):
    """[(label, d_in, d_out)] for one decoder block."""
    sh = SHAPES[model]
    names = ["qkv", "o", "gu", "d"] if fused else ["q", "k", "v", "o", "gate", "up", "down"]
    return [(n, *sh[n]) for n in names]


def layer_seed(*parts) -> int:
    """Stable 63-bit seed from a tuple of labels (hash(cfg, layer, block/step))."""
    h = hashlib.sha256("/".join(str(p) for p in parts).encode()).digest()
    return int.from_bytes(h[:8], "little") & ((1 << 63) - 1)


def gen_weight_fp16(d_in: int, d_out: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    col = rng.lognormal(0.0, 0.25, size=d_out)
    W = rng.normal(0.0, 0.02, size=(d_in, d_out)) * col[None, :]
    return W.astype(np.float16)


def gen_activations(d_in: int, n_steps: int, seed: int, kind: str = "qkv") -> np.ndarray:
    """[n_steps, d_in] fp16 outlier-heavy decode activations."""
    rng = np.random.default_rng(seed)
    sigma = rng.lognormal(0.0, 0.5, size=d_in)
    outl = rng.choice(d_in, size=min(8, d_in), replace=False)
    sigma[outl] *= 200.0 if kind in ("d", "down") else 20.0
    t = rng.standard_t(3.0, size=(n_steps, d_in))
    x = np.clip(sigma[None, :] * t, -32768.0, 32768.0)
    return x.astype(np.float16)


def gen_special_activations(d_in: int, kind: str, seed: int = 0) -> np.ndarray:
    """Correctness-only vectors: ties, signed zeros, all-equal, few distinct magnitudes."""
    rng = np.random.default_rng(seed)
    if kind == "all_equal":
        x = np.full(d_in, 1.5)
        x[rng.random(d_in) < 0.5] *= -1
    elif kind == "zeros":
        x = np.zeros(d_in)
        x[rng.random(d_in) < 0.5] = -0.0
    elif kind == "ties":
        x = rng.choice([0.0, -0.0, 0.25, -0.25, 1.0, -1.0, 3.0, -3.0], size=d_in)
    elif kind == "sparse":
        x = np.zeros(d_in)
        nz = rng.choice(d_in, size=max(1, d_in // 64), replace=False)
        x[nz] = rng.standard_normal(len(nz))
    else:
        raise ValueError(kind)
    return x.astype(np.float16)


def gen_perf_layer(d_in: int, d_out: int, bits: int, seed: int, group: int = 128, with_residual: bool = True):
    """Stored quantities of one quantized layer drawn directly (perf configs 2-5).

    Returns dict q uint8 [d_in, d_out], s fp16 [G, d_out], z uint8 [G, d_out],
    rc int8 [d_in, d_out] in [-7, 7], rS fp16 [d_out].
    """
    rng = np.random.default_rng(seed)
    G = d_in // group
    qmax = (1 << bits) - 1
    q = rng.integers(0, qmax + 1, size=(d_in, d_out), dtype=np.uint8)
    zlo = 3 if bits == 3 else 7
    z = rng.integers(zlo, zlo + 2, size=(G, d_out), dtype=np.uint8)
    s = (0.02 * np.sqrt(12.0) / (1 << bits) * rng.lognormal(0.0, 0.25, size=(G, d_out))).astype(np.float16)
    out = dict(q=q, s=s, z=z)
    if with_residual:
        out["rc"] = rng.integers(-7, 8, size=(d_in, d_out), dtype=np.int8)
        out["rS"] = (np.median(s.astype(np.float64), axis=0) / 14.0).astype(np.float16)
    return out


def gen_perf_layer_device(d_in: int, d_out: int, bits: int, seed: int, device="cuda", group: int = 128):
    """Perf-harness layer drawn directly on the GPU (torch RNG, seeded): uniformly random
    packed code bits (every layout here is a bijection between code bits and words, so
    random words == iid uniform codes), scales/zeros per the §8(d) recipe, and random
    residual row bytes (nibbles uniform on [1, 15], i.e. residual codes c = n - 8 on [-7, 7],
    the domain of Q_r) plus residual scales.
    Returns device tensors: w uint8 [d_out * d_in * bits / 8], s fp16 [d_out * G],
    z uint8 [d_out * G], r uint8 [d_in * d_out / 2], rS fp16 [d_out]."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed & 0x7FFFFFFFFFFFFFFF)
    G = d_in // group
    nb = d_out * d_in * bits // 8
    w = torch.randint(0, 256, (nb,), dtype=torch.uint8, device=device, generator=g)
    zlo = 3 if bits == 3 else 7
    z = torch.randint(zlo, zlo + 2, (d_out * G,), dtype=torch.uint8, device=device, generator=g)
    ln = torch.exp(torch.randn(d_out * G, device=device, generator=g) * 0.25)
    s = (0.02 * 12 ** 0.5 / (1 << bits) * ln).to(torch.float16)
    nb_r = d_in * d_out // 2
    lo = torch.randint(1, 16, (nb_r,), dtype=torch.uint8, device=device, generator=g)
    hi = torch.randint(1, 16, (nb_r,), dtype=torch.uint8, device=device, generator=g)
    r = lo | (hi << 4)
    rS = (s.float().view(d_out, G).median(dim=1).values / 14.0).to(torch.float16)
    return dict(w=w, s=s, z=z, r=r, rS=rS)


def gen_perf_layer_lut(d_in: int, d_out: int, bits: int, seed: int, with_residual: bool = True):
    """Stored quantities of one non-uniform (LUT) layer drawn directly (NEXT-3 perf / parity
    configs; the SqueezeLLM-style base of P:397): q ~ U[0, 2^b - 1]; per column a sorted table
    of 2^b fp16 values ~ N(0, 0.02^2) x LogNormal(0, 0.25) (a k-means table's shape); residual
    codes ~ U[-7, 7], S_j = fp16(median gap of column j's table / 14).
    Returns dict q uint8 [d_in, d_out], lut fp16 [2^b, d_out], rc, rS."""
    rng = np.random.default_rng(seed)
    n = 1 << bits
    q = rng.integers(0, n, size=(d_in, d_out), dtype=np.uint8)
    col = rng.lognormal(0.0, 0.25, size=d_out)
    lut = np.sort(rng.normal(0.0, 0.02, size=(n, d_out)) * col[None, :], axis=0).astype(np.float16)
    out = dict(q=q, lut=lut)
    if with_residual:
        out["rc"] = rng.integers(-7, 8, size=(d_in, d_out), dtype=np.int8)
        gaps = np.diff(lut.astype(np.float64), axis=0)
        out["rS"] = (np.median(gaps, axis=0) / 14.0).astype(np.float16)
    return out


def gen_perf_layer_lut_device(d_in: int, d_out: int, bits: int, seed: int, device="cuda"):
    """Perf-harness LUT layer drawn on the GPU: W4K nibble codes uniform on [0, 2^b - 1] (random
    bytes with each nibble masked; W4K is a bijection between codes and words) and per-column
    sorted fp16 tables [d_out][2^b] (the shape of gen_perf_layer_lut's)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed & 0x7FFFFFFFFFFFFFFF)
    n = 1 << bits
    mask = (n - 1) | ((n - 1) << 4)
    w = torch.randint(0, 256, (d_out * d_in // 2,), dtype=torch.uint8, device=device, generator=g) & mask
    col = torch.exp(torch.randn(d_out, 1, device=device, generator=g) * 0.25)
    lut = torch.sort(torch.randn(d_out, n, device=device, generator=g) * 0.02 * col, dim=1).values.to(torch.float16)
    return dict(w=w, lut=lut.reshape(-1))
