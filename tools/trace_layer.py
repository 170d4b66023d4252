"""Per-CTA timeline of fused layer kernels (decdec_debug_trace): runs N instances of one shape
back to back (eager, one stream, PDL as in production) with a separate trace buffer per call,
prints event times (µs, median / max over CTAs) relative to the selector start (k > 0) or the
earliest CTA start.
usage: python tools/trace_layer.py --shape 4096x14336 --kchunk 21"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_20185_b200 as dd  # noqa: E402
from synth import gen_activations, gen_perf_layer_device, layer_seed  # noqa: E402

EV = ["start", "tma0", "x_loaded", "stage0", "gemv_done", "sel_visible", "sel_staged", "gather_done", "exit"]
ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096x14336")
ap.add_argument("--bits", type=int, default=3)
ap.add_argument("--kchunk", type=int, default=0)
ap.add_argument("--n", type=int, default=6)
a = ap.parse_args()
d_in, d_out = (int(v) for v in a.shape.split("x"))
lins, hosts, xs = [], [], []
for i in range(a.n):
    g = gen_perf_layer_device(d_in, d_out, a.bits, layer_seed("trace", i))
    rb = d_out // 2
    off = (d_in * rb + 255) // 256 * 256
    hb = dd.HostBuffer(off + 2 * d_out)
    hv = torch.from_numpy(hb.numpy(np.uint8))
    hv[: d_in * rb].copy_(g["r"].cpu())
    hv[off: off + 2 * d_out].copy_(g["rS"].view(torch.uint8).cpu())
    lins.append(dd.QuantLinear.from_device_packed(d_in, d_out, a.bits, g["w"], g["s"], g["z"], host=hb, r_bits=4,
                                                  host_scales_off=off))
    hosts.append(hb)
    xs.append(torch.from_numpy(gen_activations(d_in, 1, seed=i, kind="d" if d_in > 8192 else "qkv")[0]).cuda())
k = a.kchunk * d_in // 1024
ws = dd.Workspace(max(k, 1), d_out)
y = torch.empty(d_out, dtype=torch.float16, device="cuda")
NB = 2 + 1024 * 20
bufs = [torch.zeros(NB, dtype=torch.int64, device="cuda") for _ in range(a.n)]
for rep in range(2):
    for i, lin in enumerate(lins):
        dd.decdec_debug_trace(bufs[i].data_ptr(), NB * 8)
        lin(xs[i], k, y=y, workspace=ws)
    torch.cuda.synchronize()
dd.decdec_debug_trace(0, 0)
import json  # noqa: E402
plan = json.loads(lins[0].plan(k))
grid = plan["grid"] + (1 if k else 0)  # + selector CTA
print("plan", plan)
prev_end = None
for i in range(a.n):
    t = bufs[i].cpu().numpy()
    ev = t[2: 2 + grid * 20].reshape(grid, 20).astype(np.float64)
    base = ev[:, 0][ev[:, 0] > 0].min()
    sel0, sel1 = (ev[0, 5], ev[0, 6]) if k else (0, 0)
    rel = (ev - base) / 1e3
    line = [f"call {i}"]
    if k:
        line.append(f"sel {(sel1 - sel0) / 1e3:.2f}")
    for j, name in enumerate(EV):
        col = rel[:, j][ev[:, j] > 0]
        if len(col):
            line.append(f"{name} {np.median(col):.2f}/{col.max():.2f}")
    end = max(ev[:, 4].max(), ev[:, 7].max())
    if prev_end is not None:
        line.append(f"gap_from_prev {(base - prev_end) / 1e3:.2f}")
    prev_end = end
    line.append(f"total {(end - base) / 1e3:.2f}")
    print("  ".join(line))
