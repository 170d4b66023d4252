"""Per-layer timeline of a decode-step stack (CUDA graph, PDL-chained): builds `blocks` decoder
blocks of a model's layer classes, records decdec_debug_trace events per layer, replays the
graph and prints, per layer, start (first CTA), GEMV done (last CTA), gather done, end, and the
gap from the previous layer's end (µs, relative to the first layer's start).
usage: python tools/trace_stack.py --kchunk 21 --blocks 4"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_20185_b200 as dd  # noqa: E402
from synth import gen_activations, gen_perf_layer_device, layer_seed, model_layers  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama3_8b")
ap.add_argument("--bits", type=int, default=3)
ap.add_argument("--kchunk", type=int, default=0)
ap.add_argument("--blocks", type=int, default=4)
a = ap.parse_args()
layers, hosts, xs, ys, meta = [], [], [], [], []
for b in range(a.blocks):
    for name, d_in, d_out in model_layers(a.model, fused=True):
        g = gen_perf_layer_device(d_in, d_out, a.bits, layer_seed("ts", b, name))
        rb = d_out // 2
        off = (d_in * rb + 255) // 256 * 256
        hb = dd.HostBuffer(off + 2 * d_out)
        hv = torch.from_numpy(hb.numpy(np.uint8))
        hv[: d_in * rb].copy_(g["r"].cpu())
        hv[off: off + 2 * d_out].copy_(g["rS"].view(torch.uint8).cpu())
        layers.append(dd.QuantLinear.from_device_packed(d_in, d_out, a.bits, g["w"], g["s"], g["z"], host=hb,
                                                        r_bits=4, host_scales_off=off))
        hosts.append(hb)
        xs.append(torch.from_numpy(gen_activations(d_in, 1, seed=len(xs), kind="d" if name == "d" else "qkv")[0]).cuda())
        ys.append(torch.empty(d_out, dtype=torch.float16, device="cuda"))
        meta.append((b, name, d_in, d_out))
ks = [a.kchunk * m[2] // 1024 for m in meta]
ws = dd.Workspace(max(max(ks), 1), max(m[3] for m in meta))
S = 160 * 9
NB = 2 + len(layers) * S
buf = torch.zeros(NB, dtype=torch.int64, device="cuda")
dd.decdec_debug_trace(buf.data_ptr(), NB * 8)
st = dd.Stack(layers, ks, xs, ys, ws)
dd.decdec_debug_trace(0, 0)
for _ in range(3):
    st.launch()
torch.cuda.synchronize()
buf.zero_()
st.launch()
torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.float64)
t0 = None
prev_end = None
print("layer      start  gemv_done gather_done   end    dur    gap | sel_start sel_pub  released(min/med) x_loaded(med) stage0(med) gemv_done(med)")
for i, (b, name, d_in, d_out) in enumerate(meta):
    ev = t[2 + i * S: 2 + (i + 1) * S].reshape(160, 9)
    valid = ev[:, 0] > 0
    e = ev[valid]
    start = e[:, 0].min()
    if t0 is None:
        t0 = start
    gemv = e[:, 4][e[:, 4] > 0].max() if (e[:, 4] > 0).any() else start
    gath = e[:, 7][e[:, 7] > 0].max() if (e[:, 7] > 0).any() else 0
    end = max(gemv, gath)
    gap = (start - prev_end) / 1e3 if prev_end is not None else 0.0
    print(f"{b}:{name:4s} {(start - t0) / 1e3:8.2f} {(gemv - t0) / 1e3:9.2f} {((gath - t0) / 1e3 if gath else 0):9.2f} "
          f"{(end - t0) / 1e3:8.2f} {(end - start) / 1e3:6.2f} {gap:6.2f}", end="")
    sel = ev[0] if ks[i] > 0 else None
    gm = e[1:] if ks[i] > 0 else e
    extra = ""
    if sel is not None:
        extra += f" | {(sel[5] - t0) / 1e3:8.2f} {(sel[6] - t0) / 1e3:7.2f}"
    else:
        extra += " |" + " " * 17
    med = lambda col: np.median(col[col > 0]) if (col > 0).any() else t0
    rel = gm[:, 8][gm[:, 8] > 0]
    extra += f"  {(rel.min() - t0) / 1e3 if len(rel) else 0:8.2f} {(med(gm[:, 8]) - t0) / 1e3:8.2f}"
    extra += f"  xland {(med(gm[:, 5]) - t0) / 1e3:8.2f}"
    extra += f"  {(med(gm[:, 2]) - t0) / 1e3:8.2f} {(med(gm[:, 3]) - t0) / 1e3:8.2f} {(med(gm[:, 4]) - t0) / 1e3:8.2f}"
    print(extra)
    prev_end = end
