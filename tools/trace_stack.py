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
ap.add_argument("--shard-of", type=int, default=1, help="rank 0's 1/P output-feature shard of every layer")
a = ap.parse_args()
layers, hosts, xs, ys, meta = [], [], [], [], []
for b in range(a.blocks):
    for name, d_in, d_out in model_layers(a.model, fused=True):
        d_out //= a.shard_of
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
E = 20
S = 160 * E
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
ev_all = [t[2 + i * S: 2 + (i + 1) * S].reshape(160, E) for i in range(len(meta))]
t0 = min(ev[:, 0][ev[:, 0] > 0].min() for ev in ev_all)
us = lambda v: (v - t0) / 1e3


def med(c):
    c = c[c > 0]
    return us(np.median(c)) if len(c) else float("nan")


def mx(c):
    c = c[c > 0]
    return us(c.max()) if len(c) else float("nan")


def mn(c):
    c = c[c > 0]
    return us(c.min()) if len(c) else float("nan")


print("times in µs from the first layer's start.  GEMV CTAs: released(min) x_loaded(med) gemv_done(max);"
      "  DEC CTAs: sel_start(med) sel_done(max) gather_done(max) last_arrival(max) combine_done(max);  end, next release")
ends = []
for i, (b, name, d_in, d_out) in enumerate(meta):
    ev = ev_all[i]
    dec = ev[(ev[:, 5] > 0) & (ev[:, 8] == 0)]
    gem = ev[ev[:, 8] > 0]
    end = ev[:, :E].max()
    ends.append(end)
    nxt = mn(ev_all[i + 1][:, 8]) if i + 1 < len(meta) else float("nan")
    line = f"{b}:{name:4s} start {mn(ev[:, 0]):8.2f} | rel {mn(gem[:, 8]):8.2f} x {med(gem[:, 2]):8.2f} gemv {mx(gem[:, 4]):8.2f} pub {mx(gem[:, 10]):8.2f}"
    if len(dec):
        line += (f" | sel {med(dec[:, 5]):8.2f} -> {mx(dec[:, 6]):8.2f} gath {mx(np.maximum(dec[:, 7], dec[:, 1])):8.2f}"
                 f" comb {mx(dec[:, 9]):8.2f}")
    line += f" | end {us(end):8.2f} next {nxt:8.2f}"
    print(line)
nl = len(meta) // a.blocks
if a.blocks > 1:
    print(f"last block: {(ends[-1] - ends[-1 - nl]) / 1e3:.2f} us (end to end)")
print("DEC CTAs (µs, median / max over DEC CTAs): sel_start, D placed (warp 0), gather done warp 0, last warp, all partials, combine done")
for i, (b, name, d_in, d_out) in enumerate(meta):
    ev = ev_all[i]
    dec = ev[(ev[:, 5] > 0) & (ev[:, 8] == 0)]
    if len(dec):
        cols = [5, 6, 7, 1, 12, 9]
        print(f"  {b}:{name:4s}", " | ".join(f"{med(dec[:, c]):7.2f} {mx(dec[:, c]):7.2f}" for c in cols))
rows = []
for i, (b, name, d_in, d_out) in enumerate(meta):
    ev = ev_all[i]
    dec = ev[(ev[:, 5] > 0) & (ev[:, 8] == 0)]
    if len(dec):
        d0 = dec[0]
        rows.append((f"{b}:{name}", [d0[j] - d0[15] for j in (16, 17, 18, 11, 13, 19, 14, 2, 3, 4, 10)]))
if rows:
    print("DEC CTA 0 phases (SM cycles after sel_start): loads issued, coarse bin, D placed, finisher: T found, R placed, "
          "published; warp 0 done, warp 0 first issue, first item landed, scales landed (combine), o_b seen")
    for n, r in rows[:12]:
        print(f"  {n:8s}", " ".join(f"{v:7.0f}" for v in r))
