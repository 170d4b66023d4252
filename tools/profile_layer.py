"""Run one DecDEC layer call a few times (for ncu --set full captures).
usage: python tools/profile_layer.py --shape 4096x14336 --bits 3 --kchunk 21 --iters 4"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_20185_b200 as dd  # noqa: E402
from synth import gen_activations, gen_perf_layer_device, layer_seed  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096x14336")
ap.add_argument("--bits", type=int, default=3)
ap.add_argument("--kchunk", type=int, default=0)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--instances", type=int, default=8, help="distinct weight copies (defeat L2)")
a = ap.parse_args()
d_in, d_out = (int(v) for v in a.shape.split("x"))
lins, hosts = [], []
for i in range(a.instances):
    g = gen_perf_layer_device(d_in, d_out, a.bits, layer_seed("prof", i))
    rb = d_out // 2
    off = (d_in * rb + 255) // 256 * 256
    hb = dd.HostBuffer(off + 2 * d_out)
    hv = torch.from_numpy(hb.numpy(np.uint8))
    hv[: d_in * rb].copy_(g["r"].cpu())
    hv[off: off + 2 * d_out].copy_(g["rS"].view(torch.uint8).cpu())
    lins.append(dd.QuantLinear.from_device_packed(d_in, d_out, a.bits, g["w"], g["s"], g["z"], host=hb, r_bits=4,
                                                  host_scales_off=off))
    hosts.append(hb)
x = torch.from_numpy(gen_activations(d_in, 1, seed=3, kind="d" if d_in > 8192 else "qkv")[0]).cuda()
k = a.kchunk * d_in // 1024
ws = dd.Workspace(max(k, 1), d_out)
y = torch.empty(d_out, dtype=torch.float16, device="cuda")
print("plan", lins[0].plan(k))
for it in range(a.iters):
    for lin in lins:
        lin(x, k, y=y, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for it in range(a.iters):
    for lin in lins:
        lin(x, k, y=y, workspace=ws)
e1.record()
e1.synchronize()
print(f"eager us/call {e0.elapsed_time(e1) * 1e3 / (a.iters * len(lins)):.2f}")
