"""Liveness check (run as a child process with a timeout): three streams issue compensated
decdec_linear calls on different layers / workspaces back to back, without synchronising in
between, so several fused grids (DEC CTAs that wait for GEMV CTAs of their own grid) compete for
the SMs at once.  Prints one JSON line with the per-stream results' agreement with the serial
results.  usage: python tools/concurrency_check.py [--iters 50]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2412_20185_b200 as dd  # noqa: E402
from synth import gen_activations, gen_perf_layer, layer_seed  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=50)
a = ap.parse_args()
shapes = [(4096, 6144), (14336, 4096), (4096, 28672)]
lins, xs, wss, ks = [], [], [], []
for i, (d_in, d_out) in enumerate(shapes):
    L = gen_perf_layer(d_in, d_out, 3, seed=layer_seed("conc", i))
    lins.append(dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 3, rc=L["rc"], rS=L["rS"]))
    xs.append(torch.from_numpy(gen_activations(d_in, 1, seed=layer_seed("conc", "x", i))[0]).cuda())
    ks.append(21 * d_in // 1024)
    wss.append(dd.Workspace(ks[-1], d_out))
ref = [lin(x, k, workspace=ws).clone() for lin, x, k, ws in zip(lins, xs, ks, wss)]
torch.cuda.synchronize()
streams = [torch.cuda.Stream() for _ in shapes]
outs = [torch.empty_like(r) for r in ref]
for it in range(a.iters):
    for i, st in enumerate(streams):
        with torch.cuda.stream(st):
            lins[i](xs[i], ks[i], y=outs[i], workspace=wss[i], stream=st)
torch.cuda.synchronize()
ok = all(torch.equal(o, r) for o, r in zip(outs, ref))
print(json.dumps({"streams": len(streams), "iters": a.iters, "bit_identical_to_serial": ok}), flush=True)
sys.exit(0 if ok else 1)
