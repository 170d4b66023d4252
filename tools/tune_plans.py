"""Time one layer shape under different launch plans (DECDEC_PLAN="NC,RPS"), each in its own
process (the override is read once per process).  Graph of N distinct weight instances
replayed; prints µs per layer call.
usage: python tools/tune_plans.py --shape 4096x14336 --bits 3 --kchunk 0 --configs 8,1 8,2 8,4 4,2"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, json
sys.path.insert(0, %(root)r)
import numpy as np, torch
import paper_2412_20185_b200 as dd
from synth import gen_activations, gen_perf_layer_device, layer_seed
d_in, d_out, bits, kc, n = %(d_in)d, %(d_out)d, %(bits)d, %(kc)d, %(n)d
lins, hosts, xs = [], [], []
for i in range(n):
    g = gen_perf_layer_device(d_in, d_out, bits, layer_seed("tune", i))
    rb = d_out // 2; off = (d_in * rb + 255) // 256 * 256
    hb = dd.HostBuffer(off + 2 * d_out)
    hv = torch.from_numpy(hb.numpy(np.uint8)); hv[: d_in * rb].copy_(g["r"].cpu()); hv[off: off + 2 * d_out].copy_(g["rS"].view(torch.uint8).cpu())
    lins.append(dd.QuantLinear.from_device_packed(d_in, d_out, bits, g["w"], g["s"], g["z"], host=hb, r_bits=4, host_scales_off=off)); hosts.append(hb)
    xs.append(torch.from_numpy(gen_activations(d_in, 1, seed=i, kind="d" if d_in > 8192 else "qkv")[0]).cuda())
k = kc * d_in // 1024
ws = dd.Workspace(max(k, 1), d_out)
ys = [torch.empty(d_out, dtype=torch.float16, device="cuda") for _ in range(n)]
st = dd.Stack(lins, [k] * n, xs, ys, ws)
for _ in range(5): st.launch()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = 20
e0.record()
for _ in range(R): st.launch()
e1.record(); e1.synchronize()
print(json.dumps({"plan": json.loads(lins[0].plan(k)), "us": e0.elapsed_time(e1) * 1e3 / (R * n)}))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="4096x14336")
    ap.add_argument("--bits", type=int, default=3)
    ap.add_argument("--kchunk", type=int, default=0)
    ap.add_argument("--n", type=int, default=16)
    ap.add_argument("--configs", nargs="*", default=["auto"])
    a = ap.parse_args()
    d_in, d_out = (int(v) for v in a.shape.split("x"))
    for c in a.configs:
        env = dict(os.environ)
        if c != "auto":
            env["DECDEC_PLAN"] = c
        code = CHILD % dict(root=ROOT, d_in=d_in, d_out=d_out, bits=a.bits, kc=a.kchunk, n=a.n)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        out = r.stdout.strip().splitlines()
        if r.returncode or not out:
            print(json.dumps({"config": c, "error": (r.stderr or "")[-300:]}))
            continue
        d = json.loads(out[-1])
        p = d["plan"]
        print(json.dumps({"shape": a.shape, "bits": a.bits, "kchunk": a.kchunk, "config": c, "us": round(d["us"], 3),
                          "NC": p["NC"], "RPS": p["RPS"], "TR": p["TR"], "stages": p["stages"], "tiles": p["n_tiles"]}))


if __name__ == "__main__":
    main()
