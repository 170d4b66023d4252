"""DecDEC parameter tuner on the GPU (§4.4; search in
paper_2412_20185_b200/tuner.py): measure µs per layer call for every layer class at each
(DEC CTAs n, k_chunk) of a grid, then run the paper's two-phase search for each target
slowdown and print the result in Table 2's format (n_max / (k_qkv, k_o, k_gu, k_d) -> slowdown).
usage: python tools/tune.py [--model llama3_8b] [--bits 3] [--out gpurun_out/tuner.json]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2412_20185_b200 as dd  # noqa: E402
from paper_2412_20185_b200 import tuner  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama3_8b")
ap.add_argument("--bits", type=int, default=3)
ap.add_argument("--n", default="4,8,16,24,32,48")
ap.add_argument("--kgrid", default="0,1,2,3,4,6,8,12,16,21,32")
ap.add_argument("--targets", default="0.025,0.05,0.1,0.2,0.5,1.0")
ap.add_argument("--blocks", type=int, default=8, help="instances per class timed together (defeat L2)")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "tuner.json"))
a = ap.parse_args()

bench.MODEL_BLOCKS[a.model] = a.blocks  # measure a.blocks instances per class
M = bench.Model(dd, torch, a.model, a.bits, 0, 1, 2, "cuda")
ns = [int(v) for v in a.n.split(",")]
kgrid = [int(v) for v in a.kgrid.split(",")]
ws = dd.Workspace(bench.k_of(max(kgrid), M.max_d_in), M.max_d_out)
stream = torch.cuda.current_stream()
names = []
for m in M.meta:
    if m[1] not in names:
        names.append(m[1])
table = {c: {} for c in names}
for c in names:
    idx = [i for i, m in enumerate(M.meta) if m[1] == c]
    for n in ns:
        dd.decdec_set_dec_ctas(n)
        table[c][n] = {}
        for kc in kgrid:
            lay = [M.layers[i] for i in idx]
            stacks = [dd.Stack(lay, M.ks(kc, idx), [M.xs(s)[i] for i in idx], [M.ys()[i] for i in idx], ws)
                      for s in range(2)]
            ms = bench.time_graphs(torch, None, [st.launch for st in stacks], a.reps, 3, stream, 1)
            table[c][n][kc] = 1e3 * ms / len(idx)
            for st in stacks:
                st.close()
        print(c, n, {k: round(v, 2) for k, v in table[c][n].items()}, flush=True)
dd.decdec_set_dec_ctas(0)

classes = []
for c in names:
    m = next(mm for mm in M.meta if mm[1] == c)
    classes.append(tuner.LayerClass(c, 32, m[2], m[3]))  # 32 blocks per decode step
f = tuner.interp_table(table)
res = {"model": a.model, "bits": a.bits, "n_grid": ns, "k_grid": kgrid, "table_us": table, "tuned": {}}
for t in (float(v) for v in a.targets.split(",")):
    r = tuner.tune(classes, f, t, n_max_values=ns, n_candidates=lambda c: ns, k_max=max(kgrid), base_n=ns[0])
    res["tuned"][str(t)] = {"n_max": r.n_max, "n": r.n, "k_chunk": r.k_chunk, "base_us_per_step": r.base_us,
                            "us_per_step": r.us, "slowdown": r.slowdown, "table2": r.table2()}
    print(f"target {100 * t:5.1f}%  {r.table2()}   ({r.us:.1f} us/step vs {r.base_us:.1f})", flush=True)
os.makedirs(os.path.dirname(a.out), exist_ok=True)
with open(a.out, "w") as fh:
    json.dump(res, fh, indent=1)
