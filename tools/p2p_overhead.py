"""Cost of the fused P2P all-gather machinery on ONE rank (no NVLink traffic): the Llama-3-8B
decode stack as a plain Stack vs a P2PStack over a 1-rank peer group (every output store goes
through the peer path, every CTA releases a count, the leader CTA acquires them, launches are
cooperative).  Prints one JSON line with ms per step for k_chunk 0 and 21.
usage: python tools/p2p_overhead.py [--steps 30]"""
import argparse
import json
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2412_20185_b200 as dd  # noqa: E402
from synth import gen_activations, gen_perf_layer_device, layer_seed, model_layers  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--blocks", type=int, default=32)
a = ap.parse_args()
with socket.socket() as so:
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
layers, hosts, xs, meta = [], [], [], []
for b in range(a.blocks):
    for name, d_in, d_out in model_layers("llama3_8b", fused=True):
        g = gen_perf_layer_device(d_in, d_out, 3, layer_seed("p2pov", b, name))
        rb = d_out // 2
        off = (d_in * rb + 255) // 256 * 256
        hb = dd.HostBuffer(off + 2 * d_out)
        hv = torch.from_numpy(hb.numpy(np.uint8))
        hv[: d_in * rb].copy_(g["r"].cpu())
        hv[off: off + 2 * d_out].copy_(g["rS"].view(torch.uint8).cpu())
        layers.append(dd.QuantLinear.from_device_packed(d_in, d_out, 3, g["w"], g["s"], g["z"], host=hb, r_bits=4,
                                                        host_scales_off=off))
        hosts.append(hb)
        xs.append(torch.from_numpy(gen_activations(d_in, 1, seed=len(xs), kind="d" if name == "d" else "qkv")[0]).cuda())
        meta.append((d_in, d_out))
ws = dd.Workspace(max(21 * d // 1024 for d, _ in meta), max(o for _, o in meta))
ys = [torch.empty(o, dtype=torch.float16, device="cuda") for _, o in meta]
offs, total = dd.peer_offsets([o for _, o in meta], 1)
peers = dd.Peers(total)


def timed(launch, steps):
    for _ in range(5):
        launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        launch()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


out = {"what": "Llama-3-8B 3-bit decode stack (128 layer calls), plain Stack vs P2PStack on a 1-rank peer group",
       "ms_per_step": {}}
for kc in (0, 21):
    ks = [kc * d // 1024 for d, _ in meta]
    st = dd.Stack(layers, ks, xs, ys, ws)
    ps = dd.P2PStack(layers, ks, xs, offs, ws, peers)
    r = {}
    for rep in range(2):
        r.setdefault("stack", []).append(round(timed(st.launch, a.steps), 4))
        r.setdefault("p2p_stack", []).append(round(timed(ps.launch, a.steps), 4))
    y_ok = all(torch.equal(y, yf) for y, yf in zip(ys, ps.y_full))
    r["outputs_bit_identical"] = bool(y_ok)
    out["ms_per_step"][str(kc)] = r
    st.close()
    ps.close()
print(json.dumps(out), flush=True)
peers.close()
dist.destroy_process_group()
