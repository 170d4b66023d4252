#!/usr/bin/env python
"""DecDEC decode-step benchmark (BASELINE.json metric: µs per decode linear layer & tokens/s vs
k_chunk; % of HBM+PCIe roofline), workload BASELINE.json configs[1]: Llama-3-8B decode, all
q/k/v/o/gate/up/down weights x 32 blocks, 3-bit W_hat (group 128) + 4-bit residual in pinned host
memory, exact Top-k per layer per step on outlier-heavy synthetic activations.

A "step" = one decode step's whole linear stack, called per the paper's layer classes qkv, o, gu,
d (q/k/v share x and so do gate/up, so they are one GEMV each) -- 128 layer calls, each =
exact Top-k selector + fused GEMV/zero-copy-gather/combine kernel -- replayed as one native CUDA
graph (decdec_stack_*), consecutive layers chained by programmatic dependent launch.
(--unfused: 224 separate q/k/v/o/gate/up/down calls.)  Inputs are resident in HBM when the timed
region starts; the step streams 2.8 GB of packed weights (> 126 MB L2), so no L2 flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--kchunk 21] [--sweep 0,8,21]
  python bench.py --impl reference ...      # the float64 CPU oracle, timed on host cores

N > 1 (torchrun): output-feature tensor parallelism: every rank holds the
d_out/N column shard of every layer (+ its own host residual slice) and y is assembled with an
NCCL all-gather after each layer (strong scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import MODEL_BLOCKS, gen_activations, layer_seed, model_layers  # noqa: E402

METRIC = "µs per decode linear layer & tokens/s vs k_chunk; % of HBM+PCIe roofline"
GROUP = 128


# The paper's own end-to-end results (Table 2): tuner output
# n_max / (k_qkv, k_o, k_gu, k_d) -> measured slowdown vs the uncompensated model, Llama-3-8B-Instruct
# 3-bit AWQ, per-token latency in a torch.compile pipeline.  Other hardware: context, not a target.
PAPER_SLOWDOWNS = {
    "source": "PAPER.md Table 2 (P:514-554), Llama-3-8B 3-bit AWQ, n_max/(k_qkv,k_o,k_gu,k_d) -> slowdown",
    "RTX 4090 (1008 GB/s HBM, 32 GB/s PCIe)": {"2.5%": "24/(4,4,8,9) -> 1.3%", "5%": "24/(5,7,9,10) -> 2.2%",
                                               "10%": "24/(10,11,11,11) -> 4.9%", "20%": "24/(15,15,16,15) -> 10.4%"},
    "RTX 4050 Mobile (192 GB/s, 16 GB/s PCIe)": {"2.5%": "8/(55,56,58,55) -> 1.7%", "5%": "8/(59,59,59,58) -> 3.3%",
                                                 "10%": "10/(62,62,62,62) -> 6.6%", "20%": "10/(70,70,68,68) -> 13.5%"},
    "this B200 (tools/tune.py)": "profiles/r01_tuner.json",
}


def k_of(kc: int, d_in: int) -> int:
    return (kc * d_in) // 1024  # ledger L3: k = floor(k_chunk * d_in / 1024)


def bytes_hbm(d_in, d_out, bits):
    """Algorithmic HBM bytes of one layer call: packed codes + fp16 s + u8 z + x + y."""
    return d_in * d_out * bits // 8 + (d_in // GROUP) * d_out * 3 + 2 * d_in + 2 * d_out


def bytes_pcie(k, d_out, r_bits=4):
    """Algorithmic PCIe bytes: k selected residual rows + every residual scale."""
    return 0 if k == 0 else k * d_out * r_bits // 8 + (2 * d_out if r_bits == 4 else 0)


def load_peaks():
    hbm, src = 6455.3, "MEASURED_PEAKS.json hbm_gbs"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
    except Exception:
        hbm, src = 6650.0, "fallback B200_PROFILING.md 6.65 TB/s"
    pcie, psrc = 51.4, "profiles/r01_probe_links.json zero-copy streaming read max"
    try:
        with open(os.path.join(ROOT, "profiles", "r01_probe_links.json")) as f:
            pj = json.load(f)
        pcie = max(c["GBps"] for c in pj["zc"])
    except Exception:
        pass
    return hbm, src, pcie, psrc


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.lines, self.proc = [], None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(gpu_index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [v.strip() for v in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------ model
class Model:
    """Llama-3-8B (or another model) decode linear stack on this rank."""

    def __init__(self, dd, torch, model, bits, rank, world, n_x_sets, device, fused=True, hosts=None, numa=-1,
                 shapes=None):
        """hosts: reuse another Model's host residual store (same shapes; the residual does not
        depend on the base bit width).  numa: NUMA node of the rank's residual slice."""
        self.layers, self.meta = [], []  # meta: (block, name, d_in, d_out_shard)
        self.hosts = []
        shapes = model_layers(model, fused=fused) if shapes is None else shapes
        self.n_blocks = MODEL_BLOCKS[model]
        for b in range(self.n_blocks):
            for name, d_in, d_out in shapes:
                d_out_r = d_out // world
                g = __import__("synth").gen_perf_layer_device(d_in, d_out_r, bits, layer_seed(model, b, name, rank),
                                                              device=device)
                row_bytes = d_out_r // 2
                sc_off = (d_in * row_bytes + 255) // 256 * 256
                if hosts is not None:
                    hb = hosts[len(self.hosts)]
                else:
                    hb = dd.HostBuffer(sc_off + 2 * d_out_r, numa)
                    hv = torch.from_numpy(hb.numpy(np.uint8))
                    hv[: d_in * row_bytes].copy_(g["r"].cpu())
                    hv[sc_off: sc_off + 2 * d_out_r].copy_(g["rS"].view(torch.uint8).cpu())
                del g["r"]
                lin = dd.QuantLinear.from_device_packed(d_in, d_out_r, bits, g["w"], g["s"], g["z"], host=hb,
                                                        r_bits=4, host_scales_off=sc_off)
                self.layers.append(lin)
                self.meta.append((b, name, d_in, d_out_r))
                self.hosts.append(hb)
        # activations: n_x_sets distinct decode steps, one contiguous fp16 arena per set
        self.x_off = np.cumsum([0] + [m[2] for m in self.meta])
        self.y_off = np.cumsum([0] + [m[3] for m in self.meta])
        self.x_host = []
        for sset in range(n_x_sets):
            parts = [gen_activations(d_in, 1, seed=layer_seed(model, b, name, "x", sset),
                                     kind="d" if name in ("down", "d") else "qkv")[0]
                     for (b, name, d_in, _) in self.meta]
            self.x_host.append(np.concatenate(parts))
        self.x_dev = [torch.from_numpy(h).to(device) for h in self.x_host]
        self.y_dev = torch.empty(int(self.y_off[-1]), dtype=torch.float16, device=device)
        self.max_d_out = max(m[3] for m in self.meta)
        self.max_d_in = max(m[2] for m in self.meta)

    def xs(self, sset):
        return [self.x_dev[sset][int(self.x_off[i]): int(self.x_off[i + 1])] for i in range(len(self.meta))]

    def ys(self):
        return [self.y_dev[int(self.y_off[i]): int(self.y_off[i + 1])] for i in range(len(self.meta))]

    def ks(self, kc, idx=None):
        idx = range(len(self.meta)) if idx is None else idx
        return [k_of(kc, self.meta[i][2]) for i in idx]


def time_graphs(torch, dist, launches, K, W, stream, world):
    """W warm-up replays then EXACTLY K timed replays (round-robin over `launches`),
    barrier + synchronize on both sides, CUDA events on the launching stream, max over ranks."""
    for i in range(W):
        launches[i % len(launches)]()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(K):
        launches[i % len(launches)]()
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    return ms


def time_shapes(torch, dist, dd, M, ws, sweep, steps, stream, world, bits, hbm_peak, pcie_peak, names=None):
    """µs per layer call of each shape: a graph of the model's n_blocks instances of that shape
    (distinct weights, PDL-chained), per k_chunk; with HBM/PCIe achieved GB/s and roofline fraction."""
    shape_names = []
    for (_, name, _, _) in M.meta:
        if name not in shape_names and (names is None or name in names):
            shape_names.append(name)
    per_shape = {}
    for name in shape_names:
        idx = [i for i, m in enumerate(M.meta) if m[1] == name]
        d_in, d_out = M.meta[idx[0]][2], M.meta[idx[0]][3]
        per_shape[name] = {"d_in": d_in, "d_out": d_out}
        for kc in sweep:
            lay = [M.layers[i] for i in idx]
            xs = [M.xs(s) for s in range(len(M.x_dev))]
            stacks = [dd.Stack(lay, M.ks(kc, idx), [xs[s][i] for i in idx], [M.ys()[i] for i in idx], ws)
                      for s in range(len(M.x_dev))]
            ms = time_graphs(torch, dist, [st.launch for st in stacks], max(8, steps // 4), 3, stream, world)
            us = 1e3 * ms / len(idx)
            k = k_of(kc, d_in)
            bh, bp = bytes_hbm(d_in, d_out, bits), bytes_pcie(k, d_out)
            t_roof = max(bh / (hbm_peak * 1e3), bp / (pcie_peak * 1e3))  # µs
            per_shape[name][str(kc)] = {"us": round(us, 3), "k": k, "hbm_GBps": round(bh / us / 1e3, 1),
                                        "pcie_GBps": round(bp / us / 1e3, 2), "roofline_us": round(t_roof, 3),
                                        "roofline_frac": round(t_roof / us, 3),
                                        "hbm_frac": round(bh / us / 1e3 / hbm_peak, 3)}
            for st in stacks:
                st.close()
    return per_shape


def step_sweep(torch, dist, dd, M, ws, sweep, steps, warmup, stream, world, comm=None, peers=None):
    """tokens/s of the whole decode step (all layers, one CUDA graph per activation set) per k_chunk.
    TP: peers -> fused P2P-store all-gather in every layer kernel (P2PStack); comm -> NCCL."""
    out = {}
    for kc in sweep:
        if peers is not None:
            offs, _ = dd.peer_offsets([m[3] for m in M.meta], world)
            stacks = [dd.P2PStack(M.layers, M.ks(kc), M.xs(s), offs, ws, peers) for s in range(len(M.x_dev))]
        elif comm is None:
            stacks = [dd.Stack(M.layers, M.ks(kc), M.xs(s), M.ys(), ws) for s in range(len(M.x_dev))]
        else:
            full = [torch.empty(m[3] * world, dtype=torch.float16, device="cuda") for m in M.meta]
            stacks = [dd.TPStack(M.layers, M.ks(kc), M.xs(s), full, ws, comm) for s in range(len(M.x_dev))]
        ms = time_graphs(torch, dist, [st.launch for st in stacks], steps, max(warmup, 3), stream, world)
        out[kc] = {"ms_per_step": ms, "tokens_per_s": 1e3 / ms, "kernels_per_step": stacks[0].kernels}
        for st in stacks:
            st.close()
    return out


def knee(results, bits, hbm_peak, pcie_peak, limit=1.10):
    """Measured knee: the largest swept k_chunk whose step time is <= limit x the k_chunk-0 step,
    next to the paper's prediction k_chunk = 1024 / R_bw * b / 4 (R_bw = HBM / PCIe BW)."""
    if 0 not in results:
        return None
    base = results[0]["ms_per_step"]
    ok = [kc for kc in sorted(results) if results[kc]["ms_per_step"] <= limit * base]
    r_bw = hbm_peak / pcie_peak
    return {"limit": limit, "measured_k_chunk": max(ok) if ok else 0,
            "predicted_k_chunk_P384": round(1024.0 / r_bw * bits / 4.0, 2), "R_bw": round(r_bw, 1),
            "note": "paper knee formula (P:384) with the measured HBM copy and zero-copy PCIe bandwidths"}


def cpu_oracle_block(model, bits, kc, fused=True, seed_tag="cpu"):
    """Time the oracle (as it stands) on one decoder block's layers (a bounded sample)."""
    import oracle
    from synth import gen_perf_layer

    shapes = model_layers(model, fused=fused)
    data = []
    for name, d_in, d_out in shapes:
        L = gen_perf_layer(d_in, d_out, bits, seed=layer_seed(seed_tag, name))
        x = gen_activations(d_in, 1, seed=layer_seed(seed_tag, name, "x"), kind="d" if name in ("down", "d") else "qkv")[0]
        data.append((name, d_in, L, x))
    times = {}
    for name, d_in, L, x in data:
        t0 = time.perf_counter()
        oracle.decdec_linear_ref(L["q"], L["s"], L["z"], x, k_of(kc, d_in), rc=L["rc"], rS=L["rS"])
        times[name] = time.perf_counter() - t0
    return times


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:
        return len(os.sched_getaffinity(0))


# ------------------------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """The float64 CPU oracle, as it stands, on the host cores (tier: the oracle IS the reference)."""
    if rank != 0:
        return
    import oracle
    from synth import gen_perf_layer

    model, bits, kc = args.model, args.bits, args.kchunk
    shapes = model_layers(model, fused=not args.unfused)
    data = []
    for name, d_in, d_out in shapes:
        L = gen_perf_layer(d_in, d_out, bits, seed=layer_seed("ref", name))
        X = gen_activations(d_in, 2, seed=layer_seed("ref", name, "x"), kind="d" if name in ("down", "d") else "qkv")
        data.append((name, d_in, d_out, L, X))
    per = {n: [] for n, *_ in data}

    def step(i):
        name, d_in, d_out, L, X = data[i % len(data)]
        t0 = time.perf_counter()
        oracle.decdec_linear_ref(L["q"], L["s"], L["z"], X[i % 2], k_of(kc, d_in), rc=L["rc"], rS=L["rS"])
        return name, time.perf_counter() - t0

    for i in range(args.warmup):
        step(i)
    t_all = time.perf_counter()
    for i in range(args.steps):
        n, t = step(i)
        per[n].append(t)
    t_all = time.perf_counter() - t_all
    # layer time per shape (extrapolate unmeasured shapes by weight bytes)
    meas = {n: float(np.mean(v)) for n, v in per.items() if v}
    bpl = {n: d_in * d_out for n, d_in, d_out, _, _ in data}
    rate = np.mean([meas[n] / bpl[n] for n in meas])
    block = sum(meas.get(n, rate * bpl[n]) for n in bpl)
    tok_s = 1.0 / (MODEL_BLOCKS[model] * block)
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": tok_s, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / max(args.steps, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{model} decode linear stack, w{bits} g128 + r4 residual, k_chunk={kc} "
                               "(each step = one layer call of one block, shapes cycled)", "k_chunk": kc},
        "cpu_baseline": {"value": tok_s, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                         "sample": f"{args.steps} single-layer oracle calls cycling the block's shapes; "
                                   f"tokens/s = 1/({MODEL_BLOCKS[model]} x sum_shape mean layer time)"},
        "e2e": {"value": tok_s, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "per_layer_s": meas,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------ main arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="decdec", choices=["decdec", "reference"])
    ap.add_argument("--model", default="llama3_8b")
    ap.add_argument("--bits", type=int, default=3)
    ap.add_argument("--kchunk", type=int, default=21, help="headline k_chunk (21 = 2.05%% of channels)")
    ap.add_argument("--sweep", default="0,1,2,4,6,8,12,16,21,32,48,64,82",
                    help="k_chunk sweep (µs/layer per shape + tokens/s); SURVEY §8(d) config 2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nx", type=int, default=4, help="distinct activation sets cycled across steps")
    ap.add_argument("--quick", action="store_true", help="headline step only (for ncu launch lists)")
    ap.add_argument("--sweep-only", action="store_true", help="decode-step sweep only (no per-shape table, no oracle)")
    ap.add_argument("--tp-comm", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: assemble y with the fused P2P-store all-gather (default) or NCCL")
    ap.add_argument("--shard-of", type=int, default=1,
                    help="single GPU: run rank 0's output-feature shard of a P-way TP model (d_out/P per layer, "
                         "its own host residual slice); per-rank time, all-gather NOT included (config 4/5 evidence)")
    ap.add_argument("--unfused", action="store_true",
                    help="7 separate q/k/v/o/gate/up/down calls per block instead of the paper's layer "
                         "classes qkv, o, gu, d (P:304).  Without it the per-layer table still carries the 7 "
                         "unfused shapes (per_layer_us_unfused: k/v and gate/up timed on their own instances, "
                         "q = o and down = d shapes)")
    ap.add_argument("--no-w4", action="store_true", help="skip the 4-bit (config 3) sub-object")
    ap.add_argument("--no-unfused-extra", action="store_true", help="skip timing the k/v and gate/up shapes")
    ap.add_argument("--no-lut", action="store_true", help="skip the non-uniform (LUT) base sub-object (NEXT-3)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2412_20185_b200 as dd

    # DECDEC_BENCH_SHARE_GPU=1 (tests only): every rank on GPU 0 over gloo -- exercises the N > 1
    # code path (fused P2P all-gather between processes) on a one-GPU box; its timings are not
    # bench numbers (the driver time-slices the ranks' kernels)
    share = os.environ.get("DECDEC_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = "cuda"
    stream = torch.cuda.current_stream()
    hbm_peak, hbm_src, pcie_peak, pcie_src = load_peaks()

    t_build = time.time()
    shard = world if world > 1 else max(1, args.shard_of)
    numa = dd.numa_node_of_device(local)  # the rank's residual slice sits in front of its own PCIe link
    M = Model(dd, torch, args.model, args.bits, rank, shard, args.nx, dev, fused=not args.unfused, numa=numa)
    sweep = sorted({int(v) for v in args.sweep.split(",") if v != ""} | {args.kchunk})
    if args.quick:
        sweep, args.no_cpu_baseline = [args.kchunk], True
    if args.sweep_only:
        args.no_cpu_baseline = True
    max_k = k_of(max(sweep), M.max_d_in)
    ws = dd.Workspace(max_k, M.max_d_out)
    torch.cuda.synchronize()
    t_build = time.time() - t_build
    n_layers = len(M.meta)
    comm = peers = None
    tp_comm = None
    if world > 1:
        # the y assembly: fused P2P-store all-gather in the layer kernels (default), or the
        # library-owned NCCL communicator's all-gather after each layer kernel
        if args.tp_comm == "p2p":
            err = ""
            try:
                peers = dd.Peers(dd.peer_offsets([m[3] for m in M.meta], world)[1])
            except Exception as e:  # no peer access between the GPUs: NCCL instead, said so in the line
                peers, err = None, str(e)[:80]
            ok = torch.tensor([1 if peers is not None else 0], device="cuda")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)  # every rank takes the same path
            if int(ok.item()) == 0:
                if peers is not None:
                    peers.close()
                peers = None
                tp_comm = f"nccl (p2p unavailable: {err or 'on another rank'})"
            else:
                tp_comm = "p2p (fused all-gather in the layer kernels, CUDA-IPC peer stores over NVLink)"
        if peers is None:
            comm = dd.Comm()
            tp_comm = tp_comm or "nccl (in-place all-gather after each layer kernel)"

    # ---- full decode-step graphs per k_chunk (clocks sampled over all timed regions) ---------
    sampler = ClockSampler(local) if rank == 0 else None
    results = step_sweep(torch, dist, dd, M, ws, sweep, args.steps, args.warmup, stream, world, comm, peers)
    clocks = sampler.stop() if sampler is not None else None
    headline = (results[args.kchunk]["ms_per_step"], results[args.kchunk]["kernels_per_step"])

    # ---- per-shape µs per layer (graph of the n_blocks instances of one shape) --------------
    per_shape, per_unfused, w4 = {}, None, None
    if not (args.quick or args.sweep_only):  # per rank under TP: the rank's shards, no collective
        per_shape = time_shapes(torch, dist, dd, M, ws, sweep, args.steps, stream, world, args.bits, hbm_peak,
                                pcie_peak)
        if not args.unfused and args.model == "llama3_8b" and not args.no_unfused_extra:
            # the 7 unfused shapes: q = o and down = d shapes (timed above); k/v and gate/up on their
            # own n_blocks instances
            from synth import SHAPES
            extra = [(n, *SHAPES[args.model][n]) for n in ("k", "gate")]
            MX = Model(dd, torch, args.model, args.bits, rank, shard, args.nx, dev, shapes=extra, numa=numa)
            wsx = dd.Workspace(k_of(max(sweep), MX.max_d_in), MX.max_d_out)
            px = time_shapes(torch, dist, dd, MX, wsx, sweep, args.steps, stream, world, args.bits, hbm_peak,
                             pcie_peak)
            per_unfused = {"q": per_shape["o"], "k": px["k"], "v": px["k"], "o": per_shape["o"],
                           "gate": px["gate"], "up": px["gate"], "down": per_shape["d"],
                           "_note": "same-shape pairs timed once: q = o (4096x4096), v = k (4096x1024), "
                                    "up = gate (4096x14336), down = d (14336x4096)"}
            del MX, wsx
        if not args.no_w4 and args.bits == 3 and world == 1:
            # config 3: the same stack with 4-bit base weights (the residual store is shared)
            M4 = Model(dd, torch, args.model, 4, rank, shard, args.nx, dev, fused=not args.unfused, hosts=M.hosts,
                       numa=numa)
            w4_sweep = sorted({0, 4, 8, args.kchunk})
            r4 = step_sweep(torch, dist, dd, M4, ws, w4_sweep, args.steps, args.warmup, stream, world)
            w4 = {"config": "BASELINE configs[2]: Llama-3-8B 4-bit (W4K, g128 fp16 s + u8 z) + r4 residual",
                  "sweep": {str(k): {"tokens_per_s": round(v["tokens_per_s"], 2), "ms_per_step": round(v["ms_per_step"], 4),
                                     "slowdown_vs_k0": round(v["ms_per_step"] / r4[0]["ms_per_step"], 4)}
                            for k, v in r4.items()},
                  "knee": knee(r4, 4, hbm_peak, pcie_peak),
                  "per_layer_us": time_shapes(torch, dist, dd, M4, ws, [0, args.kchunk], args.steps, stream, world, 4,
                                              hbm_peak, pcie_peak)}
            del M4

    # ---- NEXT-3: the same stack with a non-uniform (LUT) base: k_chunk 0 (k_gemv16) and the
    # headline k_chunk (fused kernel with the LUT base + compensation, same host residual) -----
    lut = None
    if not (args.quick or args.sweep_only or args.no_lut) and world == 1:
        from synth import gen_perf_layer_lut_device
        lut = {"config": "Llama-3-8B, SqueezeLLM-style per-column fp16 table of 2^b entries (P:397, P:502), "
                         f"W4K nibble codes; k_chunk 0 (base GEMV, k_gemv16) and {args.kchunk} (fused kernel, "
                         "LUT base + r4 compensation from the same host residual store)"}
        lut_sweep = sorted({0, args.kchunk})
        for lb in (3, 4):
            ML = Model.__new__(Model)
            ML.layers, ML.meta, ML.hosts, ML.n_blocks = [], [], M.hosts, M.n_blocks
            for li, (b, name, d_in, d_out) in enumerate(M.meta):
                g = gen_perf_layer_lut_device(d_in, d_out, lb, layer_seed("lut", args.model, b, name))
                ML.layers.append(dd.QuantLinear.from_device_lut(d_in, d_out, lb, g["w"], g["lut"], host=M.hosts[li],
                                                                host_scales_off=M.layers[li].host_scales_off))
                ML.meta.append((b, name, d_in, d_out))
            ML.x_off, ML.y_off, ML.x_host, ML.x_dev, ML.y_dev = M.x_off, M.y_off, M.x_host, M.x_dev, M.y_dev
            ML.max_d_out, ML.max_d_in = M.max_d_out, M.max_d_in
            rl = step_sweep(torch, dist, dd, ML, ws, lut_sweep, args.steps, args.warmup, stream, world)
            # bytes per call: 4-bit codes + fp16 table of 2^b per row + x + y (+ PCIe as the uniform base)
            per = time_shapes(torch, dist, dd, ML, ws, lut_sweep, args.steps, stream, world, 4, hbm_peak, pcie_peak)
            for n_, v_ in per.items():
                d_in, d_out = v_["d_in"], v_["d_out"]
                bh = d_in * d_out // 2 + d_out * (2 << lb) + 2 * d_in + 2 * d_out
                for key, e0 in v_.items():
                    if not isinstance(e0, dict):
                        continue
                    bp = (e0["k"] * d_out // 2 + 2 * d_out) if e0["k"] else 0
                    t_roof = max(bh / (hbm_peak * 1e3), bp / (pcie_peak * 1e3))
                    e0["hbm_GBps"] = round(bh / e0["us"] / 1e3, 1)
                    e0["roofline_us"] = round(t_roof, 3)
                    e0["roofline_frac"] = round(t_roof / e0["us"], 3)
                    e0["hbm_frac"] = round(bh / (hbm_peak * 1e3) / e0["us"], 3)
            lut[f"b{lb}"] = {"sweep": {str(k): {"tokens_per_s": round(v["tokens_per_s"], 2), "ms_per_step": round(v["ms_per_step"], 4)}
                                       for k, v in rl.items()},
                             "tokens_per_s": round(rl[0]["tokens_per_s"], 2), "ms_per_step": round(rl[0]["ms_per_step"], 4),
                             "per_layer_us": per}
            del ML

    # ---- e2e through the public API: H2D inputs + step + D2H outputs ------------------------
    e2e = None
    if world == 1 and not (args.quick or args.sweep_only):
        x_pinned = [torch.from_numpy(h).pin_memory() for h in M.x_host]
        y_pinned = torch.empty(M.y_dev.numel(), dtype=torch.float16).pin_memory()
        stack = dd.Stack(M.layers, M.ks(args.kchunk), M.xs(0), M.ys(), ws)

        def e2e_step_factory(i):
            def f():
                M.x_dev[0].copy_(x_pinned[i % len(x_pinned)], non_blocking=True)
                stack.launch()
                y_pinned.copy_(M.y_dev, non_blocking=True)
            return f
        ms_e2e = time_graphs(torch, dist, [e2e_step_factory(i) for i in range(args.nx)], args.steps,
                             max(args.warmup, 3), stream, world)
        e2e = {"value": 1e3 / ms_e2e, "unit": "tokens/s", "h2d_bytes_per_step": int(M.x_dev[0].numel() * 2),
               "d2h_bytes_per_step": int(M.y_dev.numel() * 2), "ms_per_step": ms_e2e,
               "api": "paper_2412_20185_b200.Stack (decdec_stack_launch) + pinned H2D/D2H copies"}
        stack.close()

    # ---- roofline of the dominant kernel ------------------------------------------------------
    ms_head, kernels_head = headline
    step_hbm = sum(bytes_hbm(m[2], m[3], args.bits) for m in M.meta)
    step_pcie = sum(bytes_pcie(k_of(args.kchunk, m[2]), m[3]) for m in M.meta)
    t_roof_step = sum(max(bytes_hbm(m[2], m[3], args.bits) / (hbm_peak * 1e6),
                          bytes_pcie(k_of(args.kchunk, m[2]), m[3]) / (pcie_peak * 1e6)) for m in M.meta)  # ms
    roofline = None
    if per_shape:
        dom = max(per_shape, key=lambda n: per_shape[n][str(args.kchunk)]["us"] *
                  sum(1 for m in M.meta if m[1] == n))
        e = per_shape[dom][str(args.kchunk)]
        d_in, d_out = per_shape[dom]["d_in"], per_shape[dom]["d_out"]
        bh, bp = bytes_hbm(d_in, d_out, args.bits), bytes_pcie(e["k"], d_out)
        pcie_bound = bp / pcie_peak > bh / hbm_peak
        ach = (bp if pcie_bound else bh) / e["us"] / 1e3
        peak = pcie_peak if pcie_bound else hbm_peak
        traffic = None
        if shard == 1 and args.model == "llama3_8b" and args.bits == 3:  # the captured layer's shape only
            try:
                with open(os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")) as f:
                    traffic = json.load(f).get(f"{dom}/{args.kchunk}")
            except Exception:
                pass
        roofline = {
            "bound": "pcie" if pcie_bound else "hbm", "achieved": round(ach, 2), "peak": peak, "unit": "GB/s",
            "frac": round(ach / peak, 4), "traffic": traffic,
            "kernel": f"select + k_linear<{args.bits},4> on {dom} ({d_in}x{d_out}), k={e['k']}",
            "algorithmic_bytes": {"hbm": bh, "pcie": bp},
            "hbm_frac": round(bh / e["us"] / 1e3 / hbm_peak, 4), "pcie_frac": round(bp / e["us"] / 1e3 / pcie_peak, 4),
            "layer_roofline_frac": e["roofline_frac"],
            "peak_source": {"hbm": hbm_src, "pcie": pcie_src},
            "step_roofline_ms": round(t_roof_step, 4), "step_roofline_frac": round(t_roof_step / ms_head, 4),
        }

    # ---- CPU baseline (oracle on host cores, rank 0, N = 1) ----------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        times = cpu_oracle_block(args.model, args.bits, args.kchunk, fused=not args.unfused)
        blk = sum(times.values())
        cpu = {"value": 1.0 / (M.n_blocks * blk), "unit": "tokens/s", "cores": blas_threads(), "kind": "oracle",
               "sample": f"one decoder block ({', '.join(times)}) through oracle.decdec_linear_ref at "
                         f"k_chunk={args.kchunk}, x {M.n_blocks} blocks; {blk:.1f} s of CPU work",
               "per_layer_s": {k: round(v, 3) for k, v in times.items()}}
        # also one thread, and the host it ran on
        try:
            from threadpoolctl import threadpool_limits
            with threadpool_limits(limits=1):
                t1 = cpu_oracle_block(args.model, args.bits, args.kchunk, fused=not args.unfused)
            cpu["value_1thread"] = 1.0 / (M.n_blocks * sum(t1.values()))
        except Exception as e:  # threadpoolctl missing: report why
            cpu["value_1thread"] = None
            cpu["value_1thread_error"] = str(e)[:120]
        cpu["affinity_cpus"] = len(os.sched_getaffinity(0))
        try:
            info = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
            get = lambda key: next((ln.split(":", 1)[1].strip() for ln in info.splitlines() if ln.startswith(key)), None)  # noqa: E731
            cpu["host_cpu"] = {"model": get("Model name"), "sockets": get("Socket(s)")}
        except Exception:
            pass

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(1e3 / ms_head, 2), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms_head, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": f"int{args.bits} weights x f16 activations -> f32 accumulate (f16 out); int4 residual",
            "data": "synthetic (seeded; random packed codes, outlier-heavy Student-t activations)",
            "config": {"workload": f"{args.model} decode linear stack: {n_layers // M.n_blocks} layer calls "
                                   f"({'q,k,v,o,gate,up,down' if args.unfused else 'qkv,o,gu,d classes, P:304'}) x "
                                   f"{M.n_blocks} blocks, w{args.bits} g128, r4 residual in pinned host memory, "
                                   f"exact Top-k, k_chunk={args.kchunk}",
                       "k_chunk": args.kchunk, "layers_per_step": n_layers,
                       "parallelism": (f"tp{world} (output-feature shards; y assembly: {tp_comm})" if world > 1 else
                                       f"single GPU running rank 0's 1/{shard} output-feature shard (all-gather not included)"
                                       if shard > 1 else "single GPU"),
                       "l2": f"inputs larger than L2: {step_hbm / 1e9:.2f} GB weights streamed per step",
                       "x_sets": args.nx},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": kernels_head * args.steps,
            "clocks": clocks,
            "paper_context": PAPER_SLOWDOWNS,
            "sweep": {str(k): {"tokens_per_s": round(v["tokens_per_s"], 2), "ms_per_step": round(v["ms_per_step"], 4),
                               "slowdown_vs_k0": round(v["ms_per_step"] / results[0]["ms_per_step"], 4)
                               if 0 in results else None}
                      for k, v in results.items()},
            "knee": knee(results, args.bits, hbm_peak, pcie_peak),
            "per_layer_us": per_shape,
            "per_layer_us_unfused": per_unfused,
            "w4": w4,
            "lut": lut,
            "step_bytes": {"hbm": step_hbm, "pcie": step_pcie},
            "build_s": round(t_build, 1),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
