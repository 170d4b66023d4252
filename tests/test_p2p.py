"""Fused P2P-store all-gather (include/decdec.h decdec_peers): two
ranks, separate processes, each holding its output-column shard.  decdec_linear_p2p and the
P2P step executor (P2PStack) must leave, in EVERY rank's y_full, the full y of the UNSHARDED
oracle (L9), bit-identical across ranks, over repeated calls and graph replays (slot reuse).

The ranks share GPU 0 when the box has one GPU (their region is opened through CUDA IPC as a
second mapping of the same memory; the driver time-slices the two processes' kernels), and use
GPUs 0 and 1 otherwise (NVLink peer stores)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (d_in, d_out, k): config 1 (P:1024x1024, k = 16) and a Llama-3-8B o layer at k_chunk 0 / 21
CASES = [(1024, 1024, 16), (1024, 1024, 0), (4096, 4096, 84), (4096, 4096, 0)]


def _worker(rank, world, port, out_dir, multi_gpu):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2412_20185_b200 as dd
    from paper_2412_20185_b200.tp import peer_offsets, shard_codes
    from synth import gen_activations, gen_perf_layer, layer_seed

    torch.cuda.set_device(rank if multi_gpu else 0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    lins, xs, ks = [], [], []
    for i, (d_in, d_out, k) in enumerate(CASES):
        L = gen_perf_layer(d_in, d_out, 3, seed=layer_seed("p2p", d_in, d_out))
        Sh = shard_codes(L, rank, world)
        lins.append(dd.QuantLinear.from_codes(Sh["q"], Sh["s"], Sh["z"], 3, rc=Sh["rc"], rS=Sh["rS"]))
        xs.append(torch.from_numpy(gen_activations(d_in, 1, seed=layer_seed("p2p", "x", i))[0]).cuda())
        ks.append(k)
    # two copies of the y_full layout: one for the per-call API, one for the step executor
    offs, total = peer_offsets([d for _, d, _ in CASES] * 2, world)
    peers = dd.Peers(total)
    ws = dd.Workspace(max(ks), max(d for _, d, _ in CASES) // world)
    out = {}
    try:
        for rep in range(2):  # the same slots twice: the counters reset
            for i in range(len(CASES)):
                y = dd.P2PLinear(lins[i], peers, offs[i], slot=i)(xs[i], ks[i], workspace=ws)
                torch.cuda.synchronize()
                out[f"call{rep}_{i}"] = y.cpu().numpy()
        n = len(CASES)
        st = dd.P2PStack(lins, ks, xs, offs[n:], ws, peers)
        for rep in range(3):
            for y in st.y_full:
                y.fill_(0)
            torch.cuda.synchronize()
            dist.barrier()  # nobody's replay may write into a y_full another rank is still zeroing
            st.launch()
            torch.cuda.synchronize()
            for i, y in enumerate(st.y_full):
                out[f"stack{rep}_{i}"] = y.cpu().numpy()
            dist.barrier()
        st.close()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **out)
    finally:
        peers.close()
        dist.destroy_process_group()


def _run(tmp_path, multi_gpu):
    import torch.multiprocessing as mp

    import oracle
    from synth import gen_activations, gen_perf_layer, layer_seed

    world = 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.start_processes(_worker, args=(world, port, str(tmp_path), multi_gpu), nprocs=world, join=False,
                             start_method="spawn")
    import time

    t0 = time.time()
    while not ctx.join(timeout=5):
        if time.time() - t0 > 600:
            for p in ctx.processes:
                p.kill()
            raise AssertionError("P2P ranks did not finish in 600 s")
    outs = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    for i, (d_in, d_out, k) in enumerate(CASES):
        L = gen_perf_layer(d_in, d_out, 3, seed=layer_seed("p2p", d_in, d_out))
        x = gen_activations(d_in, 1, seed=layer_seed("p2p", "x", i))[0]
        ref = oracle.decdec_linear_ref(L["q"], L["s"], L["z"], x, k, rc=L["rc"], rS=L["rS"])
        y0 = outs[0][f"call0_{i}"]
        ok, err, bound = oracle.tolerance_ok(y0, ref["y64"], ref["A"])
        assert ok.all(), (i, int((~ok).sum()))
        for r in range(world):
            for key in [f"call{j}_{i}" for j in range(2)] + [f"stack{j}_{i}" for j in range(3)]:
                assert np.array_equal(outs[r][key].view(np.uint16), y0.view(np.uint16)), (i, r, key)


def test_p2p_allgather_two_ranks_same_gpu(tmp_path):
    _run(tmp_path, multi_gpu=False)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_p2p_allgather_two_gpus(tmp_path):
    _run(tmp_path, multi_gpu=True)


def test_bench_two_ranks_fused_allgather_path():
    """bench.py under torchrun with 2 ranks (sharing GPU 0, DECDEC_BENCH_SHARE_GPU=1) takes the
    fused P2P all-gather path end to end and prints its JSON line (timings are not bench numbers:
    the two processes' kernels are time-sliced)."""
    import json
    import subprocess
    import sys

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ, DECDEC_BENCH_SHARE_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "3", "--warmup", "3", "--sweep", "0,21", "--sweep-only"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and "p2p" in line["config"]["parallelism"], line["config"]
    assert set(line["sweep"]) == {"0", "21"}


# ------------------------------------------------------------------ NEXT-4: multi-link residual fetch
ML_CASES = [(1024, 1024, 16), (4096, 4096, 84), (4096, 28672, 84), (14336, 4096, 294), (4096, 4096, 0)]


def _ml_worker(rank, world, port, out_dir, multi_gpu):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2412_20185_b200 as dd
    from synth import gen_activations, gen_perf_layer, layer_seed

    torch.cuda.set_device(rank if multi_gpu else 0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    offs, o = [], 0
    for _, d_out, _ in ML_CASES:
        offs.append(o)
        o += dd.MLLinear.area_bytes(d_out, world)
    peers = dd.Peers(o)
    out = {}
    try:
        for i, (d_in, d_out, k) in enumerate(ML_CASES):
            L = gen_perf_layer(d_in, d_out, 3, seed=layer_seed("ml", d_in, d_out))  # every rank: the full layer
            lin = dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 3, rc=L["rc"], rS=L["rS"])
            ml = dd.MLLinear(lin, peers, offs[i])
            ws = dd.Workspace(max(k, 1), d_out)
            for rep in range(3):  # the same ml area again and again: the flag / ack handshake
                x = gen_activations(d_in, 1, seed=layer_seed("ml", "x", i, rep), kind="d" if d_in > 8192 else "qkv")[0]
                sel = torch.empty(max(k, 1), dtype=torch.int32, device="cuda")
                y = ml(torch.from_numpy(x).cuda(), k, sel=sel, workspace=ws)
                torch.cuda.synchronize()
                if rank == 0:
                    out[f"y{i}_{rep}"] = y.cpu().numpy()
                    out[f"s{i}_{rep}"] = sel.cpu().numpy()[:k]
        dist.barrier()
        if rank == 0:
            np.savez(os.path.join(out_dir, "ml_rank0.npz"), **out)
    finally:
        peers.close()
        dist.destroy_process_group()


def _run_ml(tmp_path, multi_gpu):
    import time

    import torch.multiprocessing as mp

    import oracle
    from synth import gen_activations, gen_perf_layer, layer_seed

    world = 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.start_processes(_ml_worker, args=(world, port, str(tmp_path), multi_gpu), nprocs=world, join=False,
                             start_method="spawn")
    t0 = time.time()
    while not ctx.join(timeout=5):
        if time.time() - t0 > 600:
            for p in ctx.processes:
                p.kill()
            raise AssertionError("multi-link ranks did not finish in 600 s")
    out = np.load(os.path.join(tmp_path, "ml_rank0.npz"))
    for i, (d_in, d_out, k) in enumerate(ML_CASES):
        L = gen_perf_layer(d_in, d_out, 3, seed=layer_seed("ml", d_in, d_out))
        W_hat = oracle.dequantize_base(L["q"], L["s"], L["z"])
        for rep in range(3):
            x = gen_activations(d_in, 1, seed=layer_seed("ml", "x", i, rep), kind="d" if d_in > 8192 else "qkv")[0]
            ref = oracle.decdec_linear_ref(L["q"], L["s"], L["z"], x, k, rc=L["rc"], rS=L["rS"], W_hat=W_hat)
            if k:
                assert np.array_equal(out[f"s{i}_{rep}"], ref["idx"]), (i, rep)
            ok, err, bound = oracle.tolerance_ok(out[f"y{i}_{rep}"], ref["y64"], ref["A"])
            assert ok.all(), (i, rep, int((~ok).sum()))


def test_multilink_fetch_two_ranks_same_gpu(tmp_path):
    """NEXT-4: rank 1 gathers every other selected row over its own link and hands its o_dec part
    to rank 0 (here both share GPU 0 and its link); rank 0's y must equal the UNSHARDED oracle
    (all k rows) within L9, with the exact selection, over repeated calls on one ml area."""
    _run_ml(tmp_path, multi_gpu=False)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_multilink_fetch_two_gpus(tmp_path):
    _run_ml(tmp_path, multi_gpu=True)
