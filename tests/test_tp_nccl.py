"""Multi-GPU tensor parallelism on real NCCL (a7 of SURVEY.md §8(a); §8(e)): min(#GPUs, 8)
ranks, one process per GPU, each holding its output-feature shard of W_hat in HBM and its own
pinned host slice of R_hat.  decdec_linear_tp and the TP step executor (TPStack) must give, on
every rank, the full y of the UNSHARDED oracle (L9), bit-identical across ranks, with every
rank's selection equal to the oracle's (x replicated, exact selector; ledger L11).
Skips with fewer than 2 GPUs (the sandbox and the driver's 1-GPU tiers)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs >= 2 GPUs", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SHAPES = [("llama3_70b", "o", 8192, 8192), ("phi3_medium", "d", 17920, 5120), ("llama3_8b", "gu", 4096, 28672)]


def _worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import oracle
    import paper_2412_20185_b200 as dd
    from paper_2412_20185_b200.tp import shard_codes
    from synth import gen_activations, gen_perf_layer, layer_seed

    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    comm = dd.Comm()
    results = {}
    try:
        for model, name, d_in, d_out in SHAPES:
            if d_out % (32 * world):
                continue
            L = gen_perf_layer(d_in, d_out, 3, seed=layer_seed("tpnccl", model, name))
            Sh = shard_codes(L, rank, world)
            lin = dd.QuantLinear.from_codes(Sh["q"], Sh["s"], Sh["z"], 3, rc=Sh["rc"], rS=Sh["rS"],
                                            numa_node=dd.numa_node_of_device(rank))
            x = gen_activations(d_in, 1, seed=layer_seed("tpnccl", model, name, "x"), kind="d" if name == "d" else "qkv")[0]
            xd = torch.from_numpy(x).cuda()
            k = oracle.k_from_kchunk(21, d_in)
            ws = dd.Workspace(k, d_out // world)
            sel = torch.empty(k, dtype=torch.int32, device="cuda")
            y_full = dd.TPLinear(lin, comm)(xd, k, sel=sel, workspace=ws)
            ys = torch.empty(d_out, dtype=torch.float16, device="cuda")
            st = dd.TPStack([lin], [k], [xd], [ys], ws, comm)
            st.launch()
            torch.cuda.synchronize()
            st.close()
            results[name] = (y_full.cpu().numpy(), ys.cpu().numpy(), sel.cpu().numpy())
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
                 **{f"{n}_{i}": v for n, t in results.items() for i, v in enumerate(t)})
    finally:
        comm.close()
        dist.destroy_process_group()


def test_tp_nccl_multi_gpu(tmp_path):
    import torch.multiprocessing as mp

    import oracle
    from synth import gen_activations, gen_perf_layer, layer_seed

    world = min(torch.cuda.device_count(), 8)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    for model, name, d_in, d_out in SHAPES:
        if d_out % (32 * world):
            continue
        L = gen_perf_layer(d_in, d_out, 3, seed=layer_seed("tpnccl", model, name))
        x = gen_activations(d_in, 1, seed=layer_seed("tpnccl", model, name, "x"), kind="d" if name == "d" else "qkv")[0]
        k = oracle.k_from_kchunk(21, d_in)
        ref = oracle.decdec_linear_ref(L["q"], L["s"], L["z"], x, k, rc=L["rc"], rS=L["rS"])
        y0 = outs[0][f"{name}_0"]
        for r in range(world):
            y_lin, y_stack, sel = (outs[r][f"{name}_{i}"] for i in range(3))
            assert np.array_equal(sel, ref["idx"]), (name, r)
            assert np.array_equal(y_lin.view(np.uint16), y0.view(np.uint16)), (name, r)   # identical on every rank
            assert np.array_equal(y_stack.view(np.uint16), y0.view(np.uint16)), (name, r)
        ok, err, bound = oracle.tolerance_ok(y0, ref["y64"], ref["A"])
        assert ok.all(), (name, int((~ok).sum()))
