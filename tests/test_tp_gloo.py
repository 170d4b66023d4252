"""World-size-2 gloo tests of the tensor-parallel host logic (CPU): column sharding, per-rank
selection identity, and assembly of y shards by all-gather equal to the unsharded result.
Per-rank compute here is the oracle (no GPU on this host); the GPU path shares the sharding
and assembly code (paper_2412_20185_b200.tp)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tp_shard_logic():
    # import without loading the CUDA library (tp.py is pure host logic)
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("tp", os.path.join(root, "paper_2412_20185_b200", "tp.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from synth import gen_activations, gen_perf_layer

        tp = _tp_shard_logic()
        d_in, d_out, k = 1024, 512, 24
        L = gen_perf_layer(d_in, d_out, 3, seed=77)
        x = gen_activations(d_in, 1, seed=78)[0]
        sh = tp.shard_codes(L, rank, world)
        out = oracle.decdec_linear_ref(sh["q"], sh["s"], sh["z"], x, k, rc=sh["rc"], rS=sh["rS"])
        # selection identical on every rank
        idx = torch.from_numpy(out["idx"].astype(np.int64))
        gathered = [torch.empty_like(idx) for _ in range(world)]
        dist.all_gather(gathered, idx)
        same = all(torch.equal(g, gathered[0]) for g in gathered)
        # assemble y: all-gather of the shards == unsharded oracle, bit for bit
        ys = torch.from_numpy(out["y64"])
        parts = [torch.empty_like(ys) for _ in range(world)]
        dist.all_gather(parts, ys)
        y_full = torch.cat(parts).numpy()
        ref = oracle.decdec_linear_ref(L["q"], L["s"], L["z"], x, k, rc=L["rc"], rS=L["rS"])["y64"]
        # the library communicator's NCCL unique id: made on rank 0 only, identical bytes everywhere
        calls = []
        uid = tp.broadcast_unique_id(make_id=lambda: calls.append(1) or bytes(range(128)))
        uid_ok = uid == bytes(range(128)) and len(calls) == (1 if rank == 0 else 0)
        q.put((rank, same and uid_ok, bool(np.array_equal(y_full, ref)), tp.shard_columns(d_out, world)))
    finally:
        dist.destroy_process_group()


def test_shard_columns():
    tp = _tp_shard_logic()
    assert tp.shard_columns(4096, 8) == [(i * 512, (i + 1) * 512) for i in range(8)]
    assert tp.shard_columns(5120, 8)[-1] == (4480, 5120)    # Phi-3 o at P=8: 640 columns each
    with pytest.raises(ValueError):
        tp.shard_columns(1024, 3)


def test_tp_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, same, equal, cols in res:
        assert same, f"rank {rank}: selection or NCCL unique id differs across ranks"
        assert equal, f"rank {rank}: assembled y differs from unsharded oracle"
        assert cols == [(0, 256), (256, 512)]
