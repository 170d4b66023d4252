"""Output-feature tensor parallelism for DecDEC layers.

Every rank holds a contiguous, 32-column-aligned slice of the output columns of W_hat (HBM)
and of R_hat + its scales (its own pinned host slice, behind its own PCIe link).  x is
replicated, so every rank computes the identical selection S locally (the selector is exact
and deterministic) -- no index exchange.  The one real exchange step is assembling y: an
NCCL all-gather of the fp16 shards over NVLink, issued by the library (decdec_linear_tp /
decdec_stack_create_tp) on a library-owned communicator; the PyTorch process group only carries
the NCCL unique id (plumbing).
"""

from __future__ import annotations

import numpy as np

ALIGN = 32  # columns: 16-byte residual rows (4-bit) and whole 8-column words


def shard_columns(d_out: int, world: int, align: int = ALIGN):
    """[(start, stop)] contiguous column range per rank; equal widths, multiples of `align`."""
    if d_out % (world * align):
        raise ValueError(f"d_out={d_out} not divisible into {world} shards of multiples of {align}")
    w = d_out // world
    return [(r * w, (r + 1) * w) for r in range(world)]


def shard_codes(layer: dict, rank: int, world: int) -> dict:
    """Slice one layer's stored quantities (q/s/z [.., d_out], rc [d_in, d_out], rS [d_out],
    r16 [d_in, d_out]) to this rank's columns."""
    d_out = layer["q"].shape[1]
    a, b = shard_columns(d_out, world)[rank]
    out = {}
    for key, v in layer.items():
        if v is None:
            out[key] = None
        elif key in ("q", "s", "z", "rc", "r16"):
            out[key] = np.ascontiguousarray(v[:, a:b])
        elif key == "rS":
            out[key] = np.ascontiguousarray(v[a:b])
        else:
            out[key] = v
    return out


def broadcast_unique_id(group=None, make_id=None) -> bytes:
    """Rank 0 creates the 128-byte NCCL unique id (decdec_nccl_unique_id) and broadcasts it over
    the torch.distributed process group (plumbing only); every rank returns the same bytes."""
    import torch.distributed as dist

    if make_id is None:
        from paper_2412_20185_b200 import _lib

        make_id = _lib.decdec_nccl_unique_id
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return obj[0]


class Comm:
    """Library-owned NCCL communicator (decdec_comm_init) over the ranks of a torch PG."""

    def __init__(self, group=None):
        import torch.distributed as dist
        from paper_2412_20185_b200 import _lib

        self._lib = _lib
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.handle = _lib.decdec_comm_init(broadcast_unique_id(group), self.rank, self.world)

    def close(self):
        if self.handle:
            self._lib.decdec_comm_destroy(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TPLinear:
    """This rank's shard of a DecDEC layer; decdec_linear_tp runs the shard and the in-place
    NCCL all-gather that assembles y on every rank (one C-ABI call)."""

    def __init__(self, shard_linear, comm: Comm):
        self.lin = shard_linear
        self.comm = comm
        self.world = comm.world
        self.d_out_shard = shard_linear.d_out

    def __call__(self, x, k: int, chunk: int = 0, y_full=None, sel=None, workspace=None, stream=None):
        import torch
        from paper_2412_20185_b200 import _lib
        from paper_2412_20185_b200.layer import Workspace, _stream_ptr

        if y_full is None:
            y_full = torch.empty(self.d_out_shard * self.world, dtype=torch.float16, device=x.device)
        if workspace is None:
            workspace = Workspace(max(k, 1), self.d_out_shard)
        _lib.decdec_linear_tp(self.lin.struct, x.data_ptr(), k, chunk, y_full.data_ptr(),
                              sel.data_ptr() if sel is not None else 0, workspace.ptr, workspace.nbytes,
                              self.comm.handle, _stream_ptr(stream))
        return y_full


class TPStack:
    """A TP decode step (every layer on its shard + all-gather) as one native CUDA graph
    (decdec_stack_create_tp); launch/close like layer.Stack."""

    def __init__(self, layers, ks, xs, ys_full, workspace, comm: Comm, chunk: int = 0):
        from paper_2412_20185_b200 import _lib

        self._lib = _lib
        self._keep = (list(layers), list(xs), list(ys_full), workspace, comm)
        self.handle = _lib.decdec_stack_create_tp([l.struct for l in layers], ks, chunk,
                                                  [x.data_ptr() for x in xs], [y.data_ptr() for y in ys_full],
                                                  workspace.ptr, workspace.nbytes, comm.handle, 0)
        self.kernels = _lib.decdec_stack_kernels(self.handle)

    def launch(self, stream=None):
        from paper_2412_20185_b200.layer import _stream_ptr

        self._lib.decdec_stack_launch(self.handle, _stream_ptr(stream))

    def close(self):
        if self.handle:
            self._lib.decdec_stack_destroy(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ fused P2P-store all-gather
def peer_offsets(d_outs, world: int, align: int = 256):
    """Byte offsets of the y_full buffers ([world * d_out_r] fp16 each) inside a peer user
    area, and the total bytes: the same layout on every rank (symmetric memory)."""
    offs, o = [], 0
    for d in d_outs:
        offs.append(o)
        o += (world * int(d) * 2 + align - 1) // align * align
    return offs, o


class _DevView:
    """__cuda_array_interface__ over raw device memory (a torch view of the peer user area)."""

    def __init__(self, ptr: int, n: int, typestr: str = "<f2"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (int(ptr), False), "version": 3}


class Peers:
    """This rank's symmetric device region (decdec_peers_create) connected to every other rank's
    (decdec_peers_connect); the 64-byte CUDA-IPC handles travel over the torch process group
    (plumbing).  `view(off, n)` is a torch fp16 tensor over the local user area."""

    def __init__(self, user_bytes: int, group=None):
        import torch.distributed as dist
        from paper_2412_20185_b200 import _lib

        self._lib = _lib
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.handle, h = _lib.decdec_peers_create(user_bytes)
        hs = [None] * self.world
        dist.all_gather_object(hs, h, group=group)
        _lib.decdec_peers_connect(self.handle, self.rank, self.world, b"".join(hs))
        self.base = _lib.decdec_peers_buffer(self.handle)
        self.nbytes = _lib.decdec_peers_buffer_bytes(self.handle)

    def view(self, off: int, n: int):
        import torch

        if off + 2 * n > self.nbytes:
            raise ValueError("view outside the peer user area")
        return torch.as_tensor(_DevView(self.base + off, n), device="cuda")

    def close(self):
        if self.handle:
            self._lib.decdec_peers_destroy(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class P2PLinear:
    """This rank's shard of a DecDEC layer with the fused all-gather: one decdec_linear_p2p call
    writes the shard into every rank's y_full (peer user area at byte offset y_off) and returns
    when this rank's y_full is complete.  `slot` must differ between layers that may overlap."""

    def __init__(self, shard_linear, peers: Peers, y_off: int, slot: int):
        self.lin, self.peers, self.y_off, self.slot = shard_linear, peers, int(y_off), int(slot)
        self.d_out_shard = shard_linear.d_out
        self.y_full = peers.view(self.y_off, self.d_out_shard * peers.world)

    def __call__(self, x, k: int, chunk: int = 0, sel=None, workspace=None, stream=None):
        from paper_2412_20185_b200 import _lib
        from paper_2412_20185_b200.layer import Workspace, _stream_ptr

        if workspace is None:
            workspace = Workspace(max(k, 1), self.d_out_shard)
        _lib.decdec_linear_p2p(self.lin.struct, x.data_ptr(), k, chunk, self.y_off, self.slot,
                               sel.data_ptr() if sel is not None else 0, workspace.ptr, workspace.nbytes,
                               self.peers.handle, _stream_ptr(stream))
        return self.y_full


class P2PStack:
    """A TP decode step with the fused all-gather (decdec_stack_create_p2p): layer i writes every
    rank's y_full at y_offs[i] and waits on slot i; one native CUDA graph, no collective launch."""

    def __init__(self, layers, ks, xs, y_offs, workspace, peers: Peers, chunk: int = 0):
        from paper_2412_20185_b200 import _lib

        self._lib = _lib
        self._keep = (list(layers), list(xs), workspace, peers)
        self.handle = _lib.decdec_stack_create_p2p([l.struct for l in layers], ks, chunk, [x.data_ptr() for x in xs],
                                                   list(y_offs), workspace.ptr, workspace.nbytes, peers.handle, 0)
        self.kernels = _lib.decdec_stack_kernels(self.handle)
        self.y_full = [peers.view(o, l.d_out * peers.world) for o, l in zip(y_offs, layers)]

    def launch(self, stream=None):
        from paper_2412_20185_b200.layer import _stream_ptr

        self._lib.decdec_stack_launch(self.handle, _stream_ptr(stream))

    def close(self):
        if self.handle:
            self._lib.decdec_stack_destroy(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ multi-link residual fetch
class MLLinear:
    """NEXT-4 multi-link residual fetch (decdec_linear_ml): every rank of the peer group holds the
    FULL layer (its own host-mapped copy of the residual; base weights used on rank 0 only) and is
    called with the same x / k.  Rank r gathers the selected positions p with p % world == r over
    its own PCIe link; helpers (r > 0) store their o_dec parts into rank 0's user area at ml_off
    (decdec_ml_bytes) over NVLink; rank 0 writes y.  Returns y on rank 0, None on helpers."""

    def __init__(self, linear, peers: Peers, ml_off: int):
        self.lin, self.peers, self.ml_off = linear, peers, int(ml_off)

    @staticmethod
    def area_bytes(d_out: int, world: int) -> int:
        from paper_2412_20185_b200 import _lib

        return _lib.decdec_ml_bytes(d_out, world)

    def __call__(self, x, k: int, chunk: int = 0, y=None, sel=None, workspace=None, stream=None):
        import torch
        from paper_2412_20185_b200 import _lib
        from paper_2412_20185_b200.layer import Workspace, _stream_ptr

        main = self.peers.rank == 0
        if main and y is None:
            y = torch.empty(self.lin.d_out, dtype=torch.float16, device=x.device)
        if workspace is None:
            workspace = Workspace(max(k, 1), self.lin.d_out)
        _lib.decdec_linear_ml(self.lin.struct, x.data_ptr(), k, chunk, y.data_ptr() if main else 0,
                              sel.data_ptr() if (sel is not None and main) else 0, workspace.ptr, workspace.nbytes,
                              self.peers.handle, self.ml_off, _stream_ptr(stream))
        return y if main else None
