"""Output-feature tensor parallelism for DecDEC layers.

Every rank holds a contiguous, 32-column-aligned slice of the output columns of W_hat (HBM)
and of R_hat + its scales (its own pinned host slice, behind its own PCIe link).  x is
replicated, so every rank computes the identical selection S locally (the selector is exact
and deterministic) -- no index exchange.  The one real exchange step is assembling y: an
NCCL all-gather of the fp16 shards over NVLink (PyTorch process group = plumbing).
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


class TPLinear:
    """This rank's shard of a DecDEC layer + the all-gather that assembles y."""

    def __init__(self, shard_linear, group=None):
        import torch.distributed as dist

        self.lin = shard_linear
        self.group = group
        self.world = dist.get_world_size(group)
        self.d_out_shard = shard_linear.d_out

    def __call__(self, x, k: int, chunk: int = 0, y_full=None, y_shard=None, sel=None, workspace=None):
        import torch
        import torch.distributed as dist

        if y_shard is None:
            y_shard = torch.empty(self.d_out_shard, dtype=torch.float16, device=x.device)
        if y_full is None:
            y_full = torch.empty(self.d_out_shard * self.world, dtype=torch.float16, device=x.device)
        self.lin(x, k, chunk, y=y_shard, sel=sel, workspace=workspace)
        dist.all_gather_into_tensor(y_full, y_shard, group=self.group)
        return y_full
