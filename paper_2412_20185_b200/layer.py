"""Buffer ownership around the C ABI: device tensors (PyTorch = device memory and streams
only), the pinned + mapped host residual store, and the workspace.  Packing runs in the
library's C++ packers; compute runs in its CUDA kernels.  No arithmetic of the method here."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import decdec_layer

GROUP = 128


def _stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class HostBuffer:
    """Pinned, device-mapped host memory from decdec_host_alloc (zero-copy source)."""

    def __init__(self, nbytes: int, numa_node: int = -1, write_combined: bool = False):
        self.nbytes = int(nbytes)
        self.ptr = _lib.decdec_host_alloc(self.nbytes, numa_node, int(write_combined))

    def numpy(self, dtype=np.uint8, shape=None) -> np.ndarray:
        buf = (ctypes.c_uint8 * self.nbytes).from_address(self.ptr)
        a = np.frombuffer(buf, dtype=np.uint8).view(dtype)
        return a.reshape(shape) if shape is not None else a

    def free(self):
        if self.ptr:
            _lib.decdec_host_free(self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def pack_weights(q: np.ndarray, bits: int) -> np.ndarray:
    """q uint8 [d_in, d_out] -> packed uint32 [d_out, d_in*bits/32] via the C++ packer."""
    q = np.ascontiguousarray(q, dtype=np.uint8)
    d_in, d_out = q.shape
    out = np.zeros((d_out, d_in * bits // 32), dtype=np.uint32)
    _lib.decdec_pack_weights(q.ctypes.data, d_in, d_out, bits, out.ctypes.data, out.nbytes)
    return out


def pack_residual_into(c: np.ndarray, out: np.ndarray):
    """c int8 [d_in, d_out] -> Rq uint32 [d_in, d_out/8] written into `out` via the C++ packer."""
    c = np.ascontiguousarray(c, dtype=np.int8)
    d_in, d_out = c.shape
    _lib.decdec_pack_residual(c.ctypes.data, d_in, d_out, out.ctypes.data, out.nbytes)


class Workspace:
    def __init__(self, max_k: int, max_d_out: int, device="cuda", stream=None):
        self.nbytes = _lib.decdec_workspace_bytes(max_k, max_d_out)
        self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        _lib.decdec_workspace_init(self.buf.data_ptr(), self.nbytes, _stream_ptr(stream))

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()


class QuantLinear:
    """One DecDEC linear layer: packed W_hat in HBM, R_hat in pinned host memory."""

    def __init__(self):
        self.host = None
        self.host_scales_off = 0
        self.w_format = 0  # DECDEC_WFMT_UNIFORM
        self.lut = None

    @classmethod
    def from_codes(cls, q, s, z, bits, rc=None, rS=None, r16=None, device="cuda", numa_node=-1,
                   packed=None):
        """q uint8 [d_in, d_out]; s fp16 [G, d_out]; z uint8 [G, d_out] (oracle / synth layout).
        Residual: rc int8 [d_in, d_out] + rS fp16 [d_out] (r_bits 4), or r16 fp16 [d_in, d_out]."""
        self = cls()
        q = np.asarray(q)
        d_in, d_out = q.shape
        self.d_in, self.d_out, self.bits = d_in, d_out, bits
        wp = packed if packed is not None else pack_weights(q, bits)
        self.w = torch.from_numpy(wp.view(np.uint8).reshape(-1)).to(device)
        self.s = torch.from_numpy(np.ascontiguousarray(np.asarray(s, np.float16).T).reshape(-1)).to(device)
        self.z = torch.from_numpy(np.ascontiguousarray(np.asarray(z, np.uint8).T).reshape(-1)).to(device)
        self._attach_residual(rc, rS, r16, numa_node)
        self._L = self._struct()
        return self

    def _attach_residual(self, rc=None, rS=None, r16=None, numa_node=-1):
        """R_hat into pinned + mapped host memory: Rq rows + fp16 scales (r_bits 4) or fp16 rows."""
        d_in, d_out = self.d_in, self.d_out
        self.r_bits = 0
        if rc is not None:
            self.r_bits = 4
            row_bytes = d_out // 2
            sc_off = (d_in * row_bytes + 255) // 256 * 256
            self.host = HostBuffer(sc_off + 2 * d_out, numa_node)
            rows = self.host.numpy(np.uint32)[: d_in * row_bytes // 4].reshape(d_in, d_out // 8)
            pack_residual_into(rc, rows)
            self.host.numpy(np.uint8)[sc_off: sc_off + 2 * d_out].view(np.float16)[:] = np.asarray(rS, np.float16)
            self.host_scales_off = sc_off
        elif r16 is not None:
            self.r_bits = 16
            self.host = HostBuffer(d_in * d_out * 2, numa_node)
            self.host.numpy(np.float16, (d_in, d_out))[:] = np.asarray(r16, np.float16)

    @classmethod
    def from_lut_codes(cls, q, lut, bits, rc=None, rS=None, device="cuda", numa_node=-1):
        """Non-uniform (LUT) base layer (NEXT-3): q uint8 [d_in, d_out] codes < 2^bits, lut fp16
        [2^bits, d_out] (oracle layout).  Codes are packed as W4K nibbles by the C++ packer; the
        device table is [d_out][2^bits].  Optional r4 residual rc / rS as in from_codes."""
        self = cls()
        q = np.asarray(q)
        d_in, d_out = q.shape
        self.d_in, self.d_out, self.bits = d_in, d_out, bits
        self.w = torch.from_numpy(pack_weights(q, 4).view(np.uint8).reshape(-1)).to(device)
        self.lut = torch.from_numpy(np.ascontiguousarray(np.asarray(lut, np.float16).T).reshape(-1)).to(device)
        self.s = self.z = None
        self.w_format = 1
        self._attach_residual(rc, rS, None, numa_node)
        self._L = self._struct()
        return self

    @classmethod
    def from_device_lut(cls, d_in, d_out, bits, w, lut, host=None, host_scales_off=0):
        """Wrap device tensors of a LUT layer (perf harness): w uint8 W4K nibbles [d_out*d_in/2],
        lut fp16 [d_out * 2^bits]; host: optional HostBuffer with Rq rows + scales (r4)."""
        self = cls()
        self.d_in, self.d_out, self.bits = d_in, d_out, bits
        self.w, self.lut, self.s, self.z = w, lut, None, None
        self.w_format = 1
        self.host, self.r_bits, self.host_scales_off = host, (4 if host is not None else 0), host_scales_off
        self._L = self._struct()
        return self

    @classmethod
    def from_device_packed(cls, d_in, d_out, bits, w, s, z, host=None, r_bits=4, host_scales_off=0):
        """Wrap already-packed device tensors (perf harness): w uint8 [d_out*d_in*bits/8],
        s int16/fp16 [d_out*G], z uint8 [d_out*G]; host: HostBuffer with Rq rows + scales."""
        self = cls()
        self.d_in, self.d_out, self.bits = d_in, d_out, bits
        self.w, self.s, self.z = w, s, z
        self.host, self.r_bits, self.host_scales_off = host, (r_bits if host is not None else 0), host_scales_off
        self._L = self._struct()
        return self

    def _struct(self) -> decdec_layer:
        L = decdec_layer()
        L.d_in, L.d_out, L.w_bits, L.group_size = self.d_in, self.d_out, self.bits, GROUP
        L.w_packed = self.w.data_ptr()
        L.w_scales = self.s.data_ptr() if self.s is not None else None
        L.w_zeros = self.z.data_ptr() if self.z is not None else None
        L.w_format = self.w_format
        L.w_lut = self.lut.data_ptr() if self.lut is not None else None
        L.r_bits = self.r_bits or 4
        if self.host is not None:
            L.r_rows = self.host.ptr
            L.r_scales = self.host.ptr + self.host_scales_off if self.r_bits == 4 else None
        return L

    @property
    def struct(self) -> decdec_layer:
        return self._L

    def __call__(self, x: torch.Tensor, k: int, chunk: int = 0, y=None, sel=None, workspace=None, stream=None):
        if y is None:
            y = torch.empty(self.d_out, dtype=torch.float16, device=x.device)
        ws_ptr, ws_bytes = (workspace.ptr, workspace.nbytes) if workspace is not None else (0, 0)
        _lib.decdec_linear(self._L, x.data_ptr(), k, chunk, y.data_ptr(), sel.data_ptr() if sel is not None else 0,
                           ws_ptr, ws_bytes, _stream_ptr(stream))
        return y

    def gemv(self, x: torch.Tensor, y=None, stream=None):
        if y is None:
            y = torch.empty(self.d_out, dtype=torch.float16, device=x.device)
        _lib.decdec_gemv(self._L, x.data_ptr(), y.data_ptr(), 0, 0, _stream_ptr(stream))
        return y

    def debug_unpack(self) -> torch.Tensor:
        q = torch.empty((self.d_out, self.d_in), dtype=torch.uint8, device=self.w.device)
        _lib.decdec_debug_unpack_weights(self._L, q.data_ptr(), _stream_ptr())
        return q

    def plan(self, k_sel: int = 0) -> str:
        return _lib.decdec_plan_string(self._L, k_sel)


def select(x: torch.Tensor, k: int, chunk: int = 0, stream=None):
    """Step (1) alone via decdec_select -> (idx int32, xs fp16) device tensors."""
    n = _lib.decdec_num_selected(x.numel(), k, chunk)
    if n < 0:
        raise ValueError("invalid (d_in, k, chunk)")
    idx = torch.empty(max(n, 1), dtype=torch.int32, device=x.device)
    xs = torch.empty(max(n, 1), dtype=torch.float16, device=x.device)
    _lib.decdec_select(x.data_ptr(), x.numel(), k, chunk, idx.data_ptr(), xs.data_ptr(), _stream_ptr(stream))
    return idx[:n], xs[:n]


class Stack:
    """A decode step's layer calls as one native CUDA graph (decdec_stack_*)."""

    def __init__(self, layers, ks, xs, ys, workspace, chunk: int = 0, stream=None):
        self.layers = list(layers)
        self._keep = (list(xs), list(ys), workspace)
        self.handle = _lib.decdec_stack_create([l.struct for l in self.layers], ks, chunk,
                                               [x.data_ptr() for x in xs], [y.data_ptr() for y in ys],
                                               workspace.ptr, workspace.nbytes, _stream_ptr(stream))
        self.kernels = _lib.decdec_stack_kernels(self.handle)

    def launch(self, stream=None):
        _lib.decdec_stack_launch(self.handle, _stream_ptr(stream))

    def close(self):
        if self.handle:
            _lib.decdec_stack_destroy(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
