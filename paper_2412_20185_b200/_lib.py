"""Thin ctypes binding of libdecdec.so (include/decdec.h).  Argument marshalling only:
every step of the hot path runs in the library's sm_100a kernels.  There is no CPU or
PyTorch fallback: if the library is missing this module raises at import."""

from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# DECDEC_LIB: load another build of the same ABI (A/B timing of kernel variants on one box)
LIB_PATH = os.environ.get("DECDEC_LIB") or os.path.join(_PKG, "libdecdec.so")

DECDEC_OK = 0
STATUS = {0: "DECDEC_OK", -1: "DECDEC_EINVAL", -2: "DECDEC_EALIGN", -3: "DECDEC_ENOTMAPPED",
          -4: "DECDEC_EUNSUPPORTED", -5: "DECDEC_ECUDA", -6: "DECDEC_ENCCL", -7: "DECDEC_ESPACE"}


class DecdecError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {STATUS.get(status, status)} ({_lib.decdec_status_string(status).decode()})")
        self.status = status


class decdec_layer(ctypes.Structure):
    _fields_ = [
        ("d_in", ctypes.c_int32), ("d_out", ctypes.c_int32),
        ("w_bits", ctypes.c_int32), ("group_size", ctypes.c_int32),
        ("w_packed", ctypes.c_void_p), ("w_scales", ctypes.c_void_p), ("w_zeros", ctypes.c_void_p),
        ("r_bits", ctypes.c_int32),
        ("r_rows", ctypes.c_void_p), ("r_scales", ctypes.c_void_p),
        ("w_format", ctypes.c_int32), ("w_lut", ctypes.c_void_p),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libdecdec.so not found at {LIB_PATH}: build it with `python -m paper_2412_20185_b200.build` "
            "(no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, SZ, VP = ctypes.POINTER, ctypes.c_int32, ctypes.c_size_t, ctypes.c_void_p
    Lp = P(decdec_layer)
    sig = {
        "decdec_workspace_bytes": (SZ, [I32, I32]),
        "decdec_workspace_init": (I32, [VP, SZ, VP]),
        "decdec_linear": (I32, [Lp, VP, I32, I32, VP, VP, VP, SZ, VP]),
        "decdec_gemv": (I32, [Lp, VP, VP, VP, SZ, VP]),
        "decdec_select": (I32, [VP, I32, I32, I32, VP, VP, VP]),
        "decdec_num_selected": (I32, [I32, I32, I32]),
        "decdec_pack_weights": (I32, [VP, I32, I32, I32, VP, SZ]),
        "decdec_pack_residual": (I32, [VP, I32, I32, VP, SZ]),
        "decdec_host_alloc": (I32, [SZ, I32, I32, P(VP)]),
        "decdec_host_free": (None, [VP]),
        "decdec_device_numa_node": (I32, [I32]),
        "decdec_debug_unpack_weights": (I32, [Lp, VP, VP]),
        "decdec_plan_string": (I32, [Lp, I32, ctypes.c_char_p, SZ]),
        "decdec_launches_per_call": (I32, [I32]),
        "decdec_debug_trace": (I32, [VP, SZ]),
        "decdec_debug_selections": (I32, [VP, VP, I32, I32]),
        "decdec_stack_create": (I32, [Lp, I32, P(I32), I32, P(VP), P(VP), VP, SZ, VP, P(VP)]),
        "decdec_stack_launch": (I32, [VP, VP]),
        "decdec_stack_kernels": (I32, [VP]),
        "decdec_stack_destroy": (None, [VP]),
        "decdec_status_string": (ctypes.c_char_p, [I32]),
        "decdec_version": (ctypes.c_char_p, []),
        "decdec_set_dec_ctas": (I32, [I32]),
        "decdec_nccl_version": (I32, []),
        "decdec_nccl_unique_id": (I32, [VP]),
        "decdec_comm_init": (I32, [VP, I32, I32, P(VP)]),
        "decdec_comm_destroy": (None, [VP]),
        "decdec_comm_rank": (I32, [VP]),
        "decdec_comm_nranks": (I32, [VP]),
        "decdec_linear_tp": (I32, [Lp, VP, I32, I32, VP, VP, VP, SZ, VP, VP]),
        "decdec_stack_create_tp": (I32, [Lp, I32, P(I32), I32, P(VP), P(VP), VP, SZ, VP, VP, P(VP)]),
        "decdec_peers_create": (I32, [SZ, VP, P(VP)]),
        "decdec_peers_connect": (I32, [VP, I32, I32, VP]),
        "decdec_peers_buffer": (VP, [VP]),
        "decdec_peers_buffer_bytes": (SZ, [VP]),
        "decdec_peers_destroy": (None, [VP]),
        "decdec_linear_p2p": (I32, [Lp, VP, I32, I32, SZ, I32, VP, VP, SZ, VP, VP]),
        "decdec_stack_create_p2p": (I32, [Lp, I32, P(I32), I32, P(VP), P(SZ), VP, SZ, VP, VP, P(VP)]),
        "decdec_ml_bytes": (SZ, [I32, I32]),
        "decdec_linear_ml": (I32, [Lp, VP, I32, I32, VP, VP, VP, SZ, VP, SZ, VP]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("DECDEC_LIB") and not hasattr(lib, name):
            continue  # A/B against an older build: entry points it lacks stay absent
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()
EXPORTED = [
    "decdec_workspace_bytes", "decdec_workspace_init", "decdec_linear", "decdec_gemv", "decdec_select",
    "decdec_num_selected", "decdec_pack_weights", "decdec_pack_residual", "decdec_host_alloc",
    "decdec_host_free", "decdec_device_numa_node", "decdec_debug_unpack_weights", "decdec_plan_string", "decdec_launches_per_call",
    "decdec_status_string", "decdec_version", "decdec_stack_create", "decdec_stack_launch",
    "decdec_stack_kernels", "decdec_stack_destroy", "decdec_debug_trace", "decdec_debug_selections",
    "decdec_set_dec_ctas", "decdec_nccl_version", "decdec_nccl_unique_id", "decdec_comm_init", "decdec_comm_destroy",
    "decdec_comm_rank", "decdec_comm_nranks", "decdec_linear_tp", "decdec_stack_create_tp",
    "decdec_peers_create", "decdec_peers_connect", "decdec_peers_buffer", "decdec_peers_buffer_bytes",
    "decdec_peers_destroy", "decdec_linear_p2p", "decdec_stack_create_p2p", "decdec_ml_bytes", "decdec_linear_ml",
]


def _check(status: int, where: str):
    if status != DECDEC_OK:
        raise DecdecError(status, where)


def _vp(p):
    return ctypes.c_void_p(int(p) if p else 0)


# ------------------------------------------------------------------ same names as the C ABI
def decdec_workspace_bytes(max_k: int, max_d_out: int) -> int:
    return int(_lib.decdec_workspace_bytes(max_k, max_d_out))


def decdec_workspace_init(ws, ws_bytes, stream=0):
    _check(_lib.decdec_workspace_init(_vp(ws), ws_bytes, _vp(stream)), "decdec_workspace_init")


def decdec_linear(L: decdec_layer, x, k: int, chunk: int, y, sel, ws, ws_bytes: int, stream=0):
    _check(_lib.decdec_linear(ctypes.byref(L), _vp(x), k, chunk, _vp(y), _vp(sel), _vp(ws), ws_bytes, _vp(stream)),
           "decdec_linear")


def decdec_gemv(L: decdec_layer, x, y, ws=0, ws_bytes=0, stream=0):
    _check(_lib.decdec_gemv(ctypes.byref(L), _vp(x), _vp(y), _vp(ws), ws_bytes, _vp(stream)), "decdec_gemv")


def decdec_select(x, d_in: int, k: int, chunk: int, idx, xs, stream=0):
    _check(_lib.decdec_select(_vp(x), d_in, k, chunk, _vp(idx), _vp(xs), _vp(stream)), "decdec_select")


def decdec_num_selected(d_in: int, k: int, chunk: int) -> int:
    return int(_lib.decdec_num_selected(d_in, k, chunk))


def decdec_pack_weights(q_ptr, d_in, d_out, bits, out_ptr, out_bytes):
    _check(_lib.decdec_pack_weights(_vp(q_ptr), d_in, d_out, bits, _vp(out_ptr), out_bytes), "decdec_pack_weights")


def decdec_pack_residual(c_ptr, d_in, d_out, out_ptr, out_bytes):
    _check(_lib.decdec_pack_residual(_vp(c_ptr), d_in, d_out, _vp(out_ptr), out_bytes), "decdec_pack_residual")


def decdec_host_alloc(nbytes: int, numa_node: int = -1, write_combined: int = 0) -> int:
    p = ctypes.c_void_p()
    _check(_lib.decdec_host_alloc(nbytes, numa_node, write_combined, ctypes.byref(p)), "decdec_host_alloc")
    return int(p.value)


def decdec_device_numa_node(device: int) -> int:
    return int(_lib.decdec_device_numa_node(device))


def numa_node_of_device(device: int) -> int:
    """NUMA node in front of the GPU's PCIe link (-1 if unknown): where its residual slice goes."""
    return decdec_device_numa_node(device)


def decdec_host_free(p):
    _lib.decdec_host_free(_vp(p))


def decdec_debug_unpack_weights(L: decdec_layer, q_out, stream=0):
    _check(_lib.decdec_debug_unpack_weights(ctypes.byref(L), _vp(q_out), _vp(stream)), "decdec_debug_unpack_weights")


def decdec_plan_string(L: decdec_layer, k_sel: int) -> str:
    buf = ctypes.create_string_buffer(512)
    _check(_lib.decdec_plan_string(ctypes.byref(L), k_sel, buf, 512), "decdec_plan_string")
    return buf.value.decode()


def decdec_set_dec_ctas(n: int):
    _check(_lib.decdec_set_dec_ctas(n), "decdec_set_dec_ctas")


def decdec_launches_per_call(k: int) -> int:
    return int(_lib.decdec_launches_per_call(k))


def decdec_status_string(s: int) -> str:
    return _lib.decdec_status_string(s).decode()


def decdec_version() -> str:
    return _lib.decdec_version().decode()


def decdec_stack_create(layers, ks, chunk, xs, ys, ws, ws_bytes, stream=0) -> int:
    n = len(layers)
    arr = (decdec_layer * n)(*layers)
    karr = (ctypes.c_int32 * n)(*[int(k) for k in ks])
    xarr = (ctypes.c_void_p * n)(*[int(p) for p in xs])
    yarr = (ctypes.c_void_p * n)(*[int(p) for p in ys])
    out = ctypes.c_void_p()
    _check(_lib.decdec_stack_create(arr, n, karr, chunk, xarr, yarr, _vp(ws), ws_bytes, _vp(stream), ctypes.byref(out)),
           "decdec_stack_create")
    return int(out.value)


def decdec_stack_launch(s, stream=0):
    _check(_lib.decdec_stack_launch(_vp(s), _vp(stream)), "decdec_stack_launch")


def decdec_stack_kernels(s) -> int:
    return int(_lib.decdec_stack_kernels(_vp(s)))


def decdec_stack_destroy(s):
    _lib.decdec_stack_destroy(_vp(s))


def decdec_debug_trace(buf, nbytes):
    _check(_lib.decdec_debug_trace(_vp(buf), nbytes), "decdec_debug_trace")


# ------------------------------------------------------------------ tensor parallelism
def decdec_debug_selections(idx, xs, cap: int, max_ctas: int):
    """Debug: every DEC CTA c < max_ctas writes its own selection to idx/xs[c*cap ...] (0 = off)."""
    _check(_lib.decdec_debug_selections(_vp(idx), _vp(xs), cap, max_ctas), "decdec_debug_selections")


def decdec_nccl_version() -> int:
    return int(_lib.decdec_nccl_version())


def decdec_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.decdec_nccl_unique_id(buf), "decdec_nccl_unique_id")
    return buf.raw


def decdec_comm_init(uid: bytes, rank: int, nranks: int) -> int:
    if len(uid) != 128:
        raise ValueError("NCCL unique id must be 128 bytes")
    buf = ctypes.create_string_buffer(uid, 128)
    out = ctypes.c_void_p()
    _check(_lib.decdec_comm_init(buf, rank, nranks, ctypes.byref(out)), "decdec_comm_init")
    return int(out.value)


def decdec_comm_destroy(c):
    _lib.decdec_comm_destroy(_vp(c))


def decdec_comm_rank(c) -> int:
    return int(_lib.decdec_comm_rank(_vp(c)))


def decdec_comm_nranks(c) -> int:
    return int(_lib.decdec_comm_nranks(_vp(c)))


def decdec_linear_tp(L: decdec_layer, x, k: int, chunk: int, y_full, sel, ws, ws_bytes: int, comm, stream=0):
    _check(_lib.decdec_linear_tp(ctypes.byref(L), _vp(x), k, chunk, _vp(y_full), _vp(sel), _vp(ws), ws_bytes,
                                 _vp(comm), _vp(stream)), "decdec_linear_tp")


def decdec_stack_create_tp(layers, ks, chunk, xs, ys_full, ws, ws_bytes, comm, stream=0) -> int:
    n = len(layers)
    arr = (decdec_layer * n)(*layers)
    karr = (ctypes.c_int32 * n)(*[int(k) for k in ks])
    xarr = (ctypes.c_void_p * n)(*[int(p) for p in xs])
    yarr = (ctypes.c_void_p * n)(*[int(p) for p in ys_full])
    out = ctypes.c_void_p()
    _check(_lib.decdec_stack_create_tp(arr, n, karr, chunk, xarr, yarr, _vp(ws), ws_bytes, _vp(comm), _vp(stream),
                                       ctypes.byref(out)), "decdec_stack_create_tp")
    return int(out.value)


# ---- fused P2P-store all-gather (decdec_peers)
IPC_HANDLE_BYTES = 64


def decdec_peers_create(user_bytes: int):
    """-> (peers handle, 64-byte IPC handle of this rank's region)"""
    h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    out = ctypes.c_void_p()
    _check(_lib.decdec_peers_create(user_bytes, h, ctypes.byref(out)), "decdec_peers_create")
    return int(out.value), h.raw


def decdec_peers_connect(p, rank: int, nranks: int, handles: bytes):
    if len(handles) != nranks * IPC_HANDLE_BYTES:
        raise ValueError("handles must be nranks x 64 bytes")
    buf = ctypes.create_string_buffer(handles, len(handles))
    _check(_lib.decdec_peers_connect(_vp(p), rank, nranks, buf), "decdec_peers_connect")


def decdec_peers_buffer(p) -> int:
    return int(_lib.decdec_peers_buffer(_vp(p)) or 0)


def decdec_peers_buffer_bytes(p) -> int:
    return int(_lib.decdec_peers_buffer_bytes(_vp(p)))


def decdec_peers_destroy(p):
    _lib.decdec_peers_destroy(_vp(p))


def decdec_linear_p2p(L: decdec_layer, x, k: int, chunk: int, y_off: int, slot: int, sel, ws, ws_bytes: int, peers,
                      stream=0):
    _check(_lib.decdec_linear_p2p(ctypes.byref(L), _vp(x), k, chunk, y_off, slot, _vp(sel), _vp(ws), ws_bytes,
                                  _vp(peers), _vp(stream)), "decdec_linear_p2p")


def decdec_stack_create_p2p(layers, ks, chunk, xs, y_offs, ws, ws_bytes, peers, stream=0) -> int:
    n = len(layers)
    arr = (decdec_layer * n)(*layers)
    karr = (ctypes.c_int32 * n)(*[int(k) for k in ks])
    xarr = (ctypes.c_void_p * n)(*[int(p) for p in xs])
    oarr = (ctypes.c_size_t * n)(*[int(o) for o in y_offs])
    out = ctypes.c_void_p()
    _check(_lib.decdec_stack_create_p2p(arr, n, karr, chunk, xarr, oarr, _vp(ws), ws_bytes, _vp(peers), _vp(stream),
                                        ctypes.byref(out)), "decdec_stack_create_p2p")
    return int(out.value)


def decdec_ml_bytes(d_out: int, nranks: int) -> int:
    return int(_lib.decdec_ml_bytes(d_out, nranks))


def decdec_linear_ml(L: decdec_layer, x, k: int, chunk: int, y, sel, ws, ws_bytes: int, peers, ml_off: int, stream=0):
    _check(_lib.decdec_linear_ml(ctypes.byref(L), _vp(x), k, chunk, _vp(y), _vp(sel), _vp(ws), ws_bytes, _vp(peers),
                                 ml_off, _vp(stream)), "decdec_linear_ml")
