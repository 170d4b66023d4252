"""B200-native DecDEC decode hot path (arXiv 2412.20185).

    o = W_hat x + sum_{i in TopK(|x|)} x_i R_hat[i, :]

The compute lives in libdecdec.so (hand-written sm_100a CUDA behind the C ABI of
include/decdec.h); this package is the thin binding plus buffer ownership.
"""

from ._lib import (  # noqa: F401
    EXPORTED,
    LIB_PATH,
    DecdecError,
    decdec_comm_destroy,
    decdec_comm_init,
    decdec_comm_nranks,
    decdec_comm_rank,
    decdec_debug_selections,
    decdec_device_numa_node,
    numa_node_of_device,
    decdec_debug_trace,
    decdec_debug_unpack_weights,
    decdec_gemv,
    decdec_host_alloc,
    decdec_host_free,
    decdec_launches_per_call,
    decdec_layer,
    decdec_linear,
    decdec_linear_tp,
    decdec_nccl_unique_id,
    decdec_nccl_version,
    decdec_num_selected,
    decdec_pack_residual,
    decdec_pack_weights,
    decdec_plan_string,
    decdec_select,
    decdec_set_dec_ctas,
    decdec_stack_create,
    decdec_stack_create_tp,
    decdec_stack_destroy,
    decdec_stack_kernels,
    decdec_stack_launch,
    decdec_status_string,
    decdec_version,
    decdec_workspace_bytes,
    decdec_workspace_init,
)
from .tp import Comm, MLLinear, P2PLinear, P2PStack, Peers, TPLinear, TPStack, peer_offsets, shard_codes, shard_columns  # noqa: F401
from .layer import HostBuffer, QuantLinear, Stack, Workspace, pack_residual_into, pack_weights, select  # noqa: F401
