// Internal (not part of the C ABI): the all-gather step shared by decdec_linear_tp and the
// TP step executor (decdec_stack_create_tp).
#pragma once
#include <cuda_runtime.h>

#include "decdec.h"

decdec_status tp_allgather(decdec_comm* c, uint16_t* y_full, int32_t d_out_r, cudaStream_t st);
int32_t tp_rank(const decdec_comm* c);
