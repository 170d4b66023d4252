// Throughput of warp-collective and smem primitives on one SM (1 CTA x 1024 threads):
// VOTE (ballot), SHFL, REDUX (reduce_add), MATCH.ANY, LDS, smem atomics, ALU reference.
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1;} } while (0)

template <int OP>
__global__ void k_tput(unsigned* out, int iters) {
  __shared__ unsigned sm[1024];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) {  // ballot
      a0 += __ballot_sync(0xffffffffu, a0 & 1); a1 += __ballot_sync(0xffffffffu, a1 & 2);
      a2 += __ballot_sync(0xffffffffu, a2 & 4); a3 += __ballot_sync(0xffffffffu, a3 & 8);
    } else if (OP == 1) {  // shfl
      a0 += __shfl_xor_sync(0xffffffffu, a0, 1); a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
      a2 += __shfl_xor_sync(0xffffffffu, a2, 4); a3 += __shfl_xor_sync(0xffffffffu, a3, 8);
    } else if (OP == 2) {  // redux
      a0 += __reduce_add_sync(0xffffffffu, a0); a1 += __reduce_add_sync(0xffffffffu, a1);
      a2 += __reduce_add_sync(0xffffffffu, a2); a3 += __reduce_add_sync(0xffffffffu, a3);
    } else if (OP == 3) {  // match.any
      a0 += __match_any_sync(0xffffffffu, a0 & 7); a1 += __match_any_sync(0xffffffffu, a1 & 7);
      a2 += __match_any_sync(0xffffffffu, a2 & 7); a3 += __match_any_sync(0xffffffffu, a3 & 7);
    } else if (OP == 4) {  // lds
      a0 += sm[(a0 + i) & 1023]; a1 += sm[(a1 + i) & 1023]; a2 += sm[(a2 + i) & 1023]; a3 += sm[(a3 + i) & 1023];
    } else if (OP == 5) {  // smem atomics, spread
      atomicAdd(&sm[(a0 * 33 + i) & 1023], 1u); atomicAdd(&sm[(a1 * 33 + i) & 1023], 1u);
      atomicAdd(&sm[(a2 * 33 + i) & 1023], 1u); atomicAdd(&sm[(a3 * 33 + i) & 1023], 1u);
      a0 += 1; a1 += 3; a2 += 5; a3 += 7;
    } else {  // alu
      a0 = a0 * 3 + 1; a1 = a1 ^ (a1 >> 3); a2 = a2 + (a2 << 2); a3 = a3 ^ 0x5555;
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[0] = (unsigned)(t1 - t0);
  if (a0 + a1 + a2 + a3 == 0x12345) out[1] = 1;
}

int main() {
  unsigned* o; CK(cudaMalloc(&o, 64));
  const char* names[] = {"ballot", "shfl", "redux", "match_any", "lds", "atom_smem", "alu"};
  const int iters = 256;
  for (int op = 0; op < 7; ++op) {
    unsigned h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: k_tput<0><<<1, 1024>>>(o, iters); break; case 1: k_tput<1><<<1, 1024>>>(o, iters); break;
        case 2: k_tput<2><<<1, 1024>>>(o, iters); break; case 3: k_tput<3><<<1, 1024>>>(o, iters); break;
        case 4: k_tput<4><<<1, 1024>>>(o, iters); break; case 5: k_tput<5><<<1, 1024>>>(o, iters); break;
        default: k_tput<6><<<1, 1024>>>(o, iters);
      }
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(&h, o, 4, cudaMemcpyDeviceToHost));
    }
    // 32 warps x iters x 4 ops warp-instructions on one SM (4 SMSPs)
    printf("{\"op\": \"%s\", \"cycles\": %u, \"cyc_per_warp_op_per_smsp\": %.2f}\n", names[op], h, (double)h / (32.0 * iters * 4 / 4));
  }
  return 0;
}
