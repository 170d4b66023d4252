// Cost of the DEC CTA's exact Top-k (select_block_regs) in isolation: one CTA, `iters` calls
// back to back on the same x (instruction cache and L1 warm), thread 0 records SM cycles per
// phase into a trace array.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include "select.cuh"
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1;} } while (0)
using namespace decdec;

__global__ void k_sel(const uint16_t* x, int n, int q, int iters, int* idx, uint16_t* xs, unsigned long long* tr) {
  extern __shared__ __align__(16) uint8_t smem[];
  SelectSmemS* S = reinterpret_cast<SelectSmemS*>(smem);
  int* sidx = reinterpret_cast<int*>(smem + select_split_smem_bytes(n));
  uint16_t* sxs = reinterpret_cast<uint16_t*>(sidx + q);
  for (int it = 0; it < iters; ++it) {
    select_split_zero(S, n);
    __syncthreads();
    unsigned long long* t = tr + it * 20;
    if (threadIdx.x == 0) t[15] = clock64();
    select_split_any(x, n, q, sidx, sxs, nullptr, S, (blockDim.x >> 5) - 1, t);
    __syncthreads();
    if (threadIdx.x == 0) t[14] = clock64();
  }
  for (int i = threadIdx.x; i < q; i += blockDim.x) { idx[i] = sidx[i]; xs[i] = sxs[i]; }
}

int main() {
  for (int n : {4096, 14336}) {
    for (int nt : {288, 544}) {
      const int q = n / 1024 * 21;
      uint16_t* hx = (uint16_t*)malloc(n * 2);
      srand(5);
      char fname[64];
      snprintf(fname, sizeof fname, "gpurun_out/x%d.bin", n);  // synth activations (tools/select_inputs.py)
      FILE* fx = fopen(fname, "rb");
      if (fx) {
        if (fread(hx, 2, n, fx) != (size_t)n) return 1;
        fclose(fx);
      } else
      for (int i = 0; i < n; ++i) {
        float g = 0; for (int k = 0; k < 12; ++k) g += rand() / (float)RAND_MAX; g -= 6;
        float v = expf(0.5f * g) * (rand() & 1 ? 1 : -1) * 0.3f;
        __half h = __float2half(v); hx[i] = *reinterpret_cast<uint16_t*>(&h);
      }
      uint16_t *dx, *dxs; int* didx; unsigned long long* dtr;
      const int iters = getenv("ITERS") ? atoi(getenv("ITERS")) : 20;
      CK(cudaMalloc(&dx, n * 2)); CK(cudaMalloc(&didx, q * 4)); CK(cudaMalloc(&dxs, q * 2)); CK(cudaMalloc(&dtr, iters * 20 * 8));
      CK(cudaMemcpy(dx, hx, n * 2, cudaMemcpyHostToDevice));
      const size_t sm = select_split_smem_bytes(n) + q * 6 + 64;
      CK(cudaFuncSetAttribute(k_sel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      k_sel<<<1, nt, sm>>>(dx, n, q, iters, didx, dxs, dtr);
      CK(cudaDeviceSynchronize());
      {  // result checksum (order-sensitive) to compare selector variants
        int* hi = (int*)malloc(q * 4);
        CK(cudaMemcpy(hi, didx, q * 4, cudaMemcpyDeviceToHost));
        unsigned long long cs = 0;
        for (int i = 0; i < q; ++i) cs = cs * 1000003ull + (unsigned)hi[i];
        printf("checksum n=%d threads=%d: %llu\n", n, nt, cs);
        free(hi);
      }
      static unsigned long long h[1000 * 20];
      CK(cudaMemcpy(h, dtr, iters * 20 * 8, cudaMemcpyDeviceToHost));
      for (int it : {0, 1, iters - 1}) {
        unsigned long long* t = h + it * 20;
        printf("{\"n\": %d, \"threads\": %d, \"iter\": %d, \"cycles (loads, coarse, D placed, T found, R placed, published, all)\": [%lld, %lld, %lld, %lld, %lld, %lld, %lld]}\n", n, nt, it,
               (long long)(t[16] - t[15]), (long long)(t[17] - t[15]), (long long)(t[18] - t[15]), (long long)(t[11] - t[15]),
               (long long)(t[13] - t[15]), (long long)(t[19] - t[15]), (long long)(t[14] - t[15]));
        printf("   finisher: pass1 done %lld, scan done %lld\n", (long long)(t[1] - t[15]), (long long)(t[2] - t[15]));
      }
    }
  }
  return 0;
}
