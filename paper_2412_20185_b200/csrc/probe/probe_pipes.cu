// Pipe throughput of the GEMV's decode instructions on one SM (compute only, no memory):
// FHFMA (fma.rn.f32.f16), FFMA, HFMA2, LOP3, PRMT, IMAD, and the full 3-/4-bit decode bodies
// of decode.cuh with x in registers.  Reports lane-ops (or weights) per clock per SM.
// usage: probe_pipes [warps=16]
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../decode.cuh"
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1;} } while (0)

using namespace decdec;

__device__ __forceinline__ float fhfma(uint32_t a, uint32_t b, float c) {
  float d;
  asm volatile("{.reg .f16 al, ah, bl, bh;\n mov.b32 {al, ah}, %1;\n mov.b32 {bl, bh}, %2;\n fma.rn.f32.f16 %0, al, bl, %3;}"
               : "=f"(d) : "r"(a), "r"(b), "f"(c));
  return d;
}

// OP: 0 FHFMA, 1 FFMA (3-reg), 2 HFMA2, 3 LOP3, 4 PRMT, 5 IMAD, 6 LOP3+FHFMA (1:2),
//     7 w3 slice decode+FHFMA (32 weights / call), 8 w4 word x4 (32 weights / call)
template <int OP>
__global__ void k_pipe(int iters, uint32_t seed, float* out, long long* cyc) {
  const uint32_t t = threadIdx.x * 0x9E3779B9u + seed;
  uint32_t xr[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) xr[i] = (t * (i + 1)) & 0x3BFF3BFFu;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint32_t u[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) u[i] = t ^ (i * 0x01010101u);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (OP == 0) {
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i & 7] = fhfma(u[i & 7], xr[i], acc[i & 7]);
    } else if (OP == 1) {
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i & 7] = fmaf(__uint_as_float(u[i & 7]), __uint_as_float(xr[i]), acc[i & 7]);
    } else if (OP == 2) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        __half2 a = *reinterpret_cast<__half2*>(&u[i & 7]);
        __half2 b = *reinterpret_cast<__half2*>(&xr[i]);
        a = __hfma2(a, b, a);
        u[i & 7] = *reinterpret_cast<uint32_t*>(&a);
      }
    } else if (OP == 3) {
#pragma unroll
      for (int i = 0; i < 32; ++i) u[i & 7] = (u[i & 7] & xr[i]) ^ xr[i + 1];
    } else if (OP == 4) {
#pragma unroll
      for (int i = 0; i < 32; ++i) u[i & 7] = prmt(u[i & 7], xr[i], xr[i + 1]);
    } else if (OP == 5) {
#pragma unroll
      for (int i = 0; i < 32; ++i) u[i & 7] = u[i & 7] * xr[i] + xr[i + 1];
    } else if (OP == 6) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t m = u[i & 7] & 0x00070007u;
        acc[(2 * i) & 7] = fhfma_lo(m, xr[2 * i], acc[(2 * i) & 7]);
        acc[(2 * i + 1) & 7] = fhfma_hi(m, xr[2 * i], acc[(2 * i + 1) & 7]);
        u[i & 7] += 0x00010001u;
      }
    } else if (OP == 7) {
      float a[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int s = 0; s < 4; ++s) fma_w3_slice(u[3 * (s & 1)], u[3 * (s & 1) + 1], u[3 * (s & 1) + 2], xr + 16 * s, a);
      acc[it & 7] += combine_classes<3>(a);
      u[0] += 0x01010101u; u[1] ^= 0x11111111u; u[3] += 7u; u[4] ^= acc[0] > 0.f;
    } else if (OP == 8) {
      float a[4] = {0, 0, 0, 0};
#pragma unroll
      for (int s = 0; s < 16; ++s) fma_w4_word(u[s & 7], xr + 4 * s, a);
      acc[it & 7] += combine_classes<4>(a);
      u[0] += 0x01010101u; u[1] ^= 0x11111111u; u[3] += 7u;
    }
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i] + (float)(u[i] & 1);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
int run(const char* name, int warps, double per_iter_per_lane) {
  const int iters = 4096;
  float* out;
  long long* cyc;
  CK(cudaMalloc(&out, 148 * 1024 * 4));
  CK(cudaMalloc(&cyc, 148 * 8));
  k_pipe<OP><<<148, warps * 32>>>(16, 1, out, cyc);
  CK(cudaDeviceSynchronize());
  k_pipe<OP><<<148, warps * 32>>>(iters, 1, out, cyc);
  CK(cudaDeviceSynchronize());
  long long h[148];
  CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double ops = per_iter_per_lane * iters * warps * 32.0;
  printf("{\"op\": \"%s\", \"warps\": %d, \"per_sm_per_clk\": %.2f}\n", name, warps, ops / (double)mx);
  cudaFree(out);
  cudaFree(cyc);
  return 0;
}

int main(int argc, char** argv) {
  const int warps = argc > 1 ? atoi(argv[1]) : 16;
  run<0>("FHFMA lane-ops", warps, 32);
  run<1>("FFMA lane-ops", warps, 32);
  run<2>("HFMA2 lane-ops", warps, 32);
  run<3>("LOP3 lane-ops", warps, 64);
  run<4>("PRMT lane-ops", warps, 32);
  run<5>("IMAD lane-ops", warps, 32);
  run<6>("LOP3+2FHFMA weights", warps, 32);
  run<7>("w3 decode weights", warps, 128);
  run<8>("w4 decode weights", warps, 128);
  return 0;
}
