// per-SM zero-copy gather: which in-flight limit applies (instructions vs lines), LDG vs cp.async
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
// MODE 0: LDG 4B/lane, 1 row (128 B) per instr; 1: LDG 16B/lane contiguous 512 B of one row;
// 2: LDG 16B/lane, 4 random rows x 128 B per instr; 3: cp.async 4B/lane 1 row; 4: cp.async 16B 4 rows
template <int MODE>
__global__ void k(const unsigned char* src, size_t nrows, int iters, unsigned long long* sink) {
  extern __shared__ __align__(16) unsigned char smraw[];
  auto sm = reinterpret_cast<unsigned char (*)[2][8 * 512]>(smraw);
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned acc = 0;
  unsigned long long h = 1469598103934665603ull * (warp + 1);
  for (int it = 0; it < iters; ++it) {
    unsigned v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h = h * 6364136223846793005ull + 1442695040888963407ull;
      size_t row = (h >> 20) % nrows;
      if (MODE == 2 || MODE == 4) {  // each 8-lane group its own row
        unsigned long long hh = h ^ (0x9E3779B97F4A7C15ull * (lane >> 3));
        hh = hh * 6364136223846793005ull + 1442695040888963407ull;
        row = (hh >> 20) % nrows;
      }
      const unsigned char* p;
      if (MODE == 0 || MODE == 3) p = src + row * 2048 + lane * 4;
      else if (MODE == 1) p = src + row * 2048 + lane * 16;
      else p = src + row * 2048 + (lane & 7) * 16;
      if (MODE == 0) { unsigned q; asm volatile("ld.global.cv.u32 %0, [%1];" : "=r"(q) : "l"(p)); v[u] = q; }
      else if (MODE <= 2) { uint4 q; asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "l"(p)); v[u] = q.x ^ q.w; }
      else {
        unsigned d = (unsigned)__cvta_generic_to_shared(&sm[wl][it & 1][u * 512 + lane * (MODE == 3 ? 4 : 16)]);
        if (MODE == 3) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(d), "l"(p));
        else asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(d), "l"(p));
        v[u] = 0;
      }
    }
    if (MODE >= 3) { asm volatile("cp.async.commit_group;"); asm volatile("cp.async.wait_group 1;"); }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  if (MODE >= 3) asm volatile("cp.async.wait_group 0;");
  acc += sm[wl][0][lane];
  if (acc == 0x12345u) sink[0] = acc;
}
int main() {
  size_t bytes = 1ull << 30;
  void* h; CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
  memset(h, 1, bytes);
  unsigned char* d; CK(cudaHostGetDevicePointer((void**)&d, h, 0));
  unsigned long long* sink; CK(cudaMalloc(&sink, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072); cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072); cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072); cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072); cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  int nbs[] = {1, 4, 16, 32, 64};
  const char* names[] = {"ldg4_1row", "ldg16_512B", "ldg16_4rows", "cpasync4_1row", "cpasync16_4rows"};
  for (int mode = 0; mode < 5; ++mode) for (int nb : nbs) {
    const int iters = 64;
    auto launch = [&]() {
      if (mode == 0) k<0><<<nb, 512, 131072>>>(d, bytes / 2048, iters, sink);
      if (mode == 1) k<1><<<nb, 512, 131072>>>(d, bytes / 2048, iters, sink);
      if (mode == 2) k<2><<<nb, 512, 131072>>>(d, bytes / 2048, iters, sink);
      if (mode == 3) k<3><<<nb, 512, 131072>>>(d, bytes / 2048, iters, sink);
      if (mode == 4) k<4><<<nb, 512, 131072>>>(d, bytes / 2048, iters, sink);
    };
    launch(); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double B = (double)nb * 16 * iters * 8 * (mode == 0 || mode == 3 ? 128 : 512);
    printf("{\"mode\": \"%s\", \"ctas\": %d, \"GBps\": %.2f, \"per_sm_GBps\": %.2f}\n", names[mode], nb, B / (ms * 1e-3) / 1e9, B / (ms * 1e-3) / 1e9 / nb);
  }
}
