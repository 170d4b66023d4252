// Micro-latency probe of the primitives the selector is built from (1 CTA):
// __syncthreads at 4/32 warps, dependent SHFL / VOTE / LDS chains, L2-hit global load.
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1;} } while (0)

__global__ void k_prims(const unsigned* g, unsigned long long* out, int nsync) {
  __shared__ unsigned sm[1024];
  unsigned v = threadIdx.x;
  sm[threadIdx.x] = v;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < nsync; ++i) __syncthreads();
  long long t1 = clock64();
  for (int i = 0; i < 64; ++i) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
  long long t2 = clock64();
  for (int i = 0; i < 64; ++i) v = __ballot_sync(0xffffffffu, v & 1) + v;
  long long t3 = clock64();
  for (int i = 0; i < 64; ++i) v = sm[(v + i) & 1023];
  long long t4 = clock64();
  unsigned idx = v & 1023;
  for (int i = 0; i < 16; ++i) idx = g[idx] & 1023;
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / (nsync ? nsync : 1);
    out[1] = (t2 - t1) / 64;
    out[2] = (t3 - t2) / 64;
    out[3] = (t4 - t3) / 64;
    out[4] = (t5 - t4) / 16;
    out[5] = idx + v;
  }
}

int main() {
  unsigned* g; unsigned long long* o;
  CK(cudaMalloc(&g, 4096 * 4)); CK(cudaMalloc(&o, 64));
  CK(cudaMemset(g, 0, 4096 * 4));
  unsigned long long h[6];
  for (int nt : {128, 1024}) {
    for (int rep = 0; rep < 3; ++rep) k_prims<<<1, nt>>>(g, o, 100);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, o, 48, cudaMemcpyDeviceToHost));
    printf("{\"threads\": %d, \"syncthreads_cyc\": %llu, \"shfl_dep_cyc\": %llu, \"ballot_dep_cyc\": %llu, \"lds_dep_cyc\": %llu, \"ldg_l2_dep_cyc\": %llu}\n",
           nt, h[0], h[1], h[2], h[3], h[4]);
  }
  return 0;
}
