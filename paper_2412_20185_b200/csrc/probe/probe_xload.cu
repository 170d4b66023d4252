// Latency of the first global loads in a kernel: 148 CTAs x 288 threads.  Phases (clock64):
//   A: one dependent 16-B load; B: 16 independent 16-B loads (the consumer's x fetch);
//   C: 16 more (same lines, L1/L2 hit); D: one dependent load of a different 2 MB page.
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1;} } while (0)

__device__ __forceinline__ uint4 ldv(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__shared__ unsigned sink[288];
__device__ __forceinline__ long long clk(unsigned dep) {
  long long t;
  asm volatile("st.volatile.shared.u32 [%1], %2;\n\tmov.u64 %0, %%clock64;" : "=l"(t) : "r"((unsigned)__cvta_generic_to_shared(&sink[threadIdx.x])), "r"(dep) : "memory");
  return t;
}

__global__ void k_x(const uint4* x, const uint4* far, long long* out) {
  long long t[5];
  t[0] = clk(0);
  uint4 a = ldv(x + 600);
  t[1] = clk(a.x);
  const uint4* xp = x + (threadIdx.x & 31) * 16;
  uint4 v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = ldv(xp + i);
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i].x ^ v[i].y ^ v[i].z ^ v[i].w;
  t[2] = clk(s);
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = ldv(xp + i + 1);
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i].x ^ v[i].y ^ v[i].z ^ v[i].w;
  t[3] = clk(s);
  uint4 b = ldv(far + blockIdx.x * 64 + (s & 1));
  t[4] = clk(b.y);
  if (threadIdx.x == 32)
    for (int i = 0; i < 4; ++i) out[blockIdx.x * 4 + i] = t[i + 1] - t[i];
  if ((a.y ^ b.x ^ s) == 0x12345679u) out[0] = 0;
}
__global__ void k_flush(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = make_uint4(i, i, i, i);
}

int main() {
  uint4* x; uint4* big; long long* o;
  CK(cudaMalloc(&x, 16384)); CK(cudaMalloc(&big, 256u << 20)); CK(cudaMalloc(&o, 148 * 4 * 8));
  CK(cudaMemset(x, 1, 16384));
  const uint4* far = big + (64u << 20) / 16;
  long long h[148 * 4];
  const char* names[4] = {"A_one_load", "B_16_loads", "C_16_hits", "D_far_page"};
  for (int cold = 0; cold < 2; ++cold)
    for (int rep = 0; rep < 3; ++rep) {
      if (cold) k_flush<<<1184, 256>>>(big, (256u << 20) / 16);
      CK(cudaDeviceSynchronize());
      k_x<<<148, 288>>>(x, far, o);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(h, o, sizeof h, cudaMemcpyDeviceToHost));
      printf("{\"cold\": %d, \"rep\": %d", cold, rep);
      for (int p = 0; p < 4; ++p) {
        double avg = 0; long long mx = 0;
        for (int i = 0; i < 148; ++i) { avg += h[i * 4 + p]; mx = h[i * 4 + p] > mx ? h[i * 4 + p] : mx; }
        printf(", \"%s\": [%.0f, %lld]", names[p], avg / 148, mx);
      }
      printf("}\n");
    }
  return 0;
}
