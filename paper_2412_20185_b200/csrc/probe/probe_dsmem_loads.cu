// Round-2 probe (cluster-split selection study, profiles/r02_s3_experiments.json).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o build/probe_dsmem_loads paper_2412_20185_b200/csrc/probe/probe_dsmem_loads.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t ld_dsmem(const void* p, uint32_t rank) {
  uint32_t a, v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_addr(p)), "r"(rank));
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__global__ void __launch_bounds__(544, 1) k(long long* out, int CS) {
  extern __shared__ uint32_t sm[];
  uint32_t cr; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
  for (int i = threadIdx.x; i < 4 * 296; i += blockDim.x) sm[i] = i;
  cluster_sync();
  long long t0 = clock64();
  uint32_t c = 0;
  const int lane = threadIdx.x & 31;
  for (int r = 1; r < CS; ++r) {
    uint32_t rr = (cr + r) % CS, h[32];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int cp = 0; cp < 4; ++cp) h[j * 4 + cp] = ld_dsmem(&sm[cp * 296 + 9 * lane + j], rr);
#pragma unroll
    for (int i = 0; i < 32; ++i) c += h[i];
  }
  long long t1 = clock64();
  cluster_sync();
  if (threadIdx.x == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = c; }
}
int main() {
  long long* d; cudaMalloc(&d, 1 << 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  for (int cs : {2, 4}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs == 4 ? 132 : 148); cfg.blockDim = dim3(544); cfg.dynamicSmemBytes = 120 * 1024;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = 2;
    for (int rep = 0; rep < 3; ++rep) cudaLaunchKernelEx(&cfg, k, d, cs);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("cs %d: %s dsmem phase %lld cycles (sum %lld)\n", cs, cudaGetErrorString(e), h[0], h[1]);
  }
}
