// Round-2 probe (cluster-split selection study, profiles/r02_s3_experiments.json).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o build/probe_cluster_barrier paper_2412_20185_b200/csrc/probe/probe_cluster_barrier.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__global__ void __launch_bounds__(544, 1) k(long long* out, int mode) {
  extern __shared__ int sm[];
  long long t0 = clock64();
  if (mode == 0) cluster_sync();
  else { asm volatile("barrier.cluster.arrive;\n\tbarrier.cluster.wait;" ::: "memory"); }
  long long t1 = clock64();
  cluster_sync();
  long long t2 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t1; }
  sm[threadIdx.x] = 0;
}
int main() {
  long long* d; cudaMalloc(&d, 1 << 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  for (int cs : {2, 4}) for (int coop : {0, 1}) for (int mode : {0, 1}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs == 4 ? 132 : 148); cfg.blockDim = dim3(544); cfg.dynamicSmemBytes = 120 * 1024;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = 1 + coop;
    for (int rep = 0; rep < 3; ++rep) { cudaLaunchKernelEx(&cfg, k, d, mode); }
    cudaError_t e = cudaDeviceSynchronize();
    long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("cs %d coop %d mode %d: %s first %lld second %lld cycles\n", cs, coop, mode, cudaGetErrorString(e), h[0], h[1]);
  }
}
