// Round-2 probe (cluster-split selection study, profiles/r02_s3_experiments.json).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o build/probe_coop_cluster paper_2412_20185_b200/csrc/probe/probe_coop_cluster.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) {
  unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  if (threadIdx.x == 0) p[blockIdx.x] = (int)r;
}
int main() {
  int* d; cudaMalloc(&d, 4096);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  for (int cs : {2, 4}) for (int grid : {148, 132, 136}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(544); cfg.dynamicSmemBytes = 150 * 1024;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, d);
    cudaError_t e2 = cudaDeviceSynchronize();
    int n = -1; cfg.numAttrs = 1; cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cs %d grid %d: launch %s sync %s maxActiveClusters %d\n", cs, grid, cudaGetErrorString(e), cudaGetErrorString(e2), n);
    cudaGetLastError();
  }
}
