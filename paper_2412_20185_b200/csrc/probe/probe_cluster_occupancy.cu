// Round-2 probe (cluster-split selection study, profiles/r02_s3_experiments.json).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o build/probe_cluster_occupancy paper_2412_20185_b200/csrc/probe/probe_cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int smems[] = {60 * 1024, 113 * 1024, 150 * 1024, 200 * 1024};
  for (int sm : smems)
    for (int cs = 1; cs <= 16; cs *= 2) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 64);
      cfg.blockDim = dim3(544);
      cfg.dynamicSmemBytes = sm;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %d KB cluster %d: max active clusters %d -> CTAs %d (%s)\n", sm / 1024, cs, n, n * cs, cudaGetErrorString(e));
    }
  int dev; cudaGetDevice(&dev); cudaDeviceProp pr; cudaGetDeviceProperties(&pr, dev);
  printf("SMs %d\n", pr.multiProcessorCount);
}
