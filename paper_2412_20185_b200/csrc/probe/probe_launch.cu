// Launch-latency probe: per-kernel time of back-to-back dependent launches captured in a CUDA
// graph, for empty kernels of various grid / block / dynamic-smem sizes, with and without
// programmatic dependent launch (PDL) and with early griddepcontrol.launch_dependents.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

__global__ void k_empty(int* p, int trigger, int spin) {
  extern __shared__ int sm[];
  if (trigger) asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (spin) { long long t0 = clock64(); while (clock64() - t0 < spin) {} }
  if (threadIdx.x == 0 && p) p[blockIdx.x] = (int)blockIdx.x + (int)(size_t)sm * 0;
}

int main() {
  CK(cudaSetDevice(0));
  CK(cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  int* d; CK(cudaMalloc(&d, 4096 * 4));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  printf("{\"launch\": [");
  bool first = true;
  struct C { int grid, block, smem, pdl, trigger, spin; };
  C cs[] = {{1, 32, 0, 0, 0, 0}, {1, 32, 0, 1, 1, 0}, {1, 1024, 0, 0, 0, 0}, {148, 288, 0, 0, 0, 0}, {148, 288, 0, 1, 1, 0},
            {148, 288, 180 * 1024, 0, 0, 0}, {148, 288, 180 * 1024, 1, 1, 0}, {148, 288, 180 * 1024, 1, 0, 0},
            {148, 288, 180 * 1024, 0, 0, 4000}, {148, 288, 180 * 1024, 1, 1, 4000}};
  for (C c : cs) {
    const int N = 64;
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < N; ++i) {
      cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(c.grid); cfg.blockDim = dim3(c.block); cfg.dynamicSmemBytes = c.smem; cfg.stream = st;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = c.pdl ? 1 : 0;
      CK(cudaLaunchKernelEx(&cfg, k_empty, d, c.trigger, c.spin));
    }
    CK(cudaStreamEndCapture(st, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, st)); CK(cudaStreamSynchronize(st));
    CK(cudaEventRecord(e0, st)); for (int r = 0; r < 10; ++r) CK(cudaGraphLaunch(ge, st)); CK(cudaEventRecord(e1, st)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("%s{\"grid\": %d, \"block\": %d, \"smem\": %d, \"pdl\": %d, \"trigger\": %d, \"spin_cycles\": %d, \"us_per_kernel\": %.3f}", first ? "" : ", ",
           c.grid, c.block, c.smem, c.pdl, c.trigger, c.spin, ms * 1e3 / (10 * N));
    first = false;
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
  }
  printf("]}\n");
  return 0;
}
