// Cooperative launch x programmatic dependent launch (PDL) on sm_100a: does a grid launched
// with BOTH cudaLaunchAttributeCooperative and programmatic stream serialization start
// early (while the previous kernel still runs) when both grids fit on the GPU together, and
// does it wait (instead of failing or hanging) when they do not?
// Kernel A: one CTA per SM (grid = #SMs), spins `spin_ns` after griddepcontrol.launch_dependents.
// Kernel B: grid = #SMs, records %globaltimer at entry (before griddepcontrol.wait).
// Output: B's first-CTA start relative to A's end (negative = overlapped).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1;} } while (0)

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

__global__ void k_a(unsigned long long* ts, unsigned long long spin_ns) {
  extern __shared__ int sm[];
  asm volatile("griddepcontrol.launch_dependents;");
  const uint64_t t0 = gt();
  while (gt() - t0 < spin_ns) {}
  if (threadIdx.x == 0) { ts[blockIdx.x] = gt(); sm[0] = 1; }
}

__global__ void k_b(unsigned long long* ts) {
  extern __shared__ int sm[];
  const uint64_t t = gt();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) { ts[blockIdx.x] = t; sm[0] = 2; }
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int coop; CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, 0));
  CK(cudaFuncSetAttribute(k_a, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(k_b, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  unsigned long long *ta, *tb; CK(cudaMalloc(&ta, 4096 * 8)); CK(cudaMalloc(&tb, 4096 * 8));
  cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  printf("{\"sms\": %d, \"coop_attr\": %d, \"cases\": [", sms, coop);
  struct C { int a_smem_kb, b_smem_kb, pdl, coop, graph; };
  C cs[] = {{100, 100, 1, 0, 0}, {100, 100, 1, 1, 0}, {150, 100, 1, 1, 0}, {150, 100, 1, 0, 0}, {100, 100, 0, 1, 0},
            {100, 100, 1, 1, 1}, {150, 100, 1, 1, 1}};
  bool first = true;
  for (C c : cs) {
    unsigned long long ha[4096], hb[4096];
    cudaError_t eb = cudaSuccess;
    auto enqueue = [&]() {
      k_a<<<sms, 128, c.a_smem_kb * 1024, st>>>(ta, 20000ull);
      cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(sms); cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = c.b_smem_kb * 1024; cfg.stream = st;
      cudaLaunchAttribute at[2]; int n = 0;
      if (c.pdl) { at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[n].val.programmaticStreamSerializationAllowed = 1; ++n; }
      if (c.coop) { at[n].id = cudaLaunchAttributeCooperative; at[n].val.cooperative = 1; ++n; }
      cfg.attrs = at; cfg.numAttrs = n;
      eb = cudaLaunchKernelEx(&cfg, k_b, tb);
    };
    if (c.graph) {
      cudaGraph_t g; cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      enqueue();
      cudaError_t ee = cudaStreamEndCapture(st, &g);
      if (eb == cudaSuccess && ee == cudaSuccess) eb = cudaGraphInstantiate(&ge, g, 0);
      else if (eb == cudaSuccess) eb = ee;
      if (eb == cudaSuccess) { eb = cudaGraphLaunch(ge, st); }
    } else {
      enqueue();
    }
    cudaError_t es = cudaStreamSynchronize(st);
    cudaGetLastError();
    double overlap_us = 0, b_span_us = 0;
    if (eb == cudaSuccess && es == cudaSuccess) {
      CK(cudaMemcpy(ha, ta, sms * 8, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(hb, tb, sms * 8, cudaMemcpyDeviceToHost));
      unsigned long long a_end = 0, b_first = ~0ull, b_last = 0;
      for (int i = 0; i < sms; ++i) { if (ha[i] > a_end) a_end = ha[i]; if (hb[i] < b_first) b_first = hb[i]; if (hb[i] > b_last) b_last = hb[i]; }
      overlap_us = ((double)b_first - (double)a_end) / 1e3;
      b_span_us = ((double)b_last - (double)b_first) / 1e3;
    }
    printf("%s{\"a_smem_kb\": %d, \"b_smem_kb\": %d, \"pdl\": %d, \"coop\": %d, \"graph\": %d, \"launch\": \"%s\", \"sync\": \"%s\", "
           "\"b_first_start_minus_a_end_us\": %.2f, \"b_start_span_us\": %.2f}",
           first ? "" : ", ", c.a_smem_kb, c.b_smem_kb, c.pdl, c.coop, c.graph, cudaGetErrorString(eb), cudaGetErrorString(es), overlap_us,
           b_span_us);
    first = false;
  }
  printf("]}\n");
  return 0;
}
