// Zero-copy PCIe read rate by request shape: does a TMA bulk copy (cp.async.bulk, one
// instruction moving P contiguous bytes from pinned host memory into smem) read the link
// faster than 128-B warp loads?  PCIe completion efficiency rises with the payload per TLP
// (128 B: ~84 %, 256 B: ~91 %), so if the copy engine path issues larger reads the residual
// gather could beat the 51.4 GB/s measured with loads.
//   bulk  : CTAs x one issuing thread; piece P bytes, ring of S slots (mbarrier per slot),
//           random piece addresses (row-gather-like) or sequential.
//   load  : the reference: 544-thread CTAs, 16-B loads, 8 in flight per thread.
// Output: JSON lines {mode, ctas, piece, slots, GBps}.
#include <cuda_runtime.h>
#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <vector>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1;} } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_bulk(const uint8_t* __restrict__ src, size_t span, uint32_t piece, int slots, int pieces_per_cta,
                       int random, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  uint8_t* buf = sm + 64 * 8;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < slots; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sa(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t n_pieces = span / piece;
  uint32_t acc = 0;
  for (int i = 0; i < pieces_per_cta; ++i) {
    const int s = i % slots;
    if (i >= slots) {  // wait for the slot's previous copy
      const uint32_t par = ((i / slots) - 1) & 1;
      uint32_t done = 0;
      do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(sa(&bar[s])), "r"(par) : "memory");
      } while (!done);
      acc += buf[(size_t)s * piece];
    }
    size_t pi = random ? ((size_t)(blockIdx.x * 2654435761u + i * 40503u) * 7919u) % n_pieces
                       : ((size_t)blockIdx.x * pieces_per_cta + i) % n_pieces;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(piece) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(buf + (size_t)s * piece)), "l"(src + pi * piece), "r"(piece), "r"(sa(&bar[s])) : "memory");
  }
  for (int i = pieces_per_cta; i < pieces_per_cta + slots; ++i) {  // drain
    const int s = i % slots;
    if (i >= slots) {
      const uint32_t par = ((i / slots) - 1) & 1;
      uint32_t done = 0;
      do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(sa(&bar[s])), "r"(par) : "memory");
      } while (!done);
      acc += buf[(size_t)s * piece];
    }
  }
  out[blockIdx.x] = acc;
}

__global__ void k_load(const uint4* __restrict__ src, size_t n16, int iters, uint32_t* out) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const size_t i = ((size_t)it * 8 + u) * stride + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + (i % n16)));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  const size_t span = (size_t)256 << 20;  // 256 MB pinned host
  uint8_t* h;
  CK(cudaHostAlloc(&h, span, cudaHostAllocMapped));
  for (size_t i = 0; i < span; i += 4096) h[i] = (uint8_t)i;
  uint8_t* d;
  CK(cudaHostGetDevicePointer(&d, h, 0));
  uint32_t* out;
  CK(cudaMalloc(&out, 1 << 24));
  CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch, double bytes, float& gbps) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    gbps = (float)(bytes / (best * 1e-3) / 1e9);
    return cudaGetLastError();
  };
  // reference: loads
  for (int ctas : {32, 148}) {
    const int iters = 64;
    const double bytes = (double)ctas * 544 * iters * 8 * 16;
    float g;
    CK(timeit([&] { k_load<<<ctas, 544>>>(reinterpret_cast<const uint4*>(d), span / 16, iters, out); }, bytes, g));
    printf("{\"mode\": \"load16\", \"ctas\": %d, \"GBps\": %.2f}\n", ctas, g);
  }
  for (int random : {1, 0})
    for (uint32_t piece : {128u, 256u, 512u, 1024u, 2048u, 4096u, 16384u})
      for (int ctas : {8, 32, 148}) {
        const int slots = (int)std::min<size_t>(48, (160 * 1024) / piece);
        const size_t per_cta_bytes = ((size_t)64 << 20) / ctas;  // 64 MB per launch
        const int ppc = (int)(per_cta_bytes / piece);
        const size_t smem = 64 * 8 + (size_t)slots * piece;
        const double bytes = (double)ctas * ppc * piece;
        float g;
        CK(timeit([&] { k_bulk<<<ctas, 32, smem>>>(d, span, piece, slots, ppc, random, out); }, bytes, g));
        printf("{\"mode\": \"bulk\", \"random\": %d, \"ctas\": %d, \"piece\": %u, \"slots\": %d, \"GBps\": %.2f}\n",
               random, ctas, piece, slots, g);
        fflush(stdout);
      }
  return 0;
}
