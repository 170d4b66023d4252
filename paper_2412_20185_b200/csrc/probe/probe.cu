// Link / pipe probes for the DecDEC roofline denominators.
// Measures on the box: FHFMA (fma.rn.f32.f16) issue rate and fp16-subnormal
// handling, zero-copy (GPU-initiated PCIe) read bandwidth and latency from pinned
// host memory, DMA H2D bandwidth, and whether sysmem lines are cached in L2.
// Prints one JSON object on stdout.  Standalone: nvcc -o probe probe.cu
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <string>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ float fhfma_lo(unsigned a2, unsigned b2, float c) {
  float d; unsigned short a = a2 & 0xffff, b = b2 & 0xffff;
  asm volatile("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c)); return d;
}
__device__ __forceinline__ float fhfma_hi(unsigned a2, unsigned b2, float c) {
  float d; unsigned short a = a2 >> 16, b = b2 >> 16;
  asm volatile("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c)); return d;
}

// Subnormal check: a = code*2^-24 (fp16 subnormal bit pattern = code), b = x.
__global__ void k_subnormal(const unsigned* a, const unsigned* b, float* out, int n) {
  int i = threadIdx.x + blockIdx.x * blockDim.x;
  if (i < n) { out[2*i] = fhfma_lo(a[i], b[i], 0.f); out[2*i+1] = fhfma_hi(a[i], b[i], 0.f); }
}

// FHFMA throughput: 8 independent accumulators, ITER iterations of 8 FHFMA each.
template <int ITER>
__global__ void k_fhfma_rate(unsigned seed, float* out) {
  unsigned a = seed ^ threadIdx.x, b = seed * 3u + threadIdx.x;
  float c0=0,c1=0,c2=0,c3=0,c4=0,c5=0,c6=0,c7=0;
  #pragma unroll 4
  for (int i = 0; i < ITER; ++i) {
    c0 = fhfma_lo(a, b, c0); c1 = fhfma_hi(a, b, c1); c2 = fhfma_lo(b, a, c2); c3 = fhfma_hi(b, a, c3);
    c4 = fhfma_lo(a, a, c4); c5 = fhfma_hi(a, a, c5); c6 = fhfma_lo(b, b, c6); c7 = fhfma_hi(b, b, c7);
  }
  float s = c0+c1+c2+c3+c4+c5+c6+c7;
  if (s == 1.2345f) out[threadIdx.x] = s;
}
// Mixed: per 8 weights 4 LOP3 + 8 FHFMA (4-bit GEMV inner-loop shape).
template <int ITER>
__global__ void k_mix_rate(unsigned seed, float* out) {
  unsigned w = seed ^ (threadIdx.x * 2654435761u), x0 = seed + threadIdx.x, x1 = x0 * 7u, x2 = x0 * 13u, x3 = x0 * 17u;
  float a0=0,a1=0,a2=0,a3=0;
  #pragma unroll 4
  for (int i = 0; i < ITER; ++i) {
    unsigned m0 = w & 0x000F000Fu, m1 = w & 0x00F000F0u, v = w >> 8, m2 = v & 0x000F000Fu, m3 = v & 0x00F000F0u;
    a0 = fhfma_lo(m0, x0, a0); a0 = fhfma_hi(m0, x0, a0);
    a1 = fhfma_lo(m1, x1, a1); a1 = fhfma_hi(m1, x1, a1);
    a2 = fhfma_lo(m2, x2, a2); a2 = fhfma_hi(m2, x2, a2);
    a3 = fhfma_lo(m3, x3, a3); a3 = fhfma_hi(m3, x3, a3);
    w = w * 1664525u + 1013904223u;
  }
  float s = a0+a1+a2+a3;
  if (s == 1.2345f) out[threadIdx.x] = s;
}

// Zero-copy streaming read: each warp reads `line` bytes per row-request, lanes
// cooperatively; UNR independent requests per lane in flight.
template <typename T, int UNR>
__global__ void k_zc_read(const T* __restrict__ src, size_t n_elems, unsigned long long* sink) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  unsigned long long acc = 0;
  for (size_t i = tid; i < n_elems; i += stride * UNR) {
    T v[UNR];
    #pragma unroll
    for (int u = 0; u < UNR; ++u) { size_t j = i + u * stride; if (j < n_elems) v[u] = src[j]; else v[u] = T{}; }
    #pragma unroll
    for (int u = 0; u < UNR; ++u) { const unsigned* p = reinterpret_cast<const unsigned*>(&v[u]); for (int q = 0; q < (int)(sizeof(T)/4); ++q) acc += p[q]; }
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

// Row-gather pattern like DEC: k rows of `row_bytes`; warp w takes 128B-segment s of every row.
__global__ void k_zc_rows(const unsigned* __restrict__ src, const int* __restrict__ rows, int k, int row_words, unsigned long long* sink) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nseg = row_words / 32;
  unsigned acc = 0;
  for (int seg = warp; seg < nseg; seg += (gridDim.x * blockDim.x) >> 5) {
    for (int r = 0; r < k; r += 8) {
      unsigned v[8];
      #pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (r + u < k) ? src[(size_t)rows[r + u] * row_words + seg * 32 + lane] : 0u;
      #pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// Pointer chase latency.
__global__ void k_chase(const unsigned* p, int steps, unsigned* out, long long* cyc) {
  unsigned i = 0; long long t0 = clock64();
  for (int s = 0; s < steps; ++s) i = p[i];
  long long t1 = clock64(); out[0] = i; cyc[0] = t1 - t0;
}

// bulk async copy from a (possibly host-mapped) global source into smem.
__global__ void k_bulk(const void* src, int bytes, unsigned* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  unsigned bar_a = (unsigned)__cvta_generic_to_shared(&bar);
  unsigned dst = (unsigned)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar_a));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar_a), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(dst), "l"(src), "r"(bytes), "r"(bar_a) : "memory");
    unsigned ok = 0;
    while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(bar_a));
  }
  __syncthreads();
  unsigned s = 0; for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) s += reinterpret_cast<unsigned*>(sm)[i];
  atomicAdd(out, s);
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) { float ms; CK(cudaEventElapsedTime(&ms, a, b)); return ms; }

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  std::string js = "{";
  char buf[512];
  snprintf(buf, sizeof buf, "\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"sm_clock_khz_attr\": %d, \"pci_bus\": %d, \"can_map_host\": %d",
           prop.name, prop.multiProcessorCount, prop.l2CacheSize, clk_khz, prop.pciBusID, prop.canMapHostMemory);
  js += buf;

  // 1. subnormal check
  {
    const int n = 16 * 256;
    std::vector<unsigned> a(n), b(n); std::vector<float> o(2 * n);
    for (int i = 0; i < n; ++i) {
      unsigned q0 = i & 15, q1 = (i >> 4) & 15;
      a[i] = q0 | (q1 << 16) | ((i & 1) ? 0x00400040u : 0u);   // also bits 6 (x64) in some
      __half hx0 = __float2half(((i % 97) - 48) * 0.37f + 1e-3f * i), hx1 = __float2half(-3.5f * (i % 13) + 0.001f);
      unsigned short u0, u1; memcpy(&u0, &hx0, 2); memcpy(&u1, &hx1, 2);
      b[i] = u0 | ((unsigned)u1 << 16);
    }
    unsigned *da, *db; float* dout;
    CK(cudaMalloc(&da, n * 4)); CK(cudaMalloc(&db, n * 4)); CK(cudaMalloc(&dout, 2 * n * 4));
    CK(cudaMemcpy(da, a.data(), n * 4, cudaMemcpyHostToDevice)); CK(cudaMemcpy(db, b.data(), n * 4, cudaMemcpyHostToDevice));
    k_subnormal<<<n / 256, 256>>>(da, db, dout, n); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(o.data(), dout, 2 * n * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < n; ++i) {
      for (int h = 0; h < 2; ++h) {
        unsigned short ah = h ? (a[i] >> 16) : (a[i] & 0xffff), bh = h ? (b[i] >> 16) : (b[i] & 0xffff);
        __half ha, hb; memcpy(&ha, &ah, 2); memcpy(&hb, &bh, 2);
        double ref = (double)__half2float(ha) * (double)__half2float(hb);
        if ((double)o[2 * i + h] != ref) ++bad;
      }
    }
    snprintf(buf, sizeof buf, ", \"fhfma_subnormal_exact\": %s, \"fhfma_subnormal_bad\": %d", bad ? "false" : "true", bad);
    js += buf;
    cudaFree(da); cudaFree(db); cudaFree(dout);
  }
  float* dsink; CK(cudaMalloc(&dsink, 4096));
  // 2. FHFMA rate
  {
    const int IT = 4096; int blocks = prop.multiProcessorCount * 8, thr = 256;
    k_fhfma_rate<IT><<<blocks, thr>>>(1u, dsink); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); for (int r = 0; r < 5; ++r) k_fhfma_rate<IT><<<blocks, thr>>>(r, dsink); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    double ms = time_ms(e0, e1) / 5; double ops = (double)blocks * thr * IT * 8;
    snprintf(buf, sizeof buf, ", \"fhfma_lane_ops_per_s\": %.4g, \"fhfma_ms\": %.4f", ops / (ms * 1e-3), ms); js += buf;
    k_mix_rate<IT><<<blocks, thr>>>(1u, dsink); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0)); for (int r = 0; r < 5; ++r) k_mix_rate<IT><<<blocks, thr>>>(r, dsink); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    ms = time_ms(e0, e1) / 5; double w = (double)blocks * thr * IT * 8;
    snprintf(buf, sizeof buf, ", \"mix4_weights_per_s\": %.4g", w / (ms * 1e-3)); js += buf;
  }
  // 3. zero-copy read bandwidth
  size_t zc_bytes = 256ull << 20;
  for (int wc = 0; wc < 2; ++wc) {
    void* h; CK(cudaHostAlloc(&h, zc_bytes, cudaHostAllocMapped | (wc ? cudaHostAllocWriteCombined : 0)));
    memset(h, 1, zc_bytes);
    void* dptr; CK(cudaHostGetDevicePointer(&dptr, h, 0));
    unsigned long long* sink = (unsigned long long*)dsink;
    struct Cfg { int blocks, thr, vec, unr; };
    std::vector<Cfg> cfgs = {{148, 256, 16, 4}, {148, 256, 4, 8}, {296, 512, 16, 8}, {148, 64, 16, 4}, {148, 32, 16, 4}, {32, 256, 16, 4}, {148, 128, 4, 8}, {592, 256, 16, 2}};
    js += wc ? ", \"zc_wc\": [" : ", \"zc\": [";
    bool first = true;
    for (auto c : cfgs) {
      auto run = [&]() {
        if (c.vec == 16) { if (c.unr == 4) k_zc_read<uint4, 4><<<c.blocks, c.thr>>>((const uint4*)dptr, zc_bytes / 16, sink);
                           else if (c.unr == 8) k_zc_read<uint4, 8><<<c.blocks, c.thr>>>((const uint4*)dptr, zc_bytes / 16, sink);
                           else k_zc_read<uint4, 2><<<c.blocks, c.thr>>>((const uint4*)dptr, zc_bytes / 16, sink); }
        else k_zc_read<unsigned, 8><<<c.blocks, c.thr>>>((const unsigned*)dptr, zc_bytes / 4, sink);
      };
      run(); CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0)); for (int r = 0; r < 3; ++r) run(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      double ms = time_ms(e0, e1) / 3;
      snprintf(buf, sizeof buf, "%s{\"blocks\": %d, \"thr\": %d, \"vec\": %d, \"unr\": %d, \"GBps\": %.2f}", first ? "" : ", ", c.blocks, c.thr, c.vec, c.unr, zc_bytes / (ms * 1e-3) / 1e9);
      js += buf; first = false;
    }
    js += "]";
    // row-gather pattern: rows of 2048 B (d_out 4096), k selected rows
    if (!wc) {
      int row_words = 512, nrows = (int)(zc_bytes / (row_words * 4));
      std::vector<int> rows(4096); for (int i = 0; i < 4096; ++i) rows[i] = (int)(((long long)i * 7919) % nrows);
      int* drows; CK(cudaMalloc(&drows, rows.size() * 4)); CK(cudaMemcpy(drows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
      js += ", \"zc_rows\": [";
      int ks[] = {84, 336, 1024, 4096}; bool f2 = true;
      for (int k : ks) for (int wpb : {1, 4}) {
        int blocks = 16 / wpb; // 16 segments of 128B per 2048-B row
        k_zc_rows<<<blocks, 32 * wpb>>>((const unsigned*)dptr, drows, k, row_words, sink); CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0)); for (int r = 0; r < 5; ++r) k_zc_rows<<<blocks, 32 * wpb>>>((const unsigned*)dptr, drows, k, row_words, sink); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        double us = time_ms(e0, e1) / 5 * 1e3;
        snprintf(buf, sizeof buf, "%s{\"k\": %d, \"warps\": 16, \"wpb\": %d, \"us\": %.3f, \"GBps\": %.2f}", f2 ? "" : ", ", k, wpb, us, (double)k * 2048 / (us * 1e-6) / 1e9);
        js += buf; f2 = false;
      }
      js += "]";
      cudaFree(drows);
      // L2 caching of sysmem: read 8 MB twice in one kernel sequence
      size_t small = 8ull << 20;
      k_zc_read<uint4, 4><<<148, 256>>>((const uint4*)dptr, small / 16, sink); CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0)); k_zc_read<uint4, 4><<<148, 256>>>((const uint4*)dptr, small / 16, sink); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      double ms_re = time_ms(e0, e1);
      snprintf(buf, sizeof buf, ", \"zc_reread_8MB_GBps\": %.2f", small / (ms_re * 1e-3) / 1e9); js += buf;
      // latency chase over host memory (stride 4 KB random)
      {
        int nnodes = 4096; std::vector<unsigned> perm(nnodes); for (int i = 0; i < nnodes; ++i) perm[i] = i;
        srand(1); for (int i = nnodes - 1; i > 0; --i) std::swap(perm[i], perm[rand() % (i + 1)]);
        unsigned* hp = (unsigned*)h; size_t strideW = 1024;
        for (int i = 0; i < nnodes; ++i) hp[perm[i] * strideW] = perm[(i + 1) % nnodes] * strideW;
        unsigned* dout; long long* dcyc; CK(cudaMalloc(&dout, 4)); CK(cudaMalloc(&dcyc, 8));
        k_chase<<<1, 1>>>((const unsigned*)dptr, 256, dout, dcyc); CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0)); k_chase<<<1, 1>>>((const unsigned*)dptr, 2048, dout, dcyc); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        long long cyc; CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
        snprintf(buf, sizeof buf, ", \"zc_latency_ns\": %.1f, \"zc_latency_cycles\": %.1f", time_ms(e0, e1) * 1e6 / 2048, cyc / 2048.0); js += buf;
        // device memory chase for comparison
        unsigned* dmem; CK(cudaMalloc(&dmem, nnodes * strideW * 4));
        CK(cudaMemcpy(dmem, hp, nnodes * strideW * 4, cudaMemcpyHostToDevice));
        k_chase<<<1, 1>>>(dmem, 256, dout, dcyc); CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0)); k_chase<<<1, 1>>>(dmem, 2048, dout, dcyc); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
        snprintf(buf, sizeof buf, ", \"hbm_chase_ns\": %.1f, \"hbm_chase_cycles\": %.1f", time_ms(e0, e1) * 1e6 / 2048, cyc / 2048.0); js += buf;
        cudaFree(dmem); cudaFree(dout); cudaFree(dcyc);
      }
      // bulk copy from host-mapped source
      {
        unsigned* dcnt; CK(cudaMalloc(&dcnt, 4)); CK(cudaMemset(dcnt, 0, 4));
        memset(h, 0, 4096); ((unsigned*)h)[5] = 77;
        CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
        k_bulk<<<1, 128, 65536>>>(dptr, 4096, dcnt);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned cnt = 0; if (e == cudaSuccess) CK(cudaMemcpy(&cnt, dcnt, 4, cudaMemcpyDeviceToHost));
        snprintf(buf, sizeof buf, ", \"bulk_from_host\": \"%s\", \"bulk_from_host_sum\": %u", cudaGetErrorString(e), cnt); js += buf;
        if (e != cudaSuccess) { cudaGetLastError(); }
      }
    }
    // DMA H2D
    if (!wc) {
      void* dbuf; CK(cudaMalloc(&dbuf, zc_bytes));
      CK(cudaMemcpy(dbuf, h, zc_bytes, cudaMemcpyHostToDevice));
      CK(cudaEventRecord(e0)); CK(cudaMemcpyAsync(dbuf, h, zc_bytes, cudaMemcpyHostToDevice)); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      snprintf(buf, sizeof buf, ", \"dma_h2d_GBps\": %.2f", zc_bytes / (time_ms(e0, e1) * 1e-3) / 1e9); js += buf;
      CK(cudaEventRecord(e0)); CK(cudaMemcpyAsync(h, dbuf, zc_bytes, cudaMemcpyDeviceToHost)); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      snprintf(buf, sizeof buf, ", \"dma_d2h_GBps\": %.2f", zc_bytes / (time_ms(e0, e1) * 1e-3) / 1e9); js += buf;
      // HBM copy
      void* dbuf2; CK(cudaMalloc(&dbuf2, zc_bytes));
      CK(cudaMemcpy(dbuf2, dbuf, zc_bytes, cudaMemcpyDeviceToDevice));
      CK(cudaEventRecord(e0)); for (int r = 0; r < 5; ++r) CK(cudaMemcpyAsync(dbuf2, dbuf, zc_bytes, cudaMemcpyDeviceToDevice)); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      snprintf(buf, sizeof buf, ", \"d2d_copy_GBps_rw\": %.2f", 2.0 * zc_bytes * 5 / (time_ms(e0, e1) * 1e-3) / 1e9); js += buf;
      cudaFree(dbuf); cudaFree(dbuf2);
    }
    CK(cudaFreeHost(h));
  }
  js += "}";
  printf("%s\n", js.c_str());
  return 0;
}
