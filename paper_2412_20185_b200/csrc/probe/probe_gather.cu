// Random-row zero-copy gather probe: GB/s of fetching k residual rows (one 128-B line
// per row per warp-item, RB rows in flight per lane) from pinned host memory, for
// different host page backings (4 KB pinned, THP 2 MB + cudaHostRegister, hugetlbfs).
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <string>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

template <int RB, int VEC>  // VEC = bytes per lane per row (4 or 16)
__global__ void k_gather(const unsigned char* __restrict__ src, const int* __restrict__ rows, int k, int row_bytes,
                         int n_seg, unsigned* sink) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, ngw = (gridDim.x * blockDim.x) >> 5;
  const int seg_bytes = 32 * VEC;
  const int n_rb = (k + RB - 1) / RB;
  unsigned acc = 0;
  for (int item = gw; item < n_seg * n_rb; item += ngw) {
    const int seg = item % n_seg, rb = item / n_seg;
    unsigned v[RB][VEC / 4];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int rr = rb * RB + r;
      if (rr < k) {
        const unsigned char* p = src + (size_t)rows[rr] * row_bytes + seg * seg_bytes + lane * VEC;
        if (VEC == 16) {
          uint4 t;
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w) : "l"(p));
          v[r][0] = t.x; if (VEC / 4 > 1) { v[r][VEC / 4 > 1 ? 1 : 0] = t.y; v[r][VEC / 4 > 2 ? 2 : 0] = t.z; v[r][VEC / 4 > 3 ? 3 : 0] = t.w; }
        } else {
          unsigned t;
          asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(t) : "l"(p));
          v[r][0] = t;
        }
      } else {
        for (int q = 0; q < VEC / 4; ++q) v[r][q] = 0;
      }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r)
      for (int q = 0; q < VEC / 4; ++q) acc += v[r][q];
  }
  if (acc == 0x9999999u) sink[0] = acc;
}

struct Buf { unsigned char* p; size_t n; std::string kind; bool reg; };

static Buf alloc_kind(const char* kind, size_t n) {
  Buf b{nullptr, n, kind, false};
  if (!strcmp(kind, "cudaHostAlloc")) {
    void* h; CK(cudaHostAlloc(&h, n, cudaHostAllocMapped)); b.p = (unsigned char*)h; memset(h, 1, n);
  } else if (!strcmp(kind, "thp")) {
    void* h = mmap(nullptr, n + (2 << 20), PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (h == MAP_FAILED) return b;
    unsigned char* a = (unsigned char*)(((uintptr_t)h + (2 << 20) - 1) & ~((uintptr_t)(2 << 20) - 1));
    madvise(a, n, MADV_HUGEPAGE);
    memset(a, 1, n);
    if (cudaHostRegister(a, n, cudaHostRegisterMapped) != cudaSuccess) { cudaGetLastError(); return b; }
    b.p = a; b.reg = true;
  } else if (!strcmp(kind, "hugetlb")) {
    void* h = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_HUGETLB, -1, 0);
    if (h == MAP_FAILED) return b;
    memset(h, 1, n);
    if (cudaHostRegister(h, n, cudaHostRegisterMapped) != cudaSuccess) { cudaGetLastError(); return b; }
    b.p = (unsigned char*)h; b.reg = true;
  }
  return b;
}

int main() {
  CK(cudaSetDevice(0));
  unsigned* sink; CK(cudaMalloc(&sink, 4));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const size_t N = 512ull << 20;
  std::string js = "{\"gather\": [";
  bool first = true;
  for (const char* kind : {"cudaHostAlloc", "thp", "hugetlb"}) {
    Buf b = alloc_kind(kind, N);
    if (!b.p) { fprintf(stderr, "%s unavailable\n", kind); continue; }
    void* dptr; CK(cudaHostGetDevicePointer(&dptr, b.p, 0));
    for (int row_bytes : {2048, 7168}) {
      for (int k : {84, 294, 1024}) {
        for (int span_mb : {2, 512}) {
          const int nrows_span = (int)(((size_t)span_mb << 20) / row_bytes);
          std::vector<int> rows(k);
          srand(k + row_bytes);
          std::vector<int> perm(nrows_span); for (int i = 0; i < nrows_span; ++i) perm[i] = i;
          for (int i = 0; i < k && i < nrows_span; ++i) { int j = i + rand() % (nrows_span - i); std::swap(perm[i], perm[j]); }
          for (int i = 0; i < k; ++i) rows[i] = perm[i % nrows_span];
          std::sort(rows.begin(), rows.end());
          int* drows; CK(cudaMalloc(&drows, k * 4)); CK(cudaMemcpy(drows, rows.data(), k * 4, cudaMemcpyHostToDevice));
          for (int vec : {4, 16}) {
            const int n_seg = row_bytes / (32 * vec);
            for (int warps : {296, 1184}) {
              auto run = [&]() {
                if (vec == 4) k_gather<8, 4><<<warps / 4, 128>>>((const unsigned char*)dptr, drows, k, row_bytes, n_seg, sink);
                else k_gather<8, 16><<<warps / 4, 128>>>((const unsigned char*)dptr, drows, k, row_bytes, n_seg, sink);
              };
              run(); CK(cudaDeviceSynchronize());
              CK(cudaEventRecord(e0)); for (int r = 0; r < 10; ++r) run(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
              float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= 10;
              char buf[400];
              snprintf(buf, sizeof buf, "%s{\"kind\": \"%s\", \"row_bytes\": %d, \"k\": %d, \"span_mb\": %d, \"vec\": %d, \"warps\": %d, \"us\": %.2f, \"GBps\": %.2f}",
                       first ? "" : ", ", kind, row_bytes, k, span_mb, vec, warps, ms * 1e3, (double)k * row_bytes / (ms * 1e-3) / 1e9);
              js += buf; first = false;
            }
          }
          cudaFree(drows);
        }
      }
    }
    if (b.reg) cudaHostUnregister(b.p); else cudaFreeHost(b.p);
  }
  js += "]}";
  printf("%s\n", js.c_str());
  return 0;
}
