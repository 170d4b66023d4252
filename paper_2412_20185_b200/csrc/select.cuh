// Step (1) of DecDEC: exact Top-k of |x| ("Exact").
//
// Replaces the paper's 32-bucket approximate, randomly-filled chunk Top-K with
// an exact, deterministic selection on the 15-bit magnitude key bits(x) & 0x7FFF (ledger L2).
// One CTA per segment (the whole x for chunk = 0, one chunk otherwise):
//   1. every thread holds R = 8C contiguous elements in registers; one smem atomicAdd per
//      element into a 256-bin histogram of key >> 7 (measured ~4 SMSP cycles per warp-op;
//      activation exponents spread the bins, so lanes rarely collide);
//   2. one warp finds the bin holding the q-th largest key (lane l owns 8 contiguous bins,
//      suffix scan over lanes), then a 128-bin histogram of key & 127 over that bin's
//      elements gives the exact threshold T, `above` = #keys > T, need = q - above ties;
//   3. per-thread counts of key > T / key == T, one block exclusive scan in index order,
//      then each thread writes its selected indices (ties: lowest index first).
// Output ascending by index.  No per-element warp collectives (ballots cost ~8 SMSP
// cycles each on B200) and a handful of barriers.
#pragma once
#include <cstdint>
#include "ptx.cuh"

namespace decdec {

constexpr int kSelMaxWarps = 32;
constexpr int kSelMaxThreads = 1024;

// Exclusive scan of v over the block in thread order (warp shuffles + one warp over the warp
// totals).  `tmp` holds >= 32 words.  Two barriers.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* tmp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t s = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += s;
  }
  if (lane == 31) tmp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const uint32_t wt = lane < nw ? tmp[lane] : 0u;
    uint32_t wi = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t s = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += s;
    }
    tmp[lane] = wi - wt;
  }
  __syncthreads();
  return tmp[wid] + inc - v;
}

// grid = number of segments; blockDim = NT (multiple of 32, <= 1024) with NT * 8C >= len;
// dynamic smem = select_smem_bytes().
template <int C>
__global__ void __launch_bounds__(kSelMaxThreads) k_select(const uint16_t* __restrict__ x, int d_in, int k, int chunk,
                                                           int* __restrict__ idx_out, uint16_t* __restrict__ xs_out,
                                                           int* __restrict__ sel_out, unsigned long long* trace) {
  constexpr int R = 8 * C;
  if (trace && threadIdx.x == 0 && blockIdx.x == 0) {
    trace[0] = globaltimer();
    trace[2 + 1024 * 9 - 2] = clock64();
  }
  // Programmatic dependent launch: the fused layer kernel that follows may start its HBM
  // weight stream now; only its gather warps wait (griddepcontrol.wait) for our results.
  pdl_launch_dependents();
  __shared__ uint32_t histA[256];
  __shared__ uint32_t histB[128];
  __shared__ uint32_t tmp[kSelMaxWarps];
  __shared__ uint32_t s_bA, s_aboveA, s_T, s_need;
  const int seg = blockIdx.x;
  const int a = chunk ? seg * chunk : 0;
  const int n = chunk ? min(chunk, d_in - a) : d_in;
  const int q = chunk ? min(k, n) : k;
  const int out_off = chunk ? seg * k : 0;  // every earlier chunk is full length >= k
  if (q <= 0) return;
  const int t = threadIdx.x, NT = blockDim.x, lane = t & 31;
#define SEL_PHASE(i) \
  if (trace && t == 0 && blockIdx.x == 0) trace[2 + 1024 * 9 - 16 + (i)] = clock64();

  // R contiguous elements per thread (16-B loads in flight while the histograms are zeroed)
  const int base = t * R;
  uint32_t raw[R / 2];
#pragma unroll
  for (int v = 0; v < C; ++v) {
    uint4 q4 = make_uint4(0, 0, 0, 0);
    if (base + 8 * v < n) q4 = __ldg(reinterpret_cast<const uint4*>(x + a + base) + v);
    raw[4 * v + 0] = q4.x; raw[4 * v + 1] = q4.y; raw[4 * v + 2] = q4.z; raw[4 * v + 3] = q4.w;
  }
  const int nv = n - base;  // slot e < nv is a real element
  auto key_of = [&](int e) -> uint32_t { return ((e & 1) ? (raw[e >> 1] >> 16) : raw[e >> 1]) & 0x7fffu; };
  for (int i = t; i < 256; i += NT) histA[i] = 0;
  for (int i = t; i < 128; i += NT) histB[i] = 0;
  __syncthreads();
  SEL_PHASE(0);

  // ---- 1. coarse histogram (key >> 7)
#pragma unroll
  for (int e = 0; e < R; ++e)
    if (e < nv) atomicAdd(&histA[key_of(e) >> 7], 1u);
  __syncthreads();
  SEL_PHASE(1);
  // ---- 2a. warp 0: bin of the q-th largest key; lane l owns bins [8l, 8l + 8)
  if (t < 32) {
    uint32_t c[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c[j] = histA[8 * lane + j];
      sum += c[j];
    }
    // keys above lane l's bins = sum over lanes > l: inclusive scan over reversed lanes
    const uint32_t sr = __shfl_sync(0xffffffffu, sum, 31 - lane);
    uint32_t inc = sr;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    // inc at reversed position r = 31 - l is sum over lanes >= l; above_l = that - sum_l
    const uint32_t above = __shfl_sync(0xffffffffu, inc, 31 - lane) - sum;
    if (above < (uint32_t)q && above + sum >= (uint32_t)q) {
      uint32_t run = above;
#pragma unroll
      for (int j = 7; j >= 0; --j) {
        if (run + c[j] >= (uint32_t)q) {
          s_bA = 8 * lane + j;
          s_aboveA = run;
          break;
        }
        run += c[j];
      }
    }
  }
  __syncthreads();
  const uint32_t bA = s_bA, aboveA = s_aboveA;
  // ---- 2b. fine histogram (key & 127) of the elements in bin bA
#pragma unroll
  for (int e = 0; e < R; ++e) {
    const uint32_t key = key_of(e);
    if (e < nv && (key >> 7) == bA) atomicAdd(&histB[key & 127u], 1u);
  }
  __syncthreads();
  if (t < 32) {  // lane l owns fine bins [4l, 4l + 4)
    uint32_t c[4], sum = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      c[j] = histB[4 * lane + j];
      sum += c[j];
    }
    const uint32_t sr = __shfl_sync(0xffffffffu, sum, 31 - lane);
    uint32_t inc = sr;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    const uint32_t qq = (uint32_t)q - aboveA;
    const uint32_t above = __shfl_sync(0xffffffffu, inc, 31 - lane) - sum;
    if (above < qq && above + sum >= qq) {
      uint32_t run = above;
#pragma unroll
      for (int j = 3; j >= 0; --j) {
        if (run + c[j] >= qq) {
          s_T = (bA << 7) | (uint32_t)(4 * lane + j);
          s_need = qq - run;
          break;
        }
        run += c[j];
      }
    }
  }
  __syncthreads();
  const uint32_t T = s_T;
  const int need = (int)s_need;  // ties (key == T) to take, lowest index first
  SEL_PHASE(2);

  // ---- 3. per-thread counts, block exclusive scan of packed (eq << 16 | gt) in index order
  uint32_t n_gt = 0, n_eq = 0;
#pragma unroll
  for (int e = 0; e < R; ++e) {
    const uint32_t key = key_of(e);
    n_gt += e < nv && key > T;
    n_eq += e < nv && key == T;
  }
  const uint32_t v = (n_eq << 16) | n_gt;
  const uint32_t pre = block_exclusive_scan(v, tmp);
  SEL_PHASE(3);
  if (n_gt + n_eq) {
    int eq_seen = (int)(pre >> 16);
    int pos = (int)(pre & 0xffffu) + min(eq_seen, need);
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const uint32_t key = key_of(e);
      bool take = e < nv && key > T;
      if (e < nv && key == T) {
        take = eq_seen < need;
        ++eq_seen;
      }
      if (take) {
        const uint32_t h = (e & 1) ? (raw[e >> 1] >> 16) : (raw[e >> 1] & 0xffffu);
        idx_out[out_off + pos] = a + base + e;
        xs_out[out_off + pos] = (uint16_t)h;
        if (sel_out) sel_out[out_off + pos] = a + base + e;
        ++pos;
      }
    }
  }
  if (trace && t == 0 && blockIdx.x == 0) {
    trace[1] = globaltimer();
    trace[2 + 1024 * 9 - 1] = clock64();
  }
#undef SEL_PHASE
}

// launch geometry for a segment of len elements: NT threads of C 8-element chunks
inline void select_geometry(int len, int* nt, int* C) {
  int c = 1;
  while (c < 4 && (len + 8 * c - 1) / (8 * c) > kSelMaxThreads) c *= 2;
  *nt = ((len + 8 * c - 1) / (8 * c) + 31) / 32 * 32;
  *C = c;
}
inline size_t select_smem_bytes() { return 0; }

}  // namespace decdec
