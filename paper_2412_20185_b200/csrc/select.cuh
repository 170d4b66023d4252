// Step (1) of DecDEC: exact Top-k of |x| ("Exact").
//
// Replaces the paper's 32-bucket approximate, randomly-filled chunk Top-K with
// an exact, deterministic two-level radix select over the 15-bit magnitude key
// bits(x) & 0x7FFF (ledger L2): histogram of key>>7 (256 bins) locates the bin holding
// the k-th largest key, a second histogram of key&127 inside that bin gives the exact
// threshold T; then one block-wide exclusive scan (in index order) of (#key>T, #key==T)
// per thread places every selected index, taking the lowest-index ties first.  Output is
// ascending by index.  One CTA per segment: the whole vector (chunk = 0) or one
// chunk (chunk > 0, the paper's partition).
#pragma once
#include <cstdint>
#include "ptx.cuh"

namespace decdec {

template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint32_t t = lane < NT / 32 ? warp_tot[lane] : 0u;
    uint32_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += u;
    }
    if (lane < NT / 32) warp_tot[lane] = ti - t;  // exclusive prefix of warp totals
  }
  __syncthreads();
  return warp_tot[wid] + inc - v;
}

// Finds, scanning bins from the top, the bin b with  above(b) < need <= above(b) + h[b].
// Executed by warp 0; nb = 256 or 128 bins.  Writes (b, above(b)) to out[0..1].
template <int NB>
__device__ __forceinline__ void find_bin_desc(const int* h, int need, int* out) {
  constexpr int PER = NB / 32;
  const int lane = threadIdx.x & 31;
  int c[PER];
  int tot = 0;
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    c[e] = h[NB - 1 - (PER * lane + e)];
    tot += c[e];
  }
  int inc = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  int run = inc - tot;
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    if (run < need && run + c[e] >= need) {
      out[0] = NB - 1 - (PER * lane + e);
      out[1] = run;
    }
    run += c[e];
  }
}

// grid = number of segments; dynamic smem = segment length * 2 bytes.
template <int NT>
__global__ void __launch_bounds__(NT) k_select(const uint16_t* __restrict__ x, int d_in, int k, int chunk,
                                               int* __restrict__ idx_out, uint16_t* __restrict__ xs_out,
                                               int* __restrict__ sel_out) {
  // Programmatic dependent launch: the fused GEMV kernel that follows may start its
  // HBM stream now; only its gather warps wait (griddepcontrol.wait) for our results.
  pdl_launch_dependents();
  extern __shared__ uint16_t sx[];
  __shared__ int h1[256];
  __shared__ int h2[128];
  __shared__ uint32_t warp_tot[32];
  __shared__ int s_bin[2];

  const int seg = blockIdx.x;
  const int a = chunk ? seg * chunk : 0;
  const int n = chunk ? min(chunk, d_in - a) : d_in;
  const int q = chunk ? min(k, n) : k;
  const int out_off = chunk ? seg * k : 0;  // every earlier chunk is full length >= k
  if (q <= 0) return;

  for (int i = threadIdx.x; i < 256; i += NT) h1[i] = 0;
  for (int i = threadIdx.x; i < 128; i += NT) h2[i] = 0;
  for (int i = threadIdx.x; i < n; i += NT) sx[i] = x[a + i];
  __syncthreads();

  for (int i = threadIdx.x; i < n; i += NT) atomicAdd(&h1[(sx[i] & 0x7FFF) >> 7], 1);
  __syncthreads();
  if (threadIdx.x < 32) find_bin_desc<256>(h1, q, s_bin);
  __syncthreads();
  const int b1 = s_bin[0], above1 = s_bin[1];
  for (int i = threadIdx.x; i < n; i += NT) {
    const int key = sx[i] & 0x7FFF;
    if ((key >> 7) == b1) atomicAdd(&h2[key & 127], 1);
  }
  __syncthreads();
  if (threadIdx.x < 32) find_bin_desc<128>(h2, q - above1, s_bin);
  __syncthreads();
  const int T = (b1 << 7) | s_bin[0];
  const int need = q - above1 - s_bin[1];  // ties (key == T) to take, lowest index first

  // contiguous per-thread ranges, scanned in index order
  const int E = (n + NT - 1) / NT;
  const int lo = min(threadIdx.x * E, n), hi = min(lo + E, n);
  uint32_t n_gt = 0, n_eq = 0;
  for (int i = lo; i < hi; ++i) {
    const int key = sx[i] & 0x7FFF;
    n_gt += key > T;
    n_eq += key == T;
  }
  const uint32_t pre = block_exclusive_scan<NT>((n_eq << 16) | n_gt, warp_tot);
  const int eq_pre = pre >> 16, gt_pre = pre & 0xFFFF;
  int pos = gt_pre + min(eq_pre, need);
  int eq_seen = eq_pre;
  for (int i = lo; i < hi; ++i) {
    const uint16_t raw = sx[i];
    const int key = raw & 0x7FFF;
    bool take = key > T;
    if (key == T) {
      take = eq_seen < need;
      ++eq_seen;
    }
    if (take) {
      idx_out[out_off + pos] = a + i;
      xs_out[out_off + pos] = raw;
      if (sel_out) sel_out[out_off + pos] = a + i;
      ++pos;
    }
  }
}

}  // namespace decdec
