// Step (1) of DecDEC: exact Top-k of |x| ("Exact").
//
// Replaces the paper's 32-bucket approximate, randomly-filled chunk Top-K with
// an exact, deterministic radix select over the 15-bit magnitude key bits(x) & 0x7FFF
// (ledger L2).  One CTA per segment (the whole x for chunk = 0, one chunk otherwise).
// Every thread owns R = 8C contiguous elements held in registers.  Measured on B200 (probe
// profiles/r01_probe_*): a warp ballot / reduce / match costs ~8 SMSP cycles, an ALU op 0.5,
// so all per-element work is plain ALU:
//   1. level 1 (key bits 14..10): 32 byte counters per thread in 8 registers, reduced
//      through smem in two parallel steps -> bin b1 holding the q-th largest key;
//   2. candidates (key >> 10 == b1, usually a few % of x) appended to a smem list;
//   3. levels 2 and 3 (bits 9..5, 4..0) on the candidates only: per 32 candidates a warp
//      takes 5 ballots of the digit bits (+1 validity), lane b counts
//      popc(V & ~(B_j ^ bit_j(b))) -> threshold T and the number of ties `need`;
//   4. per-thread counts of key > T / key == T, one block exclusive scan in index order,
//      then each thread writes its selected indices (ties: lowest index first).
// Output ascending by index.
#pragma once
#include <cstdint>
#include "ptx.cuh"

namespace decdec {

constexpr int kSelMaxWarps = 32;
constexpr int kSelMaxThreads = 1024;

// per-bin totals `tot` held by lane b (bin b): (warp-uniformly) the bin holding the q-th
// largest key, scanning from the top; *above = keys in higher bins.
__device__ __forceinline__ int find_bin_top(uint32_t tot, int q, int* above) {
  const int lane = threadIdx.x & 31;
  const uint32_t c_rev = __shfl_sync(0xffffffffu, tot, 31 - lane);  // count of bin 31-lane
  uint32_t inc = c_rev;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  const uint32_t exc = inc - c_rev;
  const unsigned hit = __ballot_sync(0xffffffffu, exc < (uint32_t)q && inc >= (uint32_t)q);
  const int src = __ffs(hit) - 1;
  *above = (int)__shfl_sync(0xffffffffu, exc, src);
  return 31 - src;
}

// hist[w][b] (w < nw) -> every thread gets sum_w hist[w][lane] (warp 0 sums with all loads
// in flight, publishes through smem; barriers on entry and exit).
__device__ __forceinline__ uint32_t sum_warp_rows(uint32_t (*hist)[32], uint32_t* tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (wid == 0) {
    uint32_t v[kSelMaxWarps];
#pragma unroll
    for (int w = 0; w < kSelMaxWarps; ++w) v[w] = w < nw ? hist[w][lane] : 0u;
#pragma unroll
    for (int s = kSelMaxWarps / 2; s; s >>= 1)
#pragma unroll
      for (int w = 0; w < s; ++w) v[w] += v[w + s];
    tot[lane] = v[0];
  }
  __syncthreads();
  return tot[lane];
}

// level 2/3 on the candidate list: 32-bin histogram of (key >> shift) & 31 over candidates
// with key >> pshift == prefix; returns the bin of the q-th largest (see find_bin_top).
__device__ __forceinline__ int cand_level(const uint16_t* cand, int m, int shift, int pshift, int prefix, int q,
                                          uint32_t (*hist)[32], uint32_t* tot, int* above) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t inv[5];
#pragma unroll
  for (int j = 0; j < 5; ++j) inv[j] = ((lane >> j) & 1) ? 0u : 0xffffffffu;
  uint32_t cnt = 0;
#pragma unroll 1
  for (int i0 = wid * 32; i0 < m; i0 += nw * 32) {
    const int i = i0 + lane;
    const uint32_t key = i < m ? cand[i] : 0xffffu;
    uint32_t msk = __ballot_sync(0xffffffffu, i < m && (int)(key >> pshift) == prefix);
    const uint32_t d = (key >> shift) & 31u;
#pragma unroll
    for (int b = 0; b < 5; ++b) msk &= __ballot_sync(0xffffffffu, (d >> b) & 1u) ^ inv[b];
    cnt += __popc(msk);
  }
  hist[wid][lane] = cnt;
  return find_bin_top(sum_warp_rows(hist, tot), q, above);
}

// grid = number of segments; blockDim = NT (multiple of 32, <= 1024) with NT * 8C >= len;
// dynamic smem = select_smem_bytes(NT, C).
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
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ uint32_t hist[3][kSelMaxWarps][32];
  __shared__ uint32_t tots[3][32];
  __shared__ uint32_t scan_tot[kSelMaxWarps];
  __shared__ int n_cand;
  const int seg = blockIdx.x;
  const int a = chunk ? seg * chunk : 0;
  const int n = chunk ? min(chunk, d_in - a) : d_in;
  const int q = chunk ? min(k, n) : k;
  const int out_off = chunk ? seg * k : 0;  // every earlier chunk is full length >= k
  if (q <= 0) return;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
  const int NT = blockDim.x;
  uint32_t* part = reinterpret_cast<uint32_t*>(dsm);          // [NT][8] level-1 byte counters
  uint16_t* cand = reinterpret_cast<uint16_t*>(dsm + NT * 32);  // candidate keys [n]
#define SEL_PHASE(i) \
  if (trace && t == 0 && blockIdx.x == 0) trace[2 + 1024 * 9 - 16 + (i)] = clock64();

  // R contiguous elements per thread (16-B loads, all in flight before use)
  const int base = t * R;
  uint32_t raw[R / 2];
#pragma unroll
  for (int v = 0; v < C; ++v) {
    uint4 q4 = make_uint4(0, 0, 0, 0);
    if (base + 8 * v < n) q4 = __ldg(reinterpret_cast<const uint4*>(x + a + base) + v);
    raw[4 * v + 0] = q4.x; raw[4 * v + 1] = q4.y; raw[4 * v + 2] = q4.z; raw[4 * v + 3] = q4.w;
  }
  const int nv = n - base;  // slot e < nv is a real element
  auto key_of = [&](int e) -> uint32_t {
    return ((e & 1) ? (raw[e >> 1] >> 16) : raw[e >> 1]) & 0x7fffu;
  };
  if (t == 0) n_cand = 0;
  SEL_PHASE(0);

  // ---- level 1: 32 byte counters (bin = key >> 10) in 8 registers, bin b in byte b & 3 of word b >> 2
  {
    uint32_t c8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int e = 0; e < R; ++e) {
      if (e < nv) {
        const uint32_t bin = key_of(e) >> 10;
        const uint32_t inc = 1u << ((bin & 3u) << 3);
        const uint32_t w = bin >> 2;
#pragma unroll
        for (int j = 0; j < 8; ++j) c8[j] += (w == (uint32_t)j) ? inc : 0u;
      }
    }
    uint4* prow = reinterpret_cast<uint4*>(part + t * 8);
    prow[0] = make_uint4(c8[0], c8[1], c8[2], c8[3]);
    prow[1] = make_uint4(c8[4], c8[5], c8[6], c8[7]);
  }
  __syncthreads();
  {  // thread (slice s = wid, bin pair p = lane & 15, half = lane >> 4): bins 2p, 2p+1 over
     // the 32 threads of warp s, as 16-bit pair sums (no byte overflow: <= 32 * R)
    const int p = lane & 15;
    const uint32_t* col = part + (wid * 32 + (lane >> 4) * 16) * 8 + (p >> 1);
    uint32_t acc = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t wv = col[r * 8];
      acc += (p & 1) ? ((wv >> 16) & 0xffu) | ((wv >> 8) & 0xff0000u) : (wv & 0xffu) | ((wv << 8) & 0xff0000u);
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 16);  // both 16-thread halves of the warp
    // acc = (count of bin 2p+? ) ... low 16 bits: bin 4(p>>1) + 2(p&1), high: that + 1
    if (lane < 16) {
      const int b0 = 4 * (p >> 1) + 2 * (p & 1);
      hist[0][wid][b0] = acc & 0xffffu;
      hist[0][wid][b0 + 1] = acc >> 16;
    }
  }
  const uint32_t tot1 = sum_warp_rows(hist[0], tots[0]);
  SEL_PHASE(1);
  int above1, above2, above3;
  const int b1 = find_bin_top(tot1, q, &above1);
  SEL_PHASE(2);

  // ---- candidates of bin b1 -> smem list (order irrelevant: only counted)
  {
    int mine = 0;
#pragma unroll
    for (int e = 0; e < R; ++e) mine += (e < nv && (key_of(e) >> 10) == (uint32_t)b1);
    if (mine) {
      int pos = atomicAdd(&n_cand, mine);
#pragma unroll
      for (int e = 0; e < R; ++e)
        if (e < nv && (key_of(e) >> 10) == (uint32_t)b1) cand[pos++] = (uint16_t)key_of(e);
    }
  }
  __syncthreads();
  const int m = n_cand;
  SEL_PHASE(3);
  const int b2 = cand_level(cand, m, 5, 10, b1, q - above1, hist[1], tots[1], &above2);
  const int b3 = cand_level(cand, m, 0, 5, (b1 << 5) | b2, q - above1 - above2, hist[2], tots[2], &above3);
  const uint32_t T = (uint32_t)((b1 << 10) | (b2 << 5) | b3);
  const int need = q - above1 - above2 - above3;  // ties (key == T) to take, lowest index first
  SEL_PHASE(4);

  // ---- per-thread counts, block exclusive scan of packed (eq << 16 | gt) in index order
  uint32_t n_gt = 0, n_eq = 0;
#pragma unroll
  for (int e = 0; e < R; ++e) {
    const uint32_t key = key_of(e);
    n_gt += e < nv && key > T;
    n_eq += e < nv && key == T;
  }
  const uint32_t v = (n_eq << 16) | n_gt;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t s2 = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += s2;
  }
  if (lane == 31) scan_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {  // exclusive scan of the warp totals by one warp
    const uint32_t wt = lane < nw ? scan_tot[lane] : 0u;
    uint32_t wi = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t s2 = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += s2;
    }
    scan_tot[lane] = wi - wt;
  }
  __syncthreads();
  const uint32_t pre = scan_tot[wid] + inc - v;
  SEL_PHASE(5);
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
  const int t = ((len + 8 * c - 1) / (8 * c) + 31) / 32 * 32;
  *nt = t;
  *C = c;
}
inline size_t select_smem_bytes(int nt, int len) { return (size_t)nt * 32 + (size_t)len * 2 + 16; }

}  // namespace decdec
