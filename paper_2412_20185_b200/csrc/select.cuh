// Step (1) of DecDEC: exact Top-k of |x| ("Exact").
//
// Replaces the paper's 32-bucket approximate, randomly-filled chunk Top-K with
// an exact, deterministic selection on the 15-bit magnitude key bits(x) & 0x7FFF (ledger L2),
// done by ONE thread block (any size, multiple of 32) over one segment -- the whole x
// (chunk = 0) or one chunk.  In the fused layer kernel it is CTA 0's job; the
// standalone decdec_select runs it in its own kernel.
//   1. x is staged in smem; thread t owns chunks of 8 contiguous elements [tC, tC + C);
//   2. one smem atomicAdd per element into a 256-bin histogram of key >> 7 (measured ~4
//      SMSP cycles per warp-op on B200, activation exponents spread the bins); warp 0 finds
//      the bin holding the q-th largest key (lane l owns 8 contiguous bins, suffix scan over
//      lanes); a 128-bin histogram of key & 127 over that bin's elements then gives the exact
//      threshold T, `above` = #keys > T, need = q - above ties to take;
//   3. per-thread counts of key > T / key == T, one block exclusive scan in index order, and
//      each thread writes its selected indices (ties: lowest index first), ascending.
// Warp ballots / reductions cost ~8 SMSP cycles each on B200, so the per-element work avoids
// them; histogram rows are padded (stride 9 / 5 words) so warp 0's bin reads are conflict-free.
#pragma once
#include <cstdint>
#include "ptx.cuh"

namespace decdec {

constexpr int kSelMaxWarps = 32;
constexpr int kHistACopies = 4;            // coarse histogram copies (lane & 3); 8 copies measured slower
constexpr int kHistAStride = 256 + 32 + 8;  // = 8 mod 32: the copies start 8 banks apart

// shared scratch of select_block (plus the staged x: 2 * roundup(len, 8) bytes after it)
struct SelectSmem {
  uint32_t histA[256 + 32];  // bin b at b + (b >> 3)
  uint32_t histB[128 + 32];  // bin b at b + (b >> 2)
  uint32_t tmp[kSelMaxWarps];
  uint32_t bA, aboveA, T, need;
};
inline size_t select_block_smem_bytes(int len) { return sizeof(SelectSmem) + (size_t)((len + 7) / 8) * 16; }

// Exclusive scan of v over the block in thread order.  Two barriers.
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

// warp-level: lane l holds counts c[0..PER) of bins [PER*l, PER*l + PER); find the bin that
// contains the q-th largest key (scanning from the top).  Exactly one lane writes (*bin, *above).
template <int PER>
__device__ __forceinline__ void warp_find_bin(const uint32_t* c, uint32_t q, uint32_t* bin, uint32_t* above_out) {
  const int lane = threadIdx.x & 31;
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) sum += c[j];
  const uint32_t sr = __shfl_sync(0xffffffffu, sum, 31 - lane);
  uint32_t inc = sr;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  const uint32_t above = __shfl_sync(0xffffffffu, inc, 31 - lane) - sum;  // keys in lanes > l
  if (above < q && above + sum >= q) {
    uint32_t run = above;
#pragma unroll
    for (int j = PER - 1; j >= 0; --j) {
      if (run + c[j] >= q) {
        *bin = (uint32_t)(PER * lane + j);
        *above_out = run;
        break;
      }
      run += c[j];
    }
  }
}

// 16-bit element j (0..7) of a 16-B chunk
__device__ __forceinline__ uint32_t chunk_elem(const uint4& v, int j) {
  const uint32_t w = (j < 2) ? v.x : (j < 4) ? v.y : (j < 6) ? v.z : v.w;
  return (j & 1) ? (w >> 16) : (w & 0xffffu);
}

// Exact top-q of the n keys of x (global, 16-B aligned, n % 8 == 0) by the whole block.
// Writes idx_out[pos] = idx_base + i and xs_out[pos] = x[i] for the selected i in ascending
// order (pos = 0 .. q-1), and sel_out likewise if non-null.  Ends with a barrier-free tail:
// callers that consume the outputs in the same block must __syncthreads() (and fence for other
// blocks).
__device__ __forceinline__ void select_block(const uint16_t* __restrict__ x, int n, int q, int idx_base,
                                             int* __restrict__ idx_out, uint16_t* __restrict__ xs_out,
                                             int* __restrict__ sel_out, SelectSmem* S, uint4* sx4,
                                             unsigned long long* tr = nullptr) {
  // optional phase timestamps (thread 0): [16] x staged, [17] coarse bin, [18] threshold, [19] scan
#define SEL_TRACE(i)                                  \
  do {                                                \
    if (tr && threadIdx.x == 0) tr[i] = globaltimer(); \
  } while (0)
  const int t = threadIdx.x, NT = blockDim.x, lane = t & 31;
  const int n8 = n >> 3;
  const int C = (n8 + NT - 1) / NT;  // chunks of 8 per thread
  // stage x (coalesced 16-B loads) and zero the histograms
#pragma unroll 4
  for (int i = t; i < n8; i += NT) sx4[i] = __ldg(reinterpret_cast<const uint4*>(x) + i);
  for (int i = t; i < 256 + 32; i += NT) S->histA[i] = 0;
  for (int i = t; i < 128 + 32; i += NT) S->histB[i] = 0;
  __syncthreads();
  SEL_TRACE(16);
  const int c0 = t * C, c1 = min(c0 + C, n8);
  // ---- coarse histogram (key >> 7)
#pragma unroll 1
  for (int c = c0; c < c1; ++c) {
    const uint4 v = sx4[c];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t b = (chunk_elem(v, j) & 0x7fffu) >> 7;
      atomicAdd(&S->histA[b + (b >> 3)], 1u);
    }
  }
  __syncthreads();
  if (t < 32) {
    uint32_t c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = S->histA[9 * lane + j];
    warp_find_bin<8>(c, (uint32_t)q, &S->bA, &S->aboveA);
  }
  __syncthreads();
  SEL_TRACE(17);
  const uint32_t bA = S->bA, qB = (uint32_t)q - S->aboveA;
  // ---- fine histogram (key & 127) of bin bA
#pragma unroll 1
  for (int c = c0; c < c1; ++c) {
    const uint4 v = sx4[c];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t key = chunk_elem(v, j) & 0x7fffu;
      if ((key >> 7) == bA) {
        const uint32_t b = key & 127u;
        atomicAdd(&S->histB[b + (b >> 2)], 1u);
      }
    }
  }
  __syncthreads();
  if (t < 32) {
    uint32_t c[4], bin = 0, above = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = S->histB[5 * lane + j];
    bin = 0xffffffffu;
    warp_find_bin<4>(c, qB, &bin, &above);
    if (bin != 0xffffffffu) {
      S->T = (bA << 7) | bin;
      S->need = qB - above;
    }
  }
  __syncthreads();
  SEL_TRACE(18);
  const uint32_t T = S->T;
  const int need = (int)S->need;  // ties (key == T) to take, lowest index first
  // ---- counts, block scan in index order, placement
  uint32_t n_gt = 0, n_eq = 0;
#pragma unroll 1
  for (int c = c0; c < c1; ++c) {
    const uint4 v = sx4[c];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t key = chunk_elem(v, j) & 0x7fffu;
      n_gt += key > T;
      n_eq += key == T;
    }
  }
  const uint32_t pre = block_exclusive_scan((n_eq << 16) | n_gt, S->tmp);
  SEL_TRACE(19);
  if (n_gt + n_eq) {
    int eq_seen = (int)(pre >> 16);
    int pos = (int)(pre & 0xffffu) + min(eq_seen, need);
#pragma unroll 1
    for (int c = c0; c < c1; ++c) {
      const uint4 v = sx4[c];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t raw = chunk_elem(v, j);
        const uint32_t key = raw & 0x7fffu;
        bool take = key > T;
        if (key == T) {
          take = eq_seen < need;
          ++eq_seen;
        }
        if (take) {
          const int i = idx_base + 8 * c + j;
          idx_out[pos] = i;
          xs_out[pos] = (uint16_t)raw;
          if (sel_out) sel_out[pos] = i;
          ++pos;
        }
      }
    }
  }
  (void)lane;
#undef SEL_TRACE
}


// ---------------------------------------------------------------- register-resident variant
// Same result as select_block, for a block whose threads can hold the whole segment in
// registers (ceil(n / 8 / blockDim) <= MAXC chunks of 8 keys each).  Latency-oriented: three
// block barriers in total, no single-warp serial sections (every warp derives the bin /
// threshold / its output offset redundantly from shared counters), no smem staging pass, the
// coarse histogram split in 4 copies (lane & 3) against same-bin lane conflicts.  The caller
// zeroes S once before the first call (select_regs_zero + __syncthreads, e.g. before
// griddepcontrol.wait); each call leaves S zeroed again after its last barrier... except for
// the final zeroing, which the caller's barrier after the call orders before the next call.
struct SelectSmemR {
  // copy c, bin b at b + (b >> 3).  Activation magnitudes crowd a few bins, so lanes sharing a
  // copy often hit the same address (serialised atomics): 4 copies, on distinct bank offsets
  // (8 copies: the bin scan's extra reads cost more than the conflicts they save)
  uint32_t histA[kHistACopies][kHistAStride];
  uint32_t histB[128 + 32];     // bin b at b + (b >> 2)
  uint32_t wsum[kSelMaxWarps];  // per-warp (n_eq << 16 | n_gt) totals
};
__device__ __forceinline__ void select_regs_zero(SelectSmemR* S) {
  uint32_t* h = &S->histA[0][0];
  for (int i = threadIdx.x; i < kHistACopies * kHistAStride + 128 + 32; i += blockDim.x) h[i] = 0u;
}

// warp-redundant version of warp_find_bin: every lane gets (bin, above) for the q-th largest
template <int PER>
__device__ __forceinline__ void warp_find_bin_all(const uint32_t* c, uint32_t q, uint32_t* bin, uint32_t* above_out) {
  const int lane = threadIdx.x & 31;
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) sum += c[j];
  const uint32_t sr = __shfl_sync(0xffffffffu, sum, 31 - lane);
  uint32_t inc = sr;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  const uint32_t above = __shfl_sync(0xffffffffu, inc, 31 - lane) - sum;  // keys in lanes > l
  uint32_t b = 0, ab = 0;
  const bool mine = above < q && above + sum >= q;
  if (mine) {
    uint32_t run = above;
#pragma unroll
    for (int j = PER - 1; j >= 0; --j) {
      if (run + c[j] >= q) {
        b = (uint32_t)(PER * lane + j);
        ab = run;
        break;
      }
      run += c[j];
    }
  }
  const uint32_t who = __ballot_sync(0xffffffffu, mine);
  const int src = who ? __ffs(who) - 1 : 0;
  *bin = __shfl_sync(0xffffffffu, b, src);
  *above_out = __shfl_sync(0xffffffffu, ab, src);
}

template <int MAXC>
__device__ __forceinline__ void select_block_regs(const uint16_t* __restrict__ x, int n, int q, int idx_base,
                                                  int* __restrict__ idx_out, uint16_t* __restrict__ xs_out,
                                                  int* __restrict__ sel_out, SelectSmemR* S,
                                                  unsigned long long* tr = nullptr) {
#define SEL_TRACE(i)                                  \
  do {                                                \
    if (tr && threadIdx.x == 0) tr[i] = clock64();     \
  } while (0)
  const int t = threadIdx.x, NT = blockDim.x, lane = t & 31, wid = t >> 5, nw = NT >> 5;
  const int n8 = n >> 3;
  const int C = (n8 + NT - 1) / NT;  // <= MAXC (caller's guarantee)
  const int c0 = t * C;
  const int nv = max(0, min(C, n8 - c0));  // valid chunks of this thread
  uint4 v[MAXC];
  const uint4* x4 = reinterpret_cast<const uint4*>(x) + c0;
#pragma unroll
  for (int m = 0; m < MAXC; ++m) v[m] = m < nv ? __ldg(x4 + m) : make_uint4(0, 0, 0, 0);
  SEL_TRACE(16);
  // ---- coarse histogram (key >> 7), 4 copies
  uint32_t* hA = S->histA[lane & (kHistACopies - 1)];
#pragma unroll
  for (int m = 0; m < MAXC; ++m) {
    if (m < nv) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t b = (chunk_elem(v[m], j) & 0x7fffu) >> 7;
        atomicAdd(&hA[b + (b >> 3)], 1u);
      }
    }
  }
  __syncthreads();  // barrier 1
  uint32_t bA, aboveA;
  {
    uint32_t c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      c[j] = S->histA[0][9 * lane + j] + S->histA[1][9 * lane + j] + S->histA[2][9 * lane + j] + S->histA[3][9 * lane + j];
    warp_find_bin_all<8>(c, (uint32_t)q, &bA, &aboveA);
  }
  SEL_TRACE(17);
  const uint32_t qB = (uint32_t)q - aboveA;
  // ---- fine histogram (key & 127) of bin bA
#pragma unroll
  for (int m = 0; m < MAXC; ++m) {
    if (m < nv) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t key = chunk_elem(v[m], j) & 0x7fffu;
        if ((key >> 7) == bA) {
          const uint32_t b = key & 127u;
          atomicAdd(&S->histB[b + (b >> 2)], 1u);
        }
      }
    }
  }
  __syncthreads();  // barrier 2
  uint32_t T, need_u;
  {
    uint32_t c[4], bin, above;
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = S->histB[5 * lane + j];
    warp_find_bin_all<4>(c, qB, &bin, &above);
    T = (bA << 7) | bin;
    need_u = qB - above;
  }
  SEL_TRACE(18);
  const int need = (int)need_u;  // ties (key == T) to take, lowest index first
  // ---- counts, block scan in index order (one barrier), placement
  uint32_t n_gt = 0, n_eq = 0;
#pragma unroll
  for (int m = 0; m < MAXC; ++m) {
    if (m < nv) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t key = chunk_elem(v[m], j) & 0x7fffu;
        n_gt += key > T;
        n_eq += key == T;
      }
    }
  }
  const uint32_t mine = (n_eq << 16) | n_gt;
  uint32_t inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) S->wsum[wid] = inc;
  __syncthreads();  // barrier 3: histograms are no longer read, warp totals are visible
  uint32_t wpre;
  {
    const uint32_t wt = lane < nw ? S->wsum[lane] : 0u;
    uint32_t wi = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += u;
    }
    wpre = __shfl_sync(0xffffffffu, wi - wt, wid);  // exclusive prefix of this warp
  }
  SEL_TRACE(19);
  {  // zero the histograms for the next call (the caller's barrier orders it before that call)
    uint32_t* h = &S->histA[0][0];
    for (int i = t; i < kHistACopies * kHistAStride + 128 + 32; i += NT) h[i] = 0u;
  }
  const uint32_t pre = wpre + inc - mine;
  if (n_gt + n_eq) {
    int eq_seen = (int)(pre >> 16);
    int pos = (int)(pre & 0xffffu) + min(eq_seen, need);
#pragma unroll
    for (int m = 0; m < MAXC; ++m) {
      if (m < nv) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t raw = chunk_elem(v[m], j);
          const uint32_t key = raw & 0x7fffu;
          bool take = key > T;
          if (key == T) {
            take = eq_seen < need;
            ++eq_seen;
          }
          if (take) {
            const int i = idx_base + 8 * (c0 + m) + j;
            idx_out[pos] = i;
            xs_out[pos] = (uint16_t)raw;
            if (sel_out) sel_out[pos] = i;
            ++pos;
          }
        }
      }
    }
  }
#undef SEL_TRACE
}


// ---------------------------------------------------------------- DEC CTA variant (split order)
// Same selected set as select_block, placed in a different (still deterministic) order that
// lets the caller start gathering before the selection finishes:
//   positions [0, D)  : keys whose coarse bin (key >> 7) is above the threshold bin, ascending
//                       index -- known after the first histogram (three block barriers);
//   positions [D, q)  : the rest R (threshold bin: key > T, then the lowest-index ties),
//                       ascending -- written by ONE finisher warp from a bitmap of the
//                       threshold-bin candidates, published through a shared flag (no block
//                       barrier, so the other warps' gathers of [0, D) are already in flight).
// Returns D.  The caller's warps may use positions < D immediately; positions >= D after
// select_wait_rest().  If sel_out is non-null the finisher also writes the whole selection
// in ascending index order (merge of the two sorted runs; the decdec_linear `sel` contract).
constexpr int kCandList = 256;  // threshold-bin candidates kept as a sortable list (else bitmap scan)
struct SelectSmemS {
  SelectSmemR r;
  uint32_t bitmap[1024];  // threshold-bin candidates, bit i = key i (n <= 32768)
  uint32_t cand[kCandList];  // (index << 15 | key) of threshold-bin candidates: warp w's, in index
                             // order, at [w * cap, w * cap + wcand[w]), cap = kCandList / warps
  uint32_t wcand[kSelMaxWarps];  // candidates per warp (written by each warp's lane 31)
  uint32_t scratch[128];         // never read: destination of the DEC CTA's early D-row reads
  uint32_t rest_ready;
  uint32_t ncand;
  uint32_t pad[2];
  // followed by the staged keys: uint16_t [n] (select_split_smem_bytes)
};
__host__ __device__ inline size_t select_split_smem_bytes(int n) { return sizeof(SelectSmemS) + (size_t)((n + 7) / 8) * 16; }
__device__ __forceinline__ void select_split_zero(SelectSmemS* S, int n) {
  select_regs_zero(&S->r);
  for (int i = threadIdx.x; i < (n + 31) / 32; i += blockDim.x) S->bitmap[i] = 0u;
  if (threadIdx.x == 0) {
    S->rest_ready = 0u;
    S->ncand = 0u;
  }
}
__device__ __forceinline__ void select_wait_rest(const SelectSmemS* S) {
  while (*reinterpret_cast<const volatile uint32_t*>(&S->rest_ready) == 0u) __nanosleep(100);  // keep the LSU free
  __threadfence_block();
}

struct NoEarly {
  __device__ __forceinline__ bool on() const { return false; }
  __device__ __forceinline__ int cap() const { return 0; }
  __device__ __forceinline__ bool spare_finisher() const { return false; }
  __device__ __forceinline__ void operator()(int) const {}
};
template <int MAXC, typename Early = NoEarly>
__device__ __forceinline__ int select_split(const uint16_t* __restrict__ x, int n, int q, int* __restrict__ idx_out,
                                            uint16_t* __restrict__ xs_out, int* __restrict__ sel_out, SelectSmemS* SS,
                                            int finisher, unsigned long long* tr, Early early = Early()) {
#define SEL_TRACE(i)                                  \
  do {                                                \
    if (tr && threadIdx.x == 0) tr[i] = clock64();     \
  } while (0)
  SelectSmemR* S = &SS->r;
  const int t = threadIdx.x, NT = blockDim.x, lane = t & 31, wid = t >> 5, nw = NT >> 5;
  const int n8 = n >> 3;
  const int C = (n8 + NT - 1) / NT;  // <= MAXC (caller's guarantee)
  const int c0 = t * C;
  const int nv = max(0, min(C, n8 - c0));
  uint4 v[MAXC];
  const uint4* x4 = reinterpret_cast<const uint4*>(x) + c0;
#pragma unroll
  for (int m = 0; m < MAXC; ++m) v[m] = m < nv ? __ldg(x4 + m) : make_uint4(0, 0, 0, 0);
  SEL_TRACE(16);
  uint4* sx = reinterpret_cast<uint4*>(SS + 1);  // staged keys for the finisher warp
  // ---- coarse histogram (key >> 7), 4 copies.  (Measured: a pre-filter that counts only keys
  // at or above the bin of the q-th largest per-thread maximum cut the atomics ~10x but its
  // extra barrier + bin search made the coarse phase ~1100 cycles SLOWER at 4096 and 14336 keys:
  // the atomics are not what bounds this phase.)
  uint32_t* hA = S->histA[lane & (kHistACopies - 1)];
#pragma unroll
  for (int m = 0; m < MAXC; ++m) {
    if (m < nv) {
      sx[c0 + m] = v[m];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t b = (chunk_elem(v[m], j) & 0x7fffu) >> 7;
        atomicAdd(&hA[b + (b >> 3)], 1u);
      }
    }
  }
  __syncthreads();  // barrier 1
  uint32_t bA, nD;
  {
    uint32_t c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      c[j] = S->histA[0][9 * lane + j] + S->histA[1][9 * lane + j] + S->histA[2][9 * lane + j] + S->histA[3][9 * lane + j];
    warp_find_bin_all<8>(c, (uint32_t)q, &bA, &nD);
  }
  SEL_TRACE(17);
  // ---- D counts; fine histogram + candidate bitmap/list of bin bA.  Per chunk the per-key
  // work is branch-free (masks); the rare keys in bin bA take one branch per chunk.  List slots
  // are allocated once per warp (scan of the lanes' candidate counts, one atomic by lane 31):
  // per-chunk atomics on the shared counter serialised into ~1 us on d-sized inputs.
  uint32_t n_d = 0, n_c = 0, dmask[MAXC], cmask[MAXC];
#pragma unroll
  for (int m = 0; m < MAXC; ++m) {
    dmask[m] = 0;
    cmask[m] = 0;
    if (m < nv) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t b = (chunk_elem(v[m], j) & 0x7fffu) >> 7;
        dmask[m] |= (uint32_t)(b > bA) << j;
        cmask[m] |= (uint32_t)(b == bA) << j;
      }
      n_d += __popc(dmask[m]);
      n_c += __popc(cmask[m]);
    }
  }
  // one lane scan for both counts (a warp holds <= 2048 keys: 16-bit fields)
  uint32_t inc_cd = (n_c << 16) | n_d;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc_cd, o);
    if (lane >= o) inc_cd += u;
  }
  const uint32_t inc_d = inc_cd & 0xffffu;
  {
    const uint32_t inc_c = inc_cd >> 16;
    // warp-private list region: slots are in index order without any cross-warp allocation
    const uint32_t cap = (uint32_t)kCandList / (uint32_t)nw;
    if (lane == 31) SS->wcand[wid] = inc_c;
    uint32_t o = inc_c - n_c;  // this thread's first slot in its warp's region
    if (n_c) {
#pragma unroll
      for (int m = 0; m < MAXC; ++m) {
        const uint32_t bits = cmask[m];
        if (bits) {
          atomicOr(&SS->bitmap[(c0 + m) >> 2], bits << (8 * ((c0 + m) & 3)));
          for (uint32_t bb = bits; bb; bb &= bb - 1, ++o) {
            const int jj = __ffs(bb) - 1;
            const uint32_t key = chunk_elem(v[m], jj) & 0x7fffu;
            const uint32_t fb = key & 127u;
            atomicAdd(&S->histB[fb + (fb >> 2)], 1u);
            if (o < cap) SS->cand[wid * cap + o] = ((uint32_t)(8 * (c0 + m) + jj) << 15) | key;
          }
        }
      }
    }
  }
#ifndef DECDEC_NO_EARLY
  // every D key of the warp handed to `early` warp-collectively before barrier 2 (the caller
  // starts fetching those rows while the rest of the selection runs)
  // At most early.cap() rows per warp (0 = all): a warp's zero-copy requests in flight are few,
  // and a warp that waits to issue more stalls the selection at barrier 2.
  if (early.on() && (wid != finisher || !early.spare_finisher())) {
    const int cap = early.cap();
    int issued = 0;
    for (int m = 0; m < MAXC; ++m) {
      uint32_t any = __ballot_sync(0xffffffffu, dmask[m] != 0u);
      while (any && (cap == 0 || issued < cap)) {
        const int src = __ffs(any) - 1;
        any &= any - 1;
        uint32_t bits = __shfl_sync(0xffffffffu, dmask[m], src);
        const int base = 8 * (__shfl_sync(0xffffffffu, c0, src) + m);
        while (bits && (cap == 0 || issued < cap)) {
          const int jj = __ffs(bits) - 1;
          bits &= bits - 1;
          early(base + jj);
          ++issued;
        }
      }
    }
  }
#endif
  if (lane == 31) S->wsum[wid] = inc_d;
  __syncthreads();  // barrier 2: histB, bitmap, D warp totals complete
  uint32_t pre_d;
  {
    const uint32_t wt = lane < nw ? S->wsum[lane] : 0u;
    uint32_t wi = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += u;
    }
    const uint32_t wpre = __shfl_sync(0xffffffffu, wi - wt, wid);
    pre_d = wpre + inc_d - n_d;
  }
  if (n_d) {  // place D at [0, nD), ascending (only the few threads holding D keys)
    int pos = (int)pre_d;
#pragma unroll
    for (int m = 0; m < MAXC; ++m) {
      for (uint32_t bb = dmask[m]; bb; bb &= bb - 1) {
        const int jj = __ffs(bb) - 1;
        idx_out[pos] = 8 * (c0 + m) + jj;
        xs_out[pos] = (uint16_t)chunk_elem(v[m], jj);
        ++pos;
      }
    }
  }
  __syncthreads();  // barrier 3: D placed
  SEL_TRACE(18);
  if (wid == finisher) {
    // ---- threshold T inside bin bA, then R from the bitmap in index order
    uint32_t T, need;
    {
      uint32_t c[4], bin, above;
#pragma unroll
      for (int j = 0; j < 4; ++j) c[j] = S->histB[5 * lane + j];
      warp_find_bin_all<4>(c, (uint32_t)q - nD, &bin, &above);
      T = (bA << 7) | bin;
      need = (uint32_t)q - nD - above;
    }
    if (tr && lane == 0) tr[11] = clock64();
    // x values of the taken candidates come from the keys staged in smem (not a global
    // round trip on the critical path)
    const uint16_t* xk_staged = reinterpret_cast<const uint16_t*>(sx);
    const uint32_t cap = (uint32_t)kCandList / (uint32_t)nw;
    const uint32_t wc = lane < nw ? SS->wcand[lane] : 0u;
    if (!__any_sync(0xffffffffu, wc > cap)) {
      // warp-ordered lists: lane l walks warp l's candidates (index order), so the lanes'
      // prefix over (#key > T, #key == T) gives every taken candidate its position directly
      const uint32_t* L = SS->cand + lane * cap;
      uint32_t n_gt = 0, n_eq = 0;
      for (uint32_t i = 0; i < wc; ++i) {
        const uint32_t key = L[i] & 0x7fffu;
        n_gt += key > T;
        n_eq += key == T;
      }
      uint32_t inc = (n_eq << 16) | n_gt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      const uint32_t pre = inc - ((n_eq << 16) | n_gt);
      uint32_t eq_seen = pre >> 16, g_seen = pre & 0xffffu;
      for (uint32_t i = 0; i < wc; ++i) {
        const uint32_t v = L[i], key = v & 0x7fffu, ix = v >> 15;
        if (key > T) {
          const uint32_t pos = nD + g_seen + min(eq_seen, need);
          idx_out[pos] = (int)ix;
          xs_out[pos] = xk_staged[ix];
          ++g_seen;
        } else if (key == T) {
          if (eq_seen < need) {
            const uint32_t pos = nD + g_seen + eq_seen;
            idx_out[pos] = (int)ix;
            xs_out[pos] = xk_staged[ix];
          }
          ++eq_seen;
        }
      }
    } else {
    const int nwords = (n + 31) >> 5;
    const int W = (nwords + 31) >> 5;  // lane l owns bitmap words [l*W, l*W + W): index order
    const int w_lo = min(lane * W, nwords), w_hi = min(w_lo + W, nwords);
    const uint16_t* xk = reinterpret_cast<const uint16_t*>(sx);
    uint32_t n_gt = 0, n_eq = 0;  // pass 1: counts of key > T / key == T among my candidates
    for (int w = w_lo; w < w_hi; ++w) {
      for (uint32_t bb = SS->bitmap[w]; bb; bb &= bb - 1) {
        const uint32_t key = xk[32 * w + __ffs(bb) - 1] & 0x7fffu;
        n_gt += key > T;
        n_eq += key == T;
      }
    }
#ifdef DECDEC_FINISHER_TRACE
    if (tr && lane == 0) tr[1] = clock64();
#endif
    uint32_t inc = (n_eq << 16) | n_gt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    const uint32_t pre = inc - ((n_eq << 16) | n_gt);
#ifdef DECDEC_FINISHER_TRACE
    if (tr && lane == 0) tr[2] = clock64();
#endif
    uint32_t eq_seen = pre >> 16, g_seen = pre & 0xffffu;
    if (n_gt + n_eq) {  // pass 2: write my taken candidates at nD + (#taken before them)
      for (int w = w_lo; w < w_hi; ++w) {
        for (uint32_t bb = SS->bitmap[w]; bb; bb &= bb - 1) {
          const int i = 32 * w + __ffs(bb) - 1;
          const uint16_t raw = xk[i];
          const uint32_t key = raw & 0x7fffu;
          if (key > T) {
            const uint32_t pos = nD + g_seen + min(eq_seen, need);
            idx_out[pos] = i;
            xs_out[pos] = raw;
            ++g_seen;
          } else if (key == T) {
            if (eq_seen < need) {
              const uint32_t pos = nD + g_seen + eq_seen;
              idx_out[pos] = i;
              xs_out[pos] = raw;
            }
            ++eq_seen;
          }
        }
      }
    }
    }  // bitmap path
    __syncwarp();
    if (tr && lane == 0) tr[13] = clock64();
    if (sel_out) {  // merge the two ascending runs [0, nD) and [nD, q) into sel_out
      const int nR = q - (int)nD;
      for (int a = lane; a < (int)nD; a += 32) {  // D element: + #R below it
        const int v0 = idx_out[a];
        int lo = 0, hi = nR;
        while (lo < hi) { const int mid = (lo + hi) >> 1; if (idx_out[nD + mid] < v0) lo = mid + 1; else hi = mid; }
        sel_out[a + lo] = v0;
      }
      for (int r = lane; r < nR; r += 32) {  // R element: + #D below it
        const int v0 = idx_out[nD + r];
        int lo = 0, hi = (int)nD;
        while (lo < hi) { const int mid = (lo + hi) >> 1; if (idx_out[mid] < v0) lo = mid + 1; else hi = mid; }
        sel_out[r + lo] = v0;
      }
    }
    __threadfence_block();
    __syncwarp();
    if (lane == 0) {
      *reinterpret_cast<volatile uint32_t*>(&SS->rest_ready) = 1u;
      if (tr) tr[19] = clock64();
    }
  }
  return (int)nD;
#undef SEL_TRACE
}

// Dispatch on the chunks per thread (fewer unrolled slots -> less predication overhead).
__device__ __forceinline__ bool select_block_regs_any(const uint16_t* x, int n, int q, int idx_base, int* idx_out,
                                                      uint16_t* xs_out, int* sel_out, SelectSmemR* S,
                                                      unsigned long long* tr) {
  const int C = ((n >> 3) + (int)blockDim.x - 1) / (int)blockDim.x;
  if (C <= 1) select_block_regs<1>(x, n, q, idx_base, idx_out, xs_out, sel_out, S, tr);
  else if (C <= 2) select_block_regs<2>(x, n, q, idx_base, idx_out, xs_out, sel_out, S, tr);
  else if (C <= 4) select_block_regs<4>(x, n, q, idx_base, idx_out, xs_out, sel_out, S, tr);
  else if (C <= 8) select_block_regs<8>(x, n, q, idx_base, idx_out, xs_out, sel_out, S, tr);
  else return false;
  return true;
}

// Returns D (>= 0), or -1 if the segment does not fit in registers (caller falls back).
template <typename Early = NoEarly>
__device__ __forceinline__ int select_split_any(const uint16_t* x, int n, int q, int* idx_out, uint16_t* xs_out,
                                                int* sel_out, SelectSmemS* S, int finisher, unsigned long long* tr,
                                                Early early = Early()) {
  const int C = ((n >> 3) + (int)blockDim.x - 1) / (int)blockDim.x;
  if (n > 32 * 1024) return -1;
  if (C <= 1) return select_split<1>(x, n, q, idx_out, xs_out, sel_out, S, finisher, tr, early);
  if (C <= 2) return select_split<2>(x, n, q, idx_out, xs_out, sel_out, S, finisher, tr, early);
  if (C <= 4) return select_split<4>(x, n, q, idx_out, xs_out, sel_out, S, finisher, tr, early);
  if (C <= 8) return select_split<8>(x, n, q, idx_out, xs_out, sel_out, S, finisher, tr, early);
  return -1;
}


// Block-barrier variant of the split order (same positions as select_split): after D is placed
// every thread calls early(D) -- which must only issue cp.async (no register destinations:
// a block barrier would wait for those) -- then all threads place R with one more block scan.
// Four block barriers; sel_out (if non-null) in ascending order.
template <int MAXC, typename Early>
__device__ __forceinline__ int select_split_bar(const uint16_t* __restrict__ x, int n, int q, int* __restrict__ idx_out,
                                                uint16_t* __restrict__ xs_out, int* __restrict__ sel_out,
                                                SelectSmemR* S, unsigned long long* tr, Early&& early) {
#define SEL_TRACE(i)                                  \
  do {                                                \
    if (tr && threadIdx.x == 0) tr[i] = clock64();     \
  } while (0)
  const int t = threadIdx.x, NT = blockDim.x, lane = t & 31, wid = t >> 5, nw = NT >> 5;
  const int n8 = n >> 3;
  const int C = (n8 + NT - 1) / NT;
  const int c0 = t * C;
  const int nv = max(0, min(C, n8 - c0));
  uint4 v[MAXC];
  const uint4* x4 = reinterpret_cast<const uint4*>(x) + c0;
#pragma unroll
  for (int m = 0; m < MAXC; ++m) v[m] = m < nv ? __ldg(x4 + m) : make_uint4(0, 0, 0, 0);
  SEL_TRACE(16);
  uint32_t* hA = S->histA[lane & (kHistACopies - 1)];
#pragma unroll
  for (int m = 0; m < MAXC; ++m) {
    if (m < nv) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t b = (chunk_elem(v[m], j) & 0x7fffu) >> 7;
        atomicAdd(&hA[b + (b >> 3)], 1u);
      }
    }
  }
  __syncthreads();  // barrier 1
  uint32_t bA, nD;
  {
    uint32_t c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      c[j] = S->histA[0][9 * lane + j] + S->histA[1][9 * lane + j] + S->histA[2][9 * lane + j] + S->histA[3][9 * lane + j];
    warp_find_bin_all<8>(c, (uint32_t)q, &bA, &nD);
  }
  SEL_TRACE(17);
  uint32_t n_d = 0;
#pragma unroll
  for (int m = 0; m < MAXC; ++m) {
    if (m < nv) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t key = chunk_elem(v[m], j) & 0x7fffu;
        const uint32_t b = key >> 7;
        n_d += b > bA;
        if (b == bA) {
          const uint32_t fb = key & 127u;
          atomicAdd(&S->histB[fb + (fb >> 2)], 1u);
        }
      }
    }
  }
  uint32_t inc_d = n_d;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc_d, o);
    if (lane >= o) inc_d += u;
  }
  if (lane == 31) S->wsum[wid] = inc_d;
  __syncthreads();  // barrier 2: histB complete, D warp totals visible
  uint32_t pre_d;
  {
    const uint32_t wt = lane < nw ? S->wsum[lane] : 0u;
    uint32_t wi = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += u;
    }
    const uint32_t wpre = __shfl_sync(0xffffffffu, wi - wt, wid);
    pre_d = wpre + inc_d - n_d;
  }
  if (n_d) {
    int pos = (int)pre_d;
#pragma unroll
    for (int m = 0; m < MAXC; ++m) {
      if (m < nv) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t raw = chunk_elem(v[m], j);
          if (((raw & 0x7fffu) >> 7) > bA) {
            idx_out[pos] = 8 * (c0 + m) + j;
            xs_out[pos] = (uint16_t)raw;
            ++pos;
          }
        }
      }
    }
  }
  uint32_t T, need_u;
  {
    uint32_t c[4], bin, above;
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = S->histB[5 * lane + j];
    warp_find_bin_all<4>(c, (uint32_t)q - nD, &bin, &above);
    T = (bA << 7) | bin;
    need_u = (uint32_t)q - nD - above;
  }
  const int need = (int)need_u;
  uint32_t n_g = 0, n_eq = 0;
#pragma unroll
  for (int m = 0; m < MAXC; ++m) {
    if (m < nv) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t key = chunk_elem(v[m], j) & 0x7fffu;
        n_g += (key >> 7) == bA && key > T;
        n_eq += key == T;
      }
    }
  }
  const uint32_t mine = (n_eq << 16) | n_g;
  uint32_t inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  __syncthreads();  // barrier 3: D placed; wsum (D) and histB read by every warp
  SEL_TRACE(18);
  early((int)nD);
  if (lane == 31) S->wsum[wid] = inc;
  __syncthreads();  // barrier 4: R warp totals visible
  uint32_t wpre;
  {
    const uint32_t wt = lane < nw ? S->wsum[lane] : 0u;
    uint32_t wi = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += u;
    }
    wpre = __shfl_sync(0xffffffffu, wi - wt, wid);
  }
  SEL_TRACE(19);
  const uint32_t pre = wpre + inc - mine;
  if (n_g + n_eq || (sel_out && n_d)) {
    int eq_seen = (int)(pre >> 16);
    int g_seen = (int)(pre & 0xffffu);
    int d_seen = (int)pre_d;
#pragma unroll
    for (int m = 0; m < MAXC; ++m) {
      if (m < nv) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t raw = chunk_elem(v[m], j);
          const uint32_t key = raw & 0x7fffu;
          const int i = 8 * (c0 + m) + j;
          const uint32_t b = key >> 7;
          if (b > bA) {
            if (sel_out) sel_out[d_seen + g_seen + min(eq_seen, need)] = i;
            ++d_seen;
          } else if (b == bA && key > T) {
            const int r = (int)nD + g_seen + min(eq_seen, need);
            idx_out[r] = i;
            xs_out[r] = (uint16_t)raw;
            if (sel_out) sel_out[d_seen + g_seen + min(eq_seen, need)] = i;
            ++g_seen;
          } else if (key == T) {
            if (eq_seen < need) {
              idx_out[(int)nD + g_seen + eq_seen] = i;
              xs_out[(int)nD + g_seen + eq_seen] = (uint16_t)raw;
              if (sel_out) sel_out[d_seen + g_seen + eq_seen] = i;
            }
            ++eq_seen;
          }
        }
      }
    }
  }
  return (int)nD;
#undef SEL_TRACE
}

template <typename Early>
__device__ __forceinline__ int select_split_bar_any(const uint16_t* x, int n, int q, int* idx_out, uint16_t* xs_out,
                                                    int* sel_out, SelectSmemR* S, unsigned long long* tr, Early&& early) {
  const int C = ((n >> 3) + (int)blockDim.x - 1) / (int)blockDim.x;
  if (C <= 1) return select_split_bar<1>(x, n, q, idx_out, xs_out, sel_out, S, tr, early);
  if (C <= 2) return select_split_bar<2>(x, n, q, idx_out, xs_out, sel_out, S, tr, early);
  if (C <= 4) return select_split_bar<4>(x, n, q, idx_out, xs_out, sel_out, S, tr, early);
  if (C <= 8) return select_split_bar<8>(x, n, q, idx_out, xs_out, sel_out, S, tr, early);
  return -1;
}

// Standalone selector (decdec_select): one block per segment.
__global__ void __launch_bounds__(1024) k_select(const uint16_t* __restrict__ x, int d_in, int k, int chunk,
                                                 int* __restrict__ idx_out, uint16_t* __restrict__ xs_out,
                                                 int* __restrict__ sel_out) {
  extern __shared__ __align__(16) uint8_t dsm[];
  const int seg = blockIdx.x;
  const int a = chunk ? seg * chunk : 0;
  const int n = chunk ? min(chunk, d_in - a) : d_in;
  const int q = chunk ? min(k, n) : k;
  const int out_off = chunk ? seg * k : 0;  // every earlier chunk is full length >= k
  if (q <= 0) return;
  select_block(x + a, n, q, a, idx_out + out_off, xs_out + out_off, sel_out ? sel_out + out_off : nullptr,
               reinterpret_cast<SelectSmem*>(dsm), reinterpret_cast<uint4*>(dsm + sizeof(SelectSmem)));
}

}  // namespace decdec
