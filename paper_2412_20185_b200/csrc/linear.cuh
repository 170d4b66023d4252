// Fused DecDEC layer kernel for sm_100a: base GEMV (HBM stream) + dynamic error
// compensation (PCIe zero-copy gather) + deterministic combine, in ONE persistent launch.
//
// PAPER.md P:207 runs steps 2-4 "in parallel with the base GEMV on a different GPU stream";
// here they run in parallel inside one kernel by warp specialisation:
//   warp 0              producer: 1-D bulk async copies (TMA engine, cp.async.bulk) of
//                       TR packed rows + their scales/zeros into a `stages`-deep smem ring
//                       (mbarrier full/empty pairs), L2 evict-first.
//   warps 1..NC         consumers: a thread owns input group g (128 channels, x kept in 64
//                       registers for the whole launch) and a row slot; per tile it computes
//                       RPS rows, two at a time (6-8 independent FHFMA chains), decoding codes
//                       in registers (decode.cuh), fp32 accumulation, then the group's z, s.
//                       G | 32: a warp holds 32/G whole rows -> shuffle reduction only;
//                       else NKW warps per row -> shuffle + one named barrier per team/tile.
//   warps NC+1..NC+NGW  gather warps (only when k > 0): wait for the selector kernel
//                       (programmatic dependent launch), stage S and x[S] in smem, then for
//                       work item (256-column segment, j) stream row blocks j, j+gws, ... of
//                       R_hat[S, segment] from pinned host memory with zero-copy loads
//                       (P:251), double-buffered (16 rows in flight per warp), decode + FHFMA,
//                       one fp32 partial per item.
// Combine (P:207 step 4; the paper uses atomics): GEMV warps publish their o_b rows
// and gather warps their partials, each with one fence and an arrival count per 256-column
// segment; the segment's last gather warp waits for its o_b rows and writes
// y = fp16(o_b + S_j * sum_j part_j) in a fixed order, then resets the counters.  No value
// atomics -> bit-reproducible.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <type_traits>
#include "ptx.cuh"
#include "decode.cuh"
#include "p2p.cuh"
#include "select.cuh"

namespace decdec {

constexpr int kGatherRows4 = 32;  // residual rows per gather item, 4-bit R (one u32 per lane per row)
constexpr int kGatherRows16 = 8;  // ... fp16 R (16 B per lane per row)
constexpr int kSelRegChunks = 8;  // register-resident selection: <= 8 chunks of 8 keys per thread
constexpr int kSegCols = 256;     // output columns per combine segment (128 B of 4-bit codes)
constexpr int kMaxThreads = 544;  // 1 producer + <= 16 consumer warps
constexpr int kMaxRPS = 4;       // rows per slot per tile
#ifndef DECDEC_ROW_STEP
#define DECDEC_ROW_STEP 2  // consumer rows per inner step: 2 (row pairs, more ILP) or 1 (smaller loop)
#endif
constexpr int kCntSlots = 4096;   // arrival counters at the head of the workspace
constexpr int kCtrlSlots = 16;    // last slots of that region: reserved control words
// trace events (per CTA): 0 start, 1 gather done (2nd gather warp), 2 x loaded, 3 first stage landed,
// 4 GEMV done, 5 selector start, 6 selection published, 7 gather done, 8 consumers released (PDL),
// 9 last combine done (CTA), 10 last warp exits (CTA), 11 gather warps see the selection,
// 12 partials published (start), 13 last arrival seen, 14 o_b rows seen, 15 combine loads landed,
// 16-19 DEC CTA selection phases (x staged, coarse bin, threshold, scan)
constexpr int kTraceEvents = 20;
#define DECDEC_TRACE(p, ev)                                                        \
  do {                                                                             \
    if ((p).trace) (p).trace[blockIdx.x * kTraceEvents + (ev)] = globaltimer();    \
  } while (0)

struct LinearParams {
  const uint8_t* w;      // packed weights (W3K/W4K), [d_out][row_bytes]
  const uint16_t* ws;    // fp16 scales [d_out][G]
  const uint8_t* wz;     // u8 zeros [d_out][G]
  const uint16_t* x;     // fp16 [d_in]
  uint16_t* y;           // fp16 [d_out]
  int d_in, d_out, G, row_bytes;
  int TR, NC, stages, n_tiles;
  int NKW;     // warps per row team; 0 = a warp holds 32/G whole rows (G divides 32)
  int NSLOTS;  // concurrent row slots per CTA: NC*32/G (G <= 32) or NC/NKW (G > 32)
  int RPS;     // rows per slot per tile (TR = NSLOTS * RPS)
  uint32_t stage_bytes, off_s, off_z;
  // compensation (k_sel == 0: none)
  int k_sel;
  const uint8_t* r_rows;
  const uint16_t* r_scales;
  int r_row_bytes;
  float* ob;      // workspace: fp32 o_b = W_hat x (GEMV CTAs -> DEC combine); kObEmpty = not yet written
  int n_seg, gws;  // gws = gather items (row chunks) per segment
  int nparts;      // partials per segment: min(gws, warps) when one_seg, else gws
  int one_seg;     // n_seg <= n_dec: a DEC CTA owns at most one segment
  int rpi;               // selected rows per gather item (<= kGatherRows4 / kGatherRows16)
  // smem layout of a DEC CTA: SelectSmem, the staged x segment, idx int32[k_sel], xs u16[k_sel],
  // partials f32[ns][gws][kSegCols], residual scales u16[ns][kSegCols]
  uint32_t off_sel, off_part, off_rsc, off_stage;  // ... + per-warp gather staging [warps][2][rows][32]
  uint32_t off_x;        // GEMV CTAs: smem offset of the staged x (d_in fp16, 16-B units swizzled)
  unsigned long long* trace;  // optional per-CTA event timestamps [grid][kTraceEvents] (ns), or null
  // The first n_dec CTAs are DEC CTAs (steps 1-4): each computes the exact Top-k itself (same
  // deterministic result in every DEC CTA, no cross-CTA hand-off), keeps S and x[S] in smem and
  // gathers its share of the (segment, row chunk) items.  The other CTAs run the GEMV.
  int n_dec, k_req, chunk;
  int early_reads;  // read the D rows' bytes during the selection (plan: PCIe/HBM ratio window)
  int early_cap;    // ... at most this many rows per warp (0 = all)
  int prefetch;  // weight tiles requested per CTA (into smem) before griddepcontrol.wait
  int l2pf;      // further tiles per CTA prefetched into L2 only before griddepcontrol.wait
  int x_pf;      // prefetch x into L2 before griddepcontrol.wait
  int* sel_out;
  // debug (decdec_debug_selections): DEC CTA c < dbg_ctas writes its own S / x[S] (in its
  // placement order) to dbg_idx[c * dbg_cap ...] / dbg_xs[...]; null = off
  int* dbg_idx;
  uint16_t* dbg_xs;
  int dbg_cap, dbg_ctas;
  P2PParams pp;  // fused P2P all-gather (p2p.cuh); pp.nranks <= 1: plain local y stores
  // multi-link residual fetch (NEXT-4, decdec_linear_ml): the DEC CTAs gather only the selected
  // positions e with e % share_n == share_r.  A helper rank (ml_out) writes its o_dec part
  // (fp32, x S_j) into the main rank's buffer over NVLink instead of combining; the main rank
  // (ml_in) adds the helpers' parts in rank order.  Per DEC CTA c: the helper waits until its
  // ack word c is clear, sets it, writes, and releases one count to the main's flag c; the main
  // acquires share_n - 1 counts, re-arms its flag, combines, then clears every helper's ack c.
  int share_n, share_r;
  float* ml_out;                          // helper: its part buffer in the main rank's region (peer)
  unsigned int* ml_out_flag;              // helper: the main rank's flags [n_dec] (peer)
  unsigned int* ml_ack;                   // helper: its own ack words [n_dec]
  const float* ml_in;                     // main: the helpers' parts [share_n - 1][d_out] (local)
  unsigned int* ml_flag;                  // main: its flags [n_dec]
  unsigned int* ml_peer_ack[kMaxPeers];   // main: helper h's ack words (peer), h = 1 .. share_n - 1
};

// A DEC CTA (steps 1-4 of P:207).  DEC CTA c owns the output segments c, c + n_dec, ...:
//   1. every DEC CTA computes the exact Top-k itself (same deterministic result, no hand-off);
//   2-3. its warps gather the items (local segment, row chunk j) from pinned host memory with
//        zero-copy loads, double-buffered (the next item's loads are in flight while the
//        current one is decoded), one fp32 partial per item into smem;
//   4. after a CTA barrier, a warp per segment waits for the segment's o_b rows (GEMV arrival
//      count), adds S_j * sum_j part_j in fixed order and writes y.  No global partials, no
//      value atomics -> deterministic.
// MLF = 1: the multi-link residual fetch (NEXT-4) build -- position shares and the helper / main
// hand-off; MLF = 0 compiles none of it (the single-GPU and tensor-parallel paths)
template <int RBITS, int MLF = 0>
__device__ __forceinline__ void dec_cta(const LinearParams& p, uint8_t* smem, int warp, int lane) {
  SelectSmem* S = reinterpret_cast<SelectSmem*>(smem);
  uint4* sx4 = reinterpret_cast<uint4*>(smem + sizeof(SelectSmem));
  SelectSmemR* SR = reinterpret_cast<SelectSmemR*>(smem);  // register-resident selector (aliases S)
  SelectSmemS* SS = reinterpret_cast<SelectSmemS*>(smem);  // split-order selector (aliases S)
  int* sidx = reinterpret_cast<int*>(smem + p.off_sel);
  uint16_t* sxs = reinterpret_cast<uint16_t*>(sidx + p.k_sel);
  float* spart = reinterpret_cast<float*>(smem + p.off_part);    // [ns][nparts][kSegCols]
  uint16_t* srsc = reinterpret_cast<uint16_t*>(smem + p.off_rsc);  // [ns][kSegCols] residual scales
  unsigned long long* tr = p.trace ? p.trace + blockIdx.x * kTraceEvents : nullptr;
  const int seg_len = p.chunk ? min(p.chunk, p.d_in) : p.d_in;
  const bool regs = (seg_len / 8 + (int)blockDim.x - 1) / (int)blockDim.x <= kSelRegChunks;
  const bool split = !p.chunk && regs && p.d_in <= 32 * 1024;
#ifndef DECDEC_SPLIT_BARRIER
  if (split) select_split_zero(SS, p.d_in);  // before the wait: smem is ours already
#else
  if (split) select_regs_zero(SR);
#endif
  else if (regs) select_regs_zero(SR);
  const int nw = blockDim.x >> 5;
  const int ns = (p.n_seg - (int)blockIdx.x + p.n_dec - 1) / p.n_dec;  // local segments
  uint64_t* scale_bar = reinterpret_cast<uint64_t*>(srsc + ns * kSegCols);
  if (RBITS == 4 && threadIdx.x == 0) {
    // all scale factors are fetched every call; they do not depend on x, so they are
    // requested before griddepcontrol.wait, as one bulk copy (TMA) per segment: exactly the
    // segment's bytes cross PCIe (16-B cp.async per lane read every 32-B sector twice, ncu),
    // and no LSU work; the combine waits on scale_bar
    mbar_init(scale_bar, 1);
    fence_mbar_init();
    uint32_t bytes = 0;
    for (int i = 0; i < ns; ++i) {
      const int c = ((int)blockIdx.x + i * p.n_dec) * kSegCols;
      if (c < p.d_out) bytes += (uint32_t)min(kSegCols, p.d_out - c) * 2;
    }
    mbar_arrive_expect_tx(scale_bar, bytes);
    const uint64_t pol = policy_evict_first();
    for (int i = 0; i < ns; ++i) {
      const int c = ((int)blockIdx.x + i * p.n_dec) * kSegCols;
      if (c < p.d_out) bulk_g2s(srsc + i * kSegCols, p.r_scales + c, (uint32_t)min(kSegCols, p.d_out - c) * 2, scale_bar, pol);
    }
  }
  __syncthreads();
  pdl_wait();  // x may be the previous layer's product; the workspace is the previous layer's
  if (p.pp.prev_flag) {  // TP stack: the previous layer's y_full is complete on every rank
    if (threadIdx.x == 0) p2p_wait_prev(p.pp);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    DECDEC_TRACE(p, 5);
    if (tr) tr[15] = clock64();  // selection phases 16-19 are SM cycles relative to this
  }
  const int n_items = ns * p.gws;
  // this CTA's share of the selected positions (all of them unless the multi-link fetch splits
  // them across ranks): local index e -> position share_r + e * share_n
  const int share_n = MLF ? p.share_n : 1, share_r = MLF ? p.share_r : 0;
  const int k_local = MLF ? (p.k_sel - share_r + share_n - 1) / share_n : p.k_sel;
  using Vec = typename std::conditional<RBITS == 4, uint32_t, uint4>::type;
  constexpr int kGR = RBITS == 4 ? kGatherRows4 : kGatherRows16;
  // per-warp staging: 2 buffers x kGR rows x 32 lanes x Vec (cp.async destinations)
  Vec* stage = reinterpret_cast<Vec*>(smem + p.off_stage) + (size_t)warp * 2 * p.rpi * 32;
#ifndef DECDEC_NARROW_GATHER
  // 4-bit R, wide gather: ONE 16-B cp.async per lane covers 4 rows x the segment's 128 B (lanes
  // 8r..8r+7 read row r's 16-B chunks), so each warp instruction moves 512 B.  A B200 SM keeps
  // only a few zero-copy instructions in flight: 16-B requests gather ~4x faster per SM than
  // 4-B ones (csrc/probe measurement in DESIGN.md §6c), which matters when a layer has few DEC CTAs
  // (tensor-parallel shards).  Lane l accumulates the 32 columns (l & 7) * 32 .. +31 of its rows;
  // store_part folds the 4 row groups with two shuffles (fixed order).
  constexpr bool kWide = RBITS == 4;
#else
  constexpr bool kWide = false;
#endif
  constexpr int kAccN = kWide ? 32 : 8;
  auto issue = [&](int it, int bsel) {  // all zero-copy reads of item `it` (async, into smem)
    const int i = it % ns, j = it / ns;
    if constexpr (kWide) {
      const int segc0 = ((int)blockIdx.x + i * p.n_dec) * kSegCols;
      const bool cv = segc0 + (lane & 7) * 32 < p.d_out;
      const int e0 = j * p.rpi, e1 = min(e0 + p.rpi, k_local);
      uint4* dst = reinterpret_cast<uint4*>(stage) + bsel * p.rpi * 8 + lane;
#pragma unroll
      for (int r4 = 0; r4 < kGR / 4; ++r4) {
        const int rr = r4 * 4 + (lane >> 3), e = e0 + rr;
        if (rr < p.rpi && e < e1 && cv) {
          const uint8_t* rowp = p.r_rows + (size_t)sidx[share_r + e * share_n] * p.r_row_bytes;
          cp_async_16_ca(dst + r4 * 32, rowp + (segc0 >> 1) + (lane & 7) * 16);
        }
      }
      cp_async_commit();
      return;
    }
    const int col0 = ((int)blockIdx.x + i * p.n_dec) * kSegCols + lane * 8;
    const bool cv = col0 < p.d_out;
    const int e0 = j * p.rpi, e1 = min(e0 + p.rpi, k_local);
    Vec* dst = stage + bsel * p.rpi * 32 + lane;
#pragma unroll
    for (int r = 0; r < kGR; ++r) {
      const int e = e0 + r;
      if (r < p.rpi && e < e1 && cv) {
        const uint8_t* rowp = p.r_rows + (size_t)sidx[share_r + e * share_n] * p.r_row_bytes;
        if constexpr (RBITS == 4) cp_async_4(dst + r * 32, rowp + (col0 >> 1));
        else cp_async_16(dst + r * 32, rowp + col0 * 2);
      }
    }
    cp_async_commit();
  };
  auto consume = [&](int it, int bsel, float* acc) {  // decode + FHFMA into acc[kAccN]
    const int j = it / ns;
    const int e0 = j * p.rpi, e1 = min(e0 + p.rpi, k_local);
    if constexpr (kWide) {
      const uint4* src4 = reinterpret_cast<const uint4*>(stage) + bsel * p.rpi * 8 + lane;
#pragma unroll
      for (int r4 = 0; r4 < kGR / 4; ++r4) {
        const int rr = r4 * 4 + (lane >> 3), e = e0 + rr;
        if (rr < p.rpi && e < e1) {
          const uint16_t xv = sxs[share_r + e * share_n];
          const uint4 w4 = src4[r4 * 32];
          const uint32_t wd[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t cq[4];
            decode_rq_word(wd[q], cq);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              acc[8 * q + 2 * u] = fhfma_s_lo(xv, cq[u], acc[8 * q + 2 * u]);
              acc[8 * q + 2 * u + 1] = fhfma_s_hi(xv, cq[u], acc[8 * q + 2 * u + 1]);
            }
          }
        }
      }
      return;
    }
    const Vec* src = stage + bsel * p.rpi * 32 + lane;
#pragma unroll
    for (int r = 0; r < kGR; ++r) {
      const int e = e0 + r;
      if (r < p.rpi && e < e1) {
        const uint16_t xv = sxs[share_r + e * share_n];
        const Vec w = src[r * 32];
        uint32_t cq[4];
        if constexpr (RBITS == 4) {
          decode_rq_word(w, cq);
        } else {
          cq[0] = w.x; cq[1] = w.y; cq[2] = w.z; cq[3] = w.w;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc[2 * u] = fhfma_s_lo(xv, cq[u], acc[2 * u]);
          acc[2 * u + 1] = fhfma_s_hi(xv, cq[u], acc[2 * u + 1]);
        }
      }
    }
  };
  // Partials: with one local segment (ns == 1) a warp's items all belong to it, so the warp
  // accumulates them in registers and leaves ONE partial (slot = warp); otherwise one partial
  // per item (slot = row chunk j).  p.nparts = partials per segment (combined in slot order).
  auto store_part = [&](int i, int slot, float* acc) {
    if constexpr (kWide) {  // fold the 4 row groups: (g0 + g1) + (g2 + g3), then lanes 0..7 store
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 8);
        acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 16);
      }
      if (lane < 8) {
        float* pp = spart + ((size_t)i * p.nparts + slot) * kSegCols + lane * 32;
#pragma unroll
        for (int c = 0; c < 32; c += 4) *reinterpret_cast<float4*>(pp + c) = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) acc[c] = 0.f;
      return;
    }
    float* pp = spart + ((size_t)i * p.nparts + slot) * kSegCols + lane * 8;
    *reinterpret_cast<float4*>(pp) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    *reinterpret_cast<float4*>(pp + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.f;
  };
  int it = warp;
  // ---- step 1: exact Top-k (whole x, or per chunk), S and x[S] into smem.  In global mode the
  // rows whose coarse bin is above the threshold bin (positions [0, nD)) are known after three
  // block barriers; the last warp finishes the rest alone while the others start gathering.
  int nD = -1;
  bool issued = false;
  if (split) {
#ifndef DECDEC_SPLIT_BARRIER
    {
      // D rows are known before barrier 2: when the plan asks for it (p.early_reads), this CTA
      // reads their bytes of all its segments right away -- cp.async.ca into a scratch slot, so
      // the lines land in this SM's L1 and the gather that follows hits them.  Measured (1x B200,
      // Llama-3-8B step): k_chunk 21 -3.6 %, k_chunk 1-4 +2-3 % (the reads delay the selection's
      // last phases while few rows profit), hence a window on the call's PCIe/HBM ratio.
      struct Early {
        const LinearParams* pp;
        Vec* dummy;
        int ns, lane;
        __device__ __forceinline__ bool on() const { return pp->early_reads != 0; }
        __device__ __forceinline__ int cap() const { return pp->early_cap & 0xffff; }
        // the finisher warp issues none (its R placement does not queue behind zero-copy requests)
        __device__ __forceinline__ bool spare_finisher() const { return (pp->early_cap >> 16) != 0; }
        __device__ __forceinline__ void operator()(int row) const {
          const uint8_t* rowp = pp->r_rows + (size_t)row * pp->r_row_bytes;
          for (int i = 0; i < ns; ++i) {
            const int col0 = ((int)blockIdx.x + i * pp->n_dec) * kSegCols + lane * 8;
            if (col0 < pp->d_out) {
              if constexpr (RBITS == 4) cp_async_4(dummy, rowp + (col0 >> 1));
              else cp_async_16(dummy, rowp + col0 * 2);
            }
          }
        }
      } early{&p, reinterpret_cast<Vec*>(SS->scratch) + lane, ns, lane};
      nD = select_split_any(p.x, p.d_in, p.k_req, sidx, sxs, blockIdx.x == 0 ? p.sel_out : nullptr, SS, nw - 1, tr, early);
      if (p.early_reads) cp_async_commit();
    }
#else
    auto early = [&](int n_def) {  // cp.async only: the remaining block barriers do not wait for it
      if (it < n_items && min((it / ns) * p.rpi + p.rpi, p.k_sel) <= n_def) {
        issue(it, 0);
        issued = true;
      }
    };
    nD = select_split_bar_any(p.x, p.d_in, p.k_req, sidx, sxs, blockIdx.x == 0 ? p.sel_out : nullptr, SR, tr, early);
    if (nD >= 0) {
      __syncthreads();  // R placed
      nD = p.k_sel;
    }
#endif
#ifdef DECDEC_SPLIT_SERIAL
    __syncthreads();  // experiment switch: wait for the finisher before any gather
    if (nD >= 0) nD = p.k_sel;
#endif
  }
  if (nD < 0) {
    const int n_chunks = p.chunk ? (p.d_in + p.chunk - 1) / p.chunk : 1;
    for (int c = 0; c < n_chunks; ++c) {
      const int a = p.chunk ? c * p.chunk : 0;
      const int n = p.chunk ? min(p.chunk, p.d_in - a) : p.d_in;
      const int q = p.chunk ? min(p.k_req, n) : p.k_req;
      const int off = p.chunk ? c * p.k_req : 0;  // every earlier chunk is full length >= k
      int* so = (blockIdx.x == 0 && p.sel_out) ? p.sel_out + off : nullptr;
      if (regs)
        select_block_regs_any(p.x + a, n, q, a, sidx + off, sxs + off, so, SR, c == 0 ? tr : nullptr);
      else
        select_block(p.x + a, n, q, a, sidx + off, sxs + off, so, S, sx4, c == 0 ? tr : nullptr);
      __syncthreads();  // outputs complete; the selector scratch is free for the next chunk
    }
    nD = p.k_sel;
  }
  bool rest_seen = nD >= p.k_sel;
  auto ready = [&](int item) {  // the rows of `item` are placed (its last position is < nD)
    if (!rest_seen && share_r + (min((item / ns) * p.rpi + p.rpi, k_local) - 1) * share_n >= nD) {
      select_wait_rest(SS);
      rest_seen = true;
    }
  };
  if (threadIdx.x == 0) {
    DECDEC_TRACE(p, 6);
    if (tr) tr[14] = clock64();
  }
  // ---- steps 2-3: gather rows S of R_hat x x[S] for this CTA's segments (double-buffered)
  if (it < n_items && !issued) {
    ready(it);
    if (tr && warp == 0 && lane == 0) tr[2] = clock64();  // DEC CTAs: cycle stamps in slots 2-4, 10
    issue(it, 0);
  }
  float acc[kAccN];
#pragma unroll
  for (int c = 0; c < kAccN; ++c) acc[c] = 0.f;
  const bool one_seg = p.one_seg;  // plan-wide: every DEC CTA has <= 1 segment
  const bool had_item = it < n_items;
  for (int b = 0; it < n_items; b ^= 1, it += nw) {
    if (it + nw < n_items) {
      ready(it + nw);
      issue(it + nw, b ^ 1);
      cp_async_wait<1>();  // this item's group has landed (the next one may be in flight)
    } else {
      cp_async_wait<0>();
    }
    if (tr && warp == 0 && lane == 0 && it == 0) tr[3] = clock64();  // first item landed
    consume(it, b, acc);
    if (!one_seg) store_part(it % ns, it / ns, acc);
  }
  cp_async_wait<0>();  // no cp.async (gather or early read) outstanding past this point
  if (one_seg && had_item) store_part(0, warp, acc);
  if (lane == 0 && (warp == 0 || warp == nw - 1)) DECDEC_TRACE(p, warp == 0 ? 7 : 1);  // gather done
  // the combine warp of local segment `warp` reads its o_b entries before the barrier: the GEMV
  // CTAs normally stored them long ago, so the L2 round trip overlaps the slowest warp's gather
  uint4 ob0 = make_uint4(kObEmpty, kObEmpty, kObEmpty, kObEmpty), ob1 = ob0;
  {
    const int col0 = ((int)blockIdx.x + warp * p.n_dec) * kSegCols + lane * 8;
    if (warp < ns && col0 < p.d_out) {
      ob0 = ld_relaxed_gpu_u4(p.ob + col0);
      ob1 = ld_relaxed_gpu_u4(p.ob + col0 + 4);
    }
  }
  __syncthreads();  // all partials of the CTA's segments are in smem
  if (RBITS == 4 && warp < ns) mbar_wait(scale_bar, 0);  // the scales' bulk copies landed
  if (tr && threadIdx.x == 0) tr[4] = clock64();
  if (threadIdx.x == 0) DECDEC_TRACE(p, 12);
  if (MLF && p.ml_out) {  // multi-link helper: this rank's o_dec part -> the main rank, no combine
    if (threadIdx.x == 0) {  // the main rank has consumed this CTA's previous part
      const unsigned long long t0 = globaltimer();
      while (ld_acquire_sys_u32(p.ml_ack + blockIdx.x) != 0u) {
        __nanosleep(64);
        if (globaltimer() - t0 > 20000000000ull) __trap();
      }
      p.ml_ack[blockIdx.x] = 1u;
    }
    __syncthreads();
    for (int i = warp; i < ns; i += nw) {
      const int col0 = ((int)blockIdx.x + i * p.n_dec) * kSegCols + lane * 8;
      if (col0 < p.d_out) {
        float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int j = 0; j < p.nparts; ++j) {  // fixed order: slots ascending
          const float* pp = spart + ((size_t)i * p.nparts + j) * kSegCols + lane * 8;
          const float4 a = *reinterpret_cast<const float4*>(pp), b = *reinterpret_cast<const float4*>(pp + 4);
          v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
          v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
        }
        if (RBITS == 4) {
          const uint4 sv = *reinterpret_cast<const uint4*>(srsc + i * kSegCols + lane * 8);
          const uint32_t sw[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            v[2 * e] *= __half2float(__ushort_as_half((unsigned short)(sw[e] & 0xffffu)));
            v[2 * e + 1] *= __half2float(__ushort_as_half((unsigned short)(sw[e] >> 16)));
          }
        }
        *reinterpret_cast<float4*>(p.ml_out + col0) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(p.ml_out + col0 + 4) = make_float4(v[4], v[5], v[6], v[7]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p.ml_out_flag + blockIdx.x) : "memory");
    }
    return;
  }
  if (MLF && p.ml_in) {  // multi-link main: every helper's part of this CTA's segments has landed
    if (threadIdx.x == 0) {
      const unsigned long long t0 = globaltimer();
      while (ld_acquire_sys_u32(p.ml_flag + blockIdx.x) < (unsigned)(p.share_n - 1)) {
        __nanosleep(64);
        if (globaltimer() - t0 > 20000000000ull) __trap();
      }
      p.ml_flag[blockIdx.x] = 0u;  // re-armed: no helper writes again before its ack is cleared
    }
    __syncthreads();
  }
  // ---- step 4: combine, one warp per local segment.  o_b entries are self-validating (relaxed
  // stores of the GEMV CTAs, kObEmpty until written): poll them, then restore kObEmpty.
  for (int i = warp; i < ns; i += nw) {
    const int seg = (int)blockIdx.x + i * p.n_dec;
    const int col0 = seg * kSegCols + lane * 8;
    if (col0 < p.d_out) {
      uint4 o0 = ob0, o1 = ob1;
      if (i != warp) {
        o0 = ld_relaxed_gpu_u4(p.ob + col0);
        o1 = ld_relaxed_gpu_u4(p.ob + col0 + 4);
      }
      while ((o0.x == kObEmpty) | (o0.y == kObEmpty) | (o0.z == kObEmpty) | (o0.w == kObEmpty) |
             (o1.x == kObEmpty) | (o1.y == kObEmpty) | (o1.z == kObEmpty) | (o1.w == kObEmpty)) {
        __nanosleep(32);
        o0 = ld_relaxed_gpu_u4(p.ob + col0);
        o1 = ld_relaxed_gpu_u4(p.ob + col0 + 4);
      }
      if (tr && i == 0 && lane == 0) tr[10] = clock64();  // o_b rows seen
      float sum[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < p.nparts; ++j) {  // fixed order: slots ascending
        const float* pp = spart + ((size_t)i * p.nparts + j) * kSegCols + lane * 8;
        const float4 a = *reinterpret_cast<const float4*>(pp), b = *reinterpret_cast<const float4*>(pp + 4);
        sum[0] += a.x; sum[1] += a.y; sum[2] += a.z; sum[3] += a.w;
        sum[4] += b.x; sum[5] += b.y; sum[6] += b.z; sum[7] += b.w;
      }
      float Sc[8] = {1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f};
      if (RBITS == 4) {
        const uint4 sv = *reinterpret_cast<const uint4*>(srsc + i * kSegCols + lane * 8);
        const uint32_t sw[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          Sc[2 * e] = __half2float(__ushort_as_half((unsigned short)(sw[e] & 0xffffu)));
          Sc[2 * e + 1] = __half2float(__ushort_as_half((unsigned short)(sw[e] >> 16)));
        }
      }
      const float o[8] = {__uint_as_float(o0.x), __uint_as_float(o0.y), __uint_as_float(o0.z), __uint_as_float(o0.w),
                          __uint_as_float(o1.x), __uint_as_float(o1.y), __uint_as_float(o1.z), __uint_as_float(o1.w)};
      uint32_t out[4];
      if (MLF && p.ml_in) {  // own part x S_j, then the helpers' parts in rank order, then + o_b
        float d[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) d[e] = Sc[e] * sum[e];
        for (int h = 0; h < p.share_n - 1; ++h) {
          const float* hp = p.ml_in + (size_t)h * p.d_out + col0;
          const float4 a = ld_relaxed_sys_f4(hp), b = ld_relaxed_sys_f4(hp + 4);
          d[0] += a.x; d[1] += a.y; d[2] += a.z; d[3] += a.w;
          d[4] += b.x; d[5] += b.y; d[6] += b.z; d[7] += b.w;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const __half lo = __float2half_rn(o[2 * e] + d[2 * e]);
          const __half hi = __float2half_rn(o[2 * e + 1] + d[2 * e + 1]);
          out[e] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const __half lo = __float2half_rn(fmaf(Sc[2 * e], sum[2 * e], o[2 * e]));
          const __half hi = __float2half_rn(fmaf(Sc[2 * e + 1], sum[2 * e + 1], o[2 * e + 1]));
          out[e] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
        }
      }
      p2p_store_u4(p.pp, p.y, col0, make_uint4(out[0], out[1], out[2], out[3]));
      const uint4 empty = make_uint4(kObEmpty, kObEmpty, kObEmpty, kObEmpty);
      *reinterpret_cast<uint4*>(p.ob + col0) = empty;  // ready for the next call
      *reinterpret_cast<uint4*>(p.ob + col0 + 4) = empty;
    }
  }
  if (threadIdx.x == 0) DECDEC_TRACE(p, 9);
  if (MLF && p.ml_in) {  // the helpers' parts are consumed: let them write the next ones
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int h = 0; h < p.share_n - 1; ++h)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.ml_peer_ack[h] + blockIdx.x), "r"(0u) : "memory");
    }
  }
  if (p.pp.active) {  // fused all-gather: this CTA's segments are in every rank's y_full
    __syncthreads();
    if (threadIdx.x == 0) {
      p2p_signal(p.pp);
    }
  }
  if (p.dbg_idx && (int)blockIdx.x < p.dbg_ctas) {  // every DEC CTA's own selection, for tests
    if (split && nD < p.k_sel) select_wait_rest(SS);
    int* di = p.dbg_idx + (size_t)blockIdx.x * p.dbg_cap;
    uint16_t* dx = p.dbg_xs + (size_t)blockIdx.x * p.dbg_cap;
    for (int i = threadIdx.x; i < p.k_sel && i < p.dbg_cap; i += blockDim.x) {
      di[i] = sidx[i];
      dx[i] = sxs[i];
    }
  }
}

// LUTB = 0: uniform base (W3K / W4K codes, per-group fp16 scale + u8 zero); LUTB = 3 | 4: the
// non-uniform base (NEXT-3, P:397 / P:502): W4K nibble codes (BITS = 4) and, in place of the
// scales, each row's table of 2^LUTB fp16 values; no zeros.
template <int BITS, int RBITS, int LUTB = 0, int MLF = 0>
__global__ void __launch_bounds__(kMaxThreads, 1) k_linear(const LinearParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stage0 = smem;
  float* red = reinterpret_cast<float*>(smem + (size_t)p.stages * p.stage_bytes);  // [2][NSLOTS][4][NKW]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 2 * p.NSLOTS * 4 * max(p.NKW, 1));
  uint64_t* empty = full + p.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Let the next kernel of the stream launch now: its CTAs take SMs as ours retire and start
  // streaming their (static) weights while we finish (cross-layer overlap).
  pdl_launch_dependents();
  if (threadIdx.x == 0) DECDEC_TRACE(p, 0);
  // x into L2 before griddepcontrol.wait (a slice of its 128-B lines per CTA): every CTA's
  // first loads after the wait -- the selector's and the GEMV's -- then hit L2.  Safe even
  // while the previous kernel is still producing x: L2 is the coherence point.
  if (p.x_pf) {
    const int lines = (p.d_in * 2 + 127) >> 7;
    const int i = (int)threadIdx.x * 8 + ((int)blockIdx.x & 7);
    if (i < lines) prefetch_l2(reinterpret_cast<const uint8_t*>(p.x) + ((size_t)i << 7));
  }

  // ------------------------------------------------------------------ DEC CTAs (steps 1-4)
  if ((int)blockIdx.x < p.n_dec) {
    dec_cta<RBITS, MLF>(p, smem, warp, lane);
    return;
  }
  const int cta = blockIdx.x - p.n_dec, n_cta = gridDim.x - p.n_dec;  // GEMV CTA index / count
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], p.NC);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // ------------------------------------------------------------------ producer (TMA)
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const uint32_t wb = (uint32_t)p.TR * p.row_bytes;
      const uint32_t sb = LUTB ? (uint32_t)p.TR * (2u << LUTB) : (uint32_t)p.TR * p.G * 2;  // scales | tables
      const uint32_t zb = LUTB ? 0u : (uint32_t)p.TR * p.G;
      const int stages = p.stages;
      int it = 0, st = 0;
      uint32_t ph = 0;  // phase of the current pass over the ring
      // L2-only prefetch of the tiles after the smem burst: HBM -> L2 runs while the previous
      // layer finishes, without queueing ~µs of traffic in front of this SM's x loads
      for (int i = p.prefetch; i < p.prefetch + p.l2pf; ++i) {
        const int tile = cta + i * n_cta;
        if (tile >= p.n_tiles) break;
        bulk_prefetch_l2(p.w + (size_t)tile * wb, wb);
      }
      for (int tile = cta; tile < p.n_tiles; tile += n_cta, ++it) {
        // only `prefetch` tiles may be requested before the previous layer completes: a deeper
        // early burst floods the memory pipe and delays the x loads the consumers wait on
        if (it == p.prefetch) pdl_wait();
        if (it >= stages) mbar_wait(&empty[st], ph ^ 1);
        uint8_t* dst = stage0 + (size_t)st * p.stage_bytes;
        mbar_arrive_expect_tx(&full[st], wb + sb + zb);
        bulk_g2s(dst, p.w + (size_t)tile * wb, wb, &full[st], pol);
        bulk_g2s(dst + p.off_s, p.ws + (size_t)tile * p.TR * (LUTB ? (1 << LUTB) : p.G), sb, &full[st], pol);
        if (!LUTB) bulk_g2s(dst + p.off_z, p.wz + (size_t)tile * p.TR * p.G, zb, &full[st], pol);
        if (++st == stages) {
          st = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers (GEMV)
  if (warp <= p.NC) {
    constexpr int GB = 16 * BITS;  // bytes of one 128-code group
    const int ct = threadIdx.x - 32;
    const int cw = ct >> 5;
    const int G = p.G;
    const bool small_g = p.NKW == 0;  // a warp holds 32/G whole rows (G | 32); else NKW warps per row
    const int g = small_g ? (lane % G) : ((cw % p.NKW) * 32 + lane);
    const int slot = small_g ? (cw * (32 / G) + lane / G) : (cw / max(p.NKW, 1));
    const bool active = g < G;
    const int rot = (BITS == 4) ? ((g >> 1) & 3) : 0;  // 4-bit: bank-conflict-free 16-B chunk order
    // x (and the workspace) belong to the previous layer until it completes
    pdl_wait();
    if (p.pp.prev_flag) {  // TP stack: the previous layer's y_full is complete on every rank
      if (ct == 0) p2p_wait_prev(p.pp);
      named_bar_sync(12, p.NC * 32);
    }
    if (ct == 0) DECDEC_TRACE(p, 8);
    // Stage x in smem first: a lane owns 256 contiguous bytes of x, so loading its registers
    // straight from global memory touches 32 cache lines per instruction and the L1 serialises
    // them (~5000 cycles for 12 warps, measured).  Coalesced 16-B loads by all consumer threads
    // -> smem with unit c of group g stored at g*16 + (c ^ (g & 7)) -> conflict-free 16-B reads.
    uint4* xsm = reinterpret_cast<uint4*>(smem + p.off_x);
    {
      const int nx = p.d_in >> 3, nct = p.NC * 32;
      const uint4* xg = reinterpret_cast<const uint4*>(p.x);
      for (int u = ct; u < nx; u += nct) {
        const uint4 v = ld_nc_u4(xg + u);
        xsm[(u & ~15) | ((u & 15) ^ ((u >> 4) & 7))] = v;
      }
      named_bar_sync(14, nct);
    }
    uint32_t xr[64];
    float Xs = 0.f;
    if (active) {
      const uint4* xp = xsm + g * 16;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = (j + rot) & 3;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint4 v = xp[(4 * c + e) ^ (g & 7)];
          xr[16 * j + 4 * e + 0] = v.x;
          xr[16 * j + 4 * e + 1] = v.y;
          xr[16 * j + 4 * e + 2] = v.z;
          xr[16 * j + 4 * e + 3] = v.w;
        }
      }
      if (ct == 0) DECDEC_TRACE(p, 5);
#ifndef DECDEC_NO_XS
      // sum of the group's 128 x in fp32: FHFMA with 1.0 into 8 independent accumulators
      float xa[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      const uint32_t one2 = 0x3C003C00u;  // (1.0, 1.0) as half2
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        xa[i & 3] = fhfma_lo(one2, xr[i], xa[i & 3]);
        xa[4 + (i & 3)] = fhfma_hi(one2, xr[i], xa[4 + (i & 3)]);
      }
      Xs = ((xa[0] + xa[1]) + (xa[2] + xa[3])) + ((xa[4] + xa[5]) + (xa[6] + xa[7]));
#endif
      Xs *= 5.9604644775390625e-08f;  // 2^-24: same scale as the decoded codes
      if (LUTB) {
#pragma unroll
        for (int w = 0; w < 16; ++w) lut_x_pairs(xr + 4 * w);  // (c, c+2) pairing of the table lookups
      }
    } else {
#pragma unroll
      for (int i = 0; i < 64; ++i) xr[i] = 0u;
    }
    if (ct == 0) {
      asm volatile("" ::"f"(Xs));  // order the timestamp after x has landed
      DECDEC_TRACE(p, 2);
    }
    const int nkw = small_g ? 1 : p.NKW;
    const int team = cw / nkw, wi = cw % nkw;
    int nrows_tile = 0;  // o_b rows this warp writes per tile (same for every tile)
    const int stages = p.stages, RPS = p.RPS, NSLOTS = p.NSLOTS, TR = p.TR, row_bytes = p.row_bytes;
    const int rows_per_warp_tile = small_g ? RPS * (32 / G) : RPS;  // o_b rows one warp (team) writes
    int it = 0, st = 0;
    uint32_t ph = 0;
    for (int tile = cta; tile < p.n_tiles; tile += n_cta, ++it) {
      mbar_wait(&full[st], ph);
      if (it == 0 && ct == 0) DECDEC_TRACE(p, 3);
      const uint8_t* sw = stage0 + (size_t)st * p.stage_bytes;
      const uint16_t* ss = reinterpret_cast<const uint16_t*>(sw + p.off_s);
      const uint8_t* sz = sw + p.off_z;
      float part[4] = {0.f, 0.f, 0.f, 0.f};  // RPS <= 4
#ifdef DECDEC_SKIP_COMPUTE  // experiment: stream the tiles without computing (memory-bound floor)
      if (active) part[0] = __half2float(__ushort_as_half(ss[slot * G + g]));
#else
#if DECDEC_ROW_STEP == 1
      // one row per step, rolled over the tile's RPS rows: the loop body (~3.5 KB of SASS for
      // 3-bit) stays inside the ~6 KB L0 instruction cache with the tile bookkeeping
#pragma unroll 1
      for (int m = 0; m < RPS; ++m) {
        const int r0 = slot + m * NSLOTS;
        if (active) {
          const uint8_t* g0 = sw + r0 * row_bytes + g * GB;
          float a0[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          if (LUTB) {
            const float v = row_group_dot_lut<LUTB ? LUTB : 3>(
                g0, reinterpret_cast<const uint32_t*>(sw + p.off_s + (size_t)r0 * (2 << LUTB)), xr, rot);
            part[0] = m == 0 ? v : part[0];
            part[1] = m == 1 ? v : part[1];
            part[2] = m == 2 ? v : part[2];
            part[3] = m == 3 ? v : part[3];
            continue;
          }
          if (BITS == 4) {
            uint4 v0[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) v0[j] = *reinterpret_cast<const uint4*>(g0 + 16 * ((j + rot) & 3));
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              fma_w4_word(v0[j].x, xr + 16 * j + 0, a0);
              fma_w4_word(v0[j].y, xr + 16 * j + 4, a0);
              fma_w4_word(v0[j].z, xr + 16 * j + 8, a0);
              fma_w4_word(v0[j].w, xr + 16 * j + 12, a0);
            }
          } else {
            uint32_t w0[12];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              const uint4 t0 = *reinterpret_cast<const uint4*>(g0 + 16 * j);
              w0[4 * j] = t0.x; w0[4 * j + 1] = t0.y; w0[4 * j + 2] = t0.z; w0[4 * j + 3] = t0.w;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) fma_w3_slice(w0[3 * u], w0[3 * u + 1], w0[3 * u + 2], xr + 16 * u, a0);
          }
          const float t0 = combine_classes<BITS>(a0);
          const float s0 = __half2float(__ushort_as_half(ss[r0 * G + g])) * 16777216.f;  // s * 2^24
          const float z0 = (float)sz[r0 * G + g];
          const float v = s0 * fmaf(-z0, Xs, t0);  // s * sum_(i in g) (q_i - z) x_i
          part[0] = m == 0 ? v : part[0];
          part[1] = m == 1 ? v : part[1];
          part[2] = m == 2 ? v : part[2];
          part[3] = m == 3 ? v : part[3];
        }
      }
#else
#pragma unroll
      for (int m = 0; m < kMaxRPS; m += 2) {
        if (m >= RPS) break;
        const bool two = m + 1 < RPS;
        const int r0 = slot + m * NSLOTS, r1 = slot + (m + 1) * NSLOTS;
        if (active) {
          const uint8_t* g0 = sw + r0 * row_bytes + g * GB;
          const uint8_t* g1 = sw + (two ? r1 : r0) * row_bytes + g * GB;
          float a0[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, a1[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          if (LUTB) {  // non-uniform base: sum_i lut[q_i] x_i per row, no scale / zero
            const uint8_t* tb = sw + p.off_s;
            part[m] = row_group_dot_lut<LUTB ? LUTB : 3>(g0, reinterpret_cast<const uint32_t*>(tb + (size_t)r0 * (2 << LUTB)),
                                                         xr, rot);
            if (two)
              part[m + 1] = row_group_dot_lut<LUTB ? LUTB : 3>(
                  g1, reinterpret_cast<const uint32_t*>(tb + (size_t)r1 * (2 << LUTB)), xr, rot);
            continue;
          }
          if (BITS == 4) {
            uint4 v0[4], v1[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              v0[j] = *reinterpret_cast<const uint4*>(g0 + 16 * ((j + rot) & 3));
              v1[j] = *reinterpret_cast<const uint4*>(g1 + 16 * ((j + rot) & 3));
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              fma_w4_word(v0[j].x, xr + 16 * j + 0, a0);
              fma_w4_word(v1[j].x, xr + 16 * j + 0, a1);
              fma_w4_word(v0[j].y, xr + 16 * j + 4, a0);
              fma_w4_word(v1[j].y, xr + 16 * j + 4, a1);
              fma_w4_word(v0[j].z, xr + 16 * j + 8, a0);
              fma_w4_word(v1[j].z, xr + 16 * j + 8, a1);
              fma_w4_word(v0[j].w, xr + 16 * j + 12, a0);
              fma_w4_word(v1[j].w, xr + 16 * j + 12, a1);
            }
          } else {
            uint32_t w0[12], w1[12];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              const uint4 t0 = *reinterpret_cast<const uint4*>(g0 + 16 * j);
              const uint4 t1 = *reinterpret_cast<const uint4*>(g1 + 16 * j);
              w0[4 * j] = t0.x; w0[4 * j + 1] = t0.y; w0[4 * j + 2] = t0.z; w0[4 * j + 3] = t0.w;
              w1[4 * j] = t1.x; w1[4 * j + 1] = t1.y; w1[4 * j + 2] = t1.z; w1[4 * j + 3] = t1.w;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              fma_w3_slice(w0[3 * u], w0[3 * u + 1], w0[3 * u + 2], xr + 16 * u, a0);
              fma_w3_slice(w1[3 * u], w1[3 * u + 1], w1[3 * u + 2], xr + 16 * u, a1);
            }
          }
          const float t0 = combine_classes<BITS>(a0);
          const float t1 = combine_classes<BITS>(a1);
          const float s0 = __half2float(__ushort_as_half(ss[r0 * G + g])) * 16777216.f;  // s * 2^24
          const float z0 = (float)sz[r0 * G + g];
          part[m] = s0 * fmaf(-z0, Xs, t0);  // s * sum_(i in g) (q_i - z) x_i
          if (two) {
            const float s1 = __half2float(__ushort_as_half(ss[r1 * G + g])) * 16777216.f;
            const float z1 = (float)sz[r1 * G + g];
            part[m + 1] = s1 * fmaf(-z1, Xs, t1);
          }
        }
      }
#endif  // DECDEC_ROW_STEP
#endif  // DECDEC_SKIP_COMPUTE
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done reading the stage
      int nrows = 0;
      if (small_g) {
        // rows are whole inside the warp: butterfly over the G lanes of each row (fixed order)
        if (G == 32 && RPS == 4) {
          // transposed butterfly: 4 rows in 6 shuffles / 5 dependent rounds (fixed order)
          const bool hi16 = lane & 16, hi8 = lane & 8;
          float u0 = (hi16 ? part[2] : part[0]) + __shfl_xor_sync(0xffffffffu, hi16 ? part[0] : part[2], 16);
          float u1 = (hi16 ? part[3] : part[1]) + __shfl_xor_sync(0xffffffffu, hi16 ? part[1] : part[3], 16);
          float v = (hi8 ? u1 : u0) + __shfl_xor_sync(0xffffffffu, hi8 ? u0 : u1, 8);
#pragma unroll
          for (int o = 4; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if ((lane & 7) == 0) {  // lane 0 -> row 0, 8 -> 1, 16 -> 2, 24 -> 3
            const int m = (hi16 ? 2 : 0) + (hi8 ? 1 : 0);
            const int row = tile * TR + slot + m * NSLOTS;
            if (p.k_sel == 0) p2p_store_u16(p.pp, p.y, row, __half_as_ushort(__float2half_rn(v)));
            else st_relaxed_gpu_f32(p.ob + row, v);
          }
        } else if (G == 32 && RPS == 2) {
          const bool hi16 = lane & 16;
          float v = (hi16 ? part[1] : part[0]) + __shfl_xor_sync(0xffffffffu, hi16 ? part[0] : part[1], 16);
#pragma unroll
          for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if ((lane & 15) == 0) {
            const int row = tile * TR + slot + (hi16 ? 1 : 0) * NSLOTS;
            if (p.k_sel == 0) p2p_store_u16(p.pp, p.y, row, __half_as_ushort(__float2half_rn(v)));
            else st_relaxed_gpu_f32(p.ob + row, v);
          }
        } else {
#pragma unroll
          for (int m = 0; m < kMaxRPS; ++m) {
            if (m >= RPS) break;
            float v = part[m];
            for (int o = G >> 1; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (g == 0) {
              const int row = tile * TR + slot + m * NSLOTS;
              if (p.k_sel == 0) p2p_store_u16(p.pp, p.y, row, __half_as_ushort(__float2half_rn(v)));
              else st_relaxed_gpu_f32(p.ob + row, v);
            }
          }
        }
        nrows = rows_per_warp_tile;
      } else {
        // NKW warps per row: warp butterfly, then the team's first warp sums the NKW partials
        float* rbuf = red + ((it & 1) * NSLOTS + team) * 4 * p.NKW;
#pragma unroll
        for (int m = 0; m < kMaxRPS; ++m) {
          if (m >= RPS) break;
          float v = part[m];
#pragma unroll
          for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0) rbuf[m * p.NKW + wi] = v;
        }
        named_bar_sync(1 + team, p.NKW * 32);
        if (wi == 0) {
          if (lane < RPS) {
            float v = 0.f;
            for (int w = 0; w < p.NKW; ++w) v += rbuf[lane * p.NKW + w];
            const int row = tile * TR + slot + lane * NSLOTS;
            if (p.k_sel == 0) p2p_store_u16(p.pp, p.y, row, __half_as_ushort(__float2half_rn(v)));
            else st_relaxed_gpu_f32(p.ob + row, v);
          }
          nrows = RPS;
        }
      }
      nrows_tile = nrows;
      if (++st == stages) {
        st = 0;
        ph ^= 1;
      }
    }
    if (ct == 0) DECDEC_TRACE(p, 4);
    if (ct == 0) DECDEC_TRACE(p, 10);  // last o_b row stored (this warp)
    if (p.k_sel == 0 && p.pp.active) {  // fused all-gather (k = 0: the GEMV CTAs write y)
      named_bar_sync(15, p.NC * 32);
      if (ct == 0) {
        p2p_signal(p.pp);
      }
    }
    return;
  }
}

// Debug: decode packed weights with the kernel's own decode path; q_out u8 [d_out][d_in].
template <int BITS>
__global__ void k_debug_unpack(const uint8_t* __restrict__ w, int d_in, int d_out, uint8_t* __restrict__ q_out) {
  const int slices = d_in / 32;
  const long long total = (long long)d_out * slices;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t / slices), u = (int)(t % slices);
    const uint8_t* rowp = w + (size_t)j * (d_in * BITS / 8);
    uint8_t* out = q_out + (size_t)j * d_in + u * 32;
    if (BITS == 4) {
      const uint32_t* wp = reinterpret_cast<const uint32_t*>(rowp) + u * 4;
      for (int wd = 0; wd < 4; ++wd) {
        uint32_t m[4];
        decode_w4_word(wp[wd], m);
        for (int q = 0; q < 4; ++q) {
          const float sc = w4_class(q) ? 1.f / 16.f : 1.f;
          const float lo = __half2float(__ushort_as_half((unsigned short)(m[q] & 0xffffu))) * 16777216.f * sc;
          const float hi = __half2float(__ushort_as_half((unsigned short)(m[q] >> 16))) * 16777216.f * sc;
          out[wd * 8 + 2 * q] = (uint8_t)lo;
          out[wd * 8 + 2 * q + 1] = (uint8_t)hi;
        }
      }
    } else {
      const uint32_t* wp = reinterpret_cast<const uint32_t*>(rowp) + u * 3;
      uint32_t m[16];
      decode_w3_slice(wp[0], wp[1], wp[2], m);
      for (int k = 0; k < 16; ++k) {
        const int cls = w3_class(k);
        const float sc = cls == 0 ? 1.f : (cls == 1 ? 0.125f : 0.015625f);
        const float lo = __half2float(__ushort_as_half((unsigned short)(m[k] & 0xffffu))) * 16777216.f * sc;
        const float hi = __half2float(__ushort_as_half((unsigned short)(m[k] >> 16))) * 16777216.f * sc;
        out[2 * k] = (uint8_t)lo;
        out[2 * k + 1] = (uint8_t)hi;
      }
    }
  }
}

}  // namespace decdec
