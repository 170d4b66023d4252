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
#include "select.cuh"

namespace decdec {

constexpr int kRB = 8;            // residual rows per gather work item (in flight per lane)
constexpr int kSegCols = 256;     // output columns per combine segment (128 B of 4-bit codes)
constexpr int kMaxThreads = 480;  // 1 producer + <= 12 consumer + 2 gather warps
constexpr int kMaxRPS = 4;       // rows per slot per tile
constexpr int kCntSlots = 4096;   // arrival counters at the head of the workspace
constexpr int kCtrlSlots = 16;    // last slots of that region: control words (sel_ready, cta_done)
// trace events (per CTA): 0 start, 1 first TMA issued, 2 x loaded, 3 first stage landed,
// 4 GEMV done, 5 selector start, 6 selection published, 7 gather done, 8 consumers released (PDL)
constexpr int kTraceEvents = 9;
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
  const int* idx;
  const uint16_t* xs;
  const uint8_t* r_rows;
  const uint16_t* r_scales;
  int r_row_bytes;
  float* ob;
  float* part;
  uint16_t* sdev;
  uint32_t* cnt;
  int n_seg, n_rb, gws, NGW;  // gws = gather warps per segment (each takes row blocks j, j+gws, ...)
  uint32_t off_sel;            // smem offset of the staged selection (idx int32[k], xs u16[k])
  uint32_t off_x;              // smem offset of the staged x (d_in fp16, 16-B units swizzled)
  unsigned long long* trace;   // optional per-CTA event timestamps [grid][kTraceEvents] (ns), or null
  // step (1) runs on the first sel_ctas CTAs (one per selection segment: the whole x, or one
  // chunk); each bumps *sel_ready when its indices are written; gather warps wait for
  // *sel_ready == sel_ctas.  The last CTA to exit resets *sel_ready and *cta_done.
  int sel_ctas, k_req, chunk;
  int prefetch;  // weight tiles requested per CTA before griddepcontrol.wait
  int* sel_out;
  uint32_t* sel_ready;
  uint32_t* cta_done;
};

template <int RBITS>
__device__ __forceinline__ void combine_segment(const LinearParams& p, int seg, int lane) {
  const int col0 = seg * kSegCols + lane * 8;
  if (col0 >= p.d_out) return;
  const float4 o0 = ld_cg_f4(p.ob + col0), o1 = ld_cg_f4(p.ob + col0 + 4);
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int j = 0; j < p.gws; ++j) {  // fixed order: gather warps of the segment ascending
    const float* pp = p.part + (size_t)j * p.d_out + col0;
    const float4 a = ld_cg_f4(pp), b = ld_cg_f4(pp + 4);
    s[0] += a.x; s[1] += a.y; s[2] += a.z; s[3] += a.w;
    s[4] += b.x; s[5] += b.y; s[6] += b.z; s[7] += b.w;
  }
  float S[8] = {1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f, 1.f};
  if (RBITS == 4) {
    const uint4 sv = ld_cg_u4(p.sdev + col0);
    const uint32_t sw[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      S[2 * e] = __half2float(__ushort_as_half((unsigned short)(sw[e] & 0xffffu)));
      S[2 * e + 1] = __half2float(__ushort_as_half((unsigned short)(sw[e] >> 16)));
    }
  }
  const float o[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
  uint32_t out[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const __half lo = __float2half_rn(fmaf(S[2 * e], s[2 * e], o[2 * e]));
    const __half hi = __float2half_rn(fmaf(S[2 * e + 1], s[2 * e + 1], o[2 * e + 1]));
    out[e] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
  }
  *reinterpret_cast<uint4*>(p.y + col0) = make_uint4(out[0], out[1], out[2], out[3]);
}

// GEMV side: publish `rows` o_b rows of segment `seg` (caller fenced its stores).
__device__ __forceinline__ void gemv_publish(const LinearParams& p, int seg, uint32_t rows, int lane) {
  __syncwarp();
  if (lane == 0) atomicAdd(p.cnt + seg, rows);
}

// Gather side: publish one partial of segment `seg` (caller fenced).  The last of the
// segment's gws gather warps waits for the segment's o_b rows, combines, and resets both
// counters for the next call.  Combines are thus spread over the gather warps (one per
// segment) and never run on the GEMV warps.
template <int RBITS>
__device__ __forceinline__ void gather_publish(const LinearParams& p, int seg, int lane) {
  __syncwarp();
  uint32_t old = 0;
  if (lane == 0) old = atomicAdd(p.cnt + p.n_seg + seg, 1u);
  old = __shfl_sync(0xffffffffu, old, 0);
  if (old + 1 != (uint32_t)p.gws) return;
  const uint32_t seg_cols = (uint32_t)min(kSegCols, p.d_out - seg * kSegCols);
  if (lane == 0) {
    while (ld_acquire_gpu(p.cnt + seg) != seg_cols) __nanosleep(32);
  }
  __syncwarp();
  __threadfence();
  combine_segment<RBITS>(p, seg, lane);
  if (lane == 0) {
    p.cnt[seg] = 0;  // ready for the next call
    p.cnt[p.n_seg + seg] = 0;
  }
}

// Called by every warp when it is done (all lanes).  With compensation (k_sel > 0) the last
// warp of the last CTA resets the PDL-chain control words for the next layer.
__device__ __forceinline__ void warp_exit(const LinearParams& p, uint32_t* warps_done, int lane) {
  if (p.k_sel <= 0) return;
  __syncwarp();
  if (lane == 0) {
    if (atomicAdd(warps_done, 1u) == (blockDim.x >> 5) - 1) {       // last warp of this CTA
      if (atomicAdd(p.cta_done, 1u) == gridDim.x - 1) {               // last CTA of the grid
        *p.cta_done = 0u;
        *p.sel_ready = 0u;
      }
    }
  }
}

template <int BITS, int RBITS>
__global__ void __launch_bounds__(kMaxThreads, 1) k_linear(const LinearParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stage0 = smem;
  float* red = reinterpret_cast<float*>(smem + (size_t)p.stages * p.stage_bytes);  // [2][NSLOTS][4][NKW]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 2 * p.NSLOTS * 4 * max(p.NKW, 1));
  uint64_t* empty = full + p.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ uint32_t warps_done;
  // Let the next kernel of the stream launch now: its CTAs take SMs as ours retire and start
  // streaming their (static) weights while we finish (cross-layer overlap).
  pdl_launch_dependents();

  if (threadIdx.x == 0) {
    warps_done = 0;
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], p.NC);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) DECDEC_TRACE(p, 0);

  // ------------------------------------------------------------------ selector CTAs (step 1)
  if ((int)blockIdx.x < p.sel_ctas) {
    pdl_wait();  // x may be the previous layer's product
    if (threadIdx.x == 0) DECDEC_TRACE(p, 5);
    const int seg = blockIdx.x;
    const int a = p.chunk ? seg * p.chunk : 0;
    const int n = p.chunk ? min(p.chunk, p.d_in - a) : p.d_in;
    const int q = p.chunk ? min(p.k_req, n) : p.k_req;
    const int off = p.chunk ? seg * p.k_req : 0;
    select_block(p.x + a, n, q, a, const_cast<int*>(p.idx) + off, const_cast<uint16_t*>(p.xs) + off,
                 p.sel_out ? p.sel_out + off : nullptr, reinterpret_cast<SelectSmem*>(smem),
                 reinterpret_cast<uint4*>(smem + sizeof(SelectSmem)));
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(p.sel_ready, 1u);
      DECDEC_TRACE(p, 6);
    }
    warp_exit(p, &warps_done, lane);
    return;
  }
  const int cta = blockIdx.x - p.sel_ctas, n_cta = gridDim.x - p.sel_ctas;  // GEMV CTA index / count

  // ------------------------------------------------------------------ producer (TMA)
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const uint32_t wb = (uint32_t)p.TR * p.row_bytes, sb = (uint32_t)p.TR * p.G * 2, zb = (uint32_t)p.TR * p.G;
      const int stages = p.stages;
      int it = 0, st = 0;
      uint32_t ph = 0;  // phase of the current pass over the ring
      for (int tile = cta; tile < p.n_tiles; tile += n_cta, ++it) {
        // only `prefetch` tiles may be requested before the previous layer completes: a deeper
        // early burst floods the memory pipe and delays the x loads the consumers wait on
        if (it == p.prefetch) pdl_wait();
        if (it >= stages) mbar_wait(&empty[st], ph ^ 1);
        uint8_t* dst = stage0 + (size_t)st * p.stage_bytes;
        mbar_arrive_expect_tx(&full[st], wb + sb + zb);
        bulk_g2s(dst, p.w + (size_t)tile * wb, wb, &full[st], pol);
        bulk_g2s(dst + p.off_s, p.ws + (size_t)tile * p.TR * p.G, sb, &full[st], pol);
        bulk_g2s(dst + p.off_z, p.wz + (size_t)tile * p.TR * p.G, zb, &full[st], pol);
        if (it == 0) DECDEC_TRACE(p, 1);
        if (++st == stages) {
          st = 0;
          ph ^= 1;
        }
      }
    }
    warp_exit(p, &warps_done, lane);
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
#pragma unroll
      for (int m = 0; m < kMaxRPS; m += 2) {
        if (m >= RPS) break;
        const bool two = m + 1 < RPS;
        const int r0 = slot + m * NSLOTS, r1 = slot + (m + 1) * NSLOTS;
        if (active) {
          const uint8_t* g0 = sw + r0 * row_bytes + g * GB;
          const uint8_t* g1 = sw + (two ? r1 : r0) * row_bytes + g * GB;
          float a0[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, a1[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
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
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done reading the stage
      int nrows = 0;
      if (small_g) {
        // rows are whole inside the warp: butterfly over the G lanes of each row (fixed order)
#pragma unroll
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
            if (p.k_sel == 0) p.y[row] = __half_as_ushort(__float2half_rn(v));
            else p.ob[row] = v;
          }
        } else if (G == 32 && RPS == 2) {
          const bool hi16 = lane & 16;
          float v = (hi16 ? part[1] : part[0]) + __shfl_xor_sync(0xffffffffu, hi16 ? part[0] : part[1], 16);
#pragma unroll
          for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if ((lane & 15) == 0) {
            const int row = tile * TR + slot + (hi16 ? 1 : 0) * NSLOTS;
            if (p.k_sel == 0) p.y[row] = __half_as_ushort(__float2half_rn(v));
            else p.ob[row] = v;
          }
        } else {
#pragma unroll
          for (int m = 0; m < kMaxRPS; ++m) {
            if (m >= RPS) break;
            float v = part[m];
            for (int o = G >> 1; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (g == 0) {
              const int row = tile * TR + slot + m * NSLOTS;
              if (p.k_sel == 0) p.y[row] = __half_as_ushort(__float2half_rn(v));
              else p.ob[row] = v;
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
            if (p.k_sel == 0) p.y[row] = __half_as_ushort(__float2half_rn(v));
            else p.ob[row] = v;
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
    // Publish o_b rows once per warp (one fence for all tiles, then one arrival per tile):
    // a fence per tile stalled the GEMV stream by ~1 µs each.
    if (p.k_sel > 0 && nrows_tile > 0) {
      __threadfence();
      for (int tile = cta; tile < p.n_tiles; tile += n_cta)
        gemv_publish(p, (tile * TR) / kSegCols, (uint32_t)nrows_tile, lane);
    }
    warp_exit(p, &warps_done, lane);
    return;
  }

  // ------------------------------------------------------------------ gather warps (DEC)
  if (p.k_sel <= 0) return;  // (no gather warps are launched without compensation)
  const int gwi = warp - 1 - p.NC;
  int* sidx = reinterpret_cast<int*>(smem + p.off_sel);
  uint16_t* sxs = reinterpret_cast<uint16_t*>(sidx + p.k_sel);
  pdl_wait();  // the workspace belongs to the previous layer until it completes
  if (lane == 0) {
    while (ld_acquire_gpu(p.sel_ready) < (uint32_t)p.sel_ctas) __nanosleep(20);
  }
  __syncwarp();
  for (int i = gwi * 32 + lane; i < p.k_sel; i += p.NGW * 32) {
    sidx[i] = __ldcg(p.idx + i);
    sxs[i] = __ldcg(p.xs + i);
  }
  named_bar_sync(15, p.NGW * 32);
  if (gwi == 0 && lane == 0) DECDEC_TRACE(p, 6);
  const int gw = gwi + p.NGW * cta, ngw = p.NGW * n_cta;
  for (int pair = gw; pair < p.n_seg * p.gws; pair += ngw) {
    const int seg = pair % p.n_seg, j = pair / p.n_seg;
    const int col0 = seg * kSegCols + lane * 8;
    const bool cv = col0 < p.d_out;
    if (RBITS == 4 && j == 0 && cv) {  // all scale factors are fetched every call
      const uint4 sv = ld_zc_u4(p.r_scales + col0);
      *reinterpret_cast<uint4*>(p.sdev + col0) = sv;
    }
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    // row blocks rb = j, j + gws, ... (8 rows each), double-buffered: next block's zero-copy
    // loads are in flight while the current block is decoded.
    using Vec = typename std::conditional<RBITS == 4, uint32_t, uint4>::type;
    auto load = [&](int rb, Vec* buf) {
#pragma unroll
      for (int r = 0; r < kRB; ++r) {
        const int e = rb * kRB + r;
        if (e < p.k_sel && cv) {
          const uint8_t* rowp = p.r_rows + (size_t)sidx[e] * p.r_row_bytes;
          if constexpr (RBITS == 4) buf[r] = ld_zc_u32(rowp + (col0 >> 1));
          else buf[r] = ld_zc_u4(rowp + col0 * 2);
        } else {
          if constexpr (RBITS == 4) buf[r] = 0u;
          else buf[r] = make_uint4(0, 0, 0, 0);
        }
      }
    };
    auto consume = [&](int rb, const Vec* buf) {
#pragma unroll
      for (int r = 0; r < kRB; ++r) {
        const int e = rb * kRB + r;
        if (e < p.k_sel) {
          const uint16_t xv = sxs[e];
          uint32_t c[4];
          if constexpr (RBITS == 4) {
            decode_rq_word(buf[r], c);
          } else {
            c[0] = buf[r].x; c[1] = buf[r].y; c[2] = buf[r].z; c[3] = buf[r].w;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[2 * q] = fhfma_s_lo(xv, c[q], acc[2 * q]);
            acc[2 * q + 1] = fhfma_s_hi(xv, c[q], acc[2 * q + 1]);
          }
        }
      }
    };
    Vec bufA[kRB], bufB[kRB];
    int rb = j;
    load(rb, bufA);
    while (true) {
      if (rb + p.gws < p.n_rb) load(rb + p.gws, bufB);
      consume(rb, bufA);
      rb += p.gws;
      if (rb >= p.n_rb) break;
      if (rb + p.gws < p.n_rb) load(rb + p.gws, bufA);
      consume(rb, bufB);
      rb += p.gws;
      if (rb >= p.n_rb) break;
    }
    if (cv) {
      float* pp = p.part + (size_t)j * p.d_out + col0;
      *reinterpret_cast<float4*>(pp) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      *reinterpret_cast<float4*>(pp + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
  }
  if (gwi == 0 && lane == 0) DECDEC_TRACE(p, 7);
  __threadfence();  // one fence for all of this warp's partials, then the arrivals
  for (int pair = gw; pair < p.n_seg * p.gws; pair += ngw) gather_publish<RBITS>(p, pair % p.n_seg, lane);
  warp_exit(p, &warps_done, lane);
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
