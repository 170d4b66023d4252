// Fused DecDEC layer kernel for sm_100a: base GEMV (HBM stream) + dynamic error
// compensation (PCIe zero-copy gather) + deterministic combine, in ONE persistent launch.
//
// PAPER.md P:207 runs steps 2-4 "in parallel with the base GEMV on a different GPU stream";
// here they run in parallel inside one kernel by warp specialisation:
//   warp 0              producer: 1-D bulk async copies (TMA engine, cp.async.bulk) of
//                       TR packed rows + their scales/zeros into a `stages`-deep smem ring
//                       (mbarrier full/empty pairs), L2 evict-first.
//   warps 1..NC         consumers: thread (g, rp) owns input group g (128 channels, x kept
//                       in 64 registers for the whole launch) and row phase rp; decodes
//                       codes in registers (decode.cuh), FHFMA fp32 accumulation, applies
//                       the group's z and s, writes a partial per (row, group) to smem; one
//                       named barrier per tile, then a fixed-order warp reduction per row.
//   warps NC+1..NC+NGW  gather warps (only when k > 0): wait for the selector kernel
//                       (programmatic dependent launch), then stream residual rows
//                       R_hat[S, 256-column segment] from pinned host memory with zero-copy
//                       loads, RB rows in flight per warp, decode + FHFMA, write a
//                       per-row-block partial.  Work item = (segment, row block).
// Combine (P:207 step 4; the paper uses atomics): every producer of a 256-column
// segment (GEMV rows, gather row blocks) publishes with a fence and bumps the segment's
// arrival counter; the last arriver sums  y = fp16(o_b + S_j * sum_rb part_rb)  in a fixed
// order and resets the counter.  No value atomics -> bit-reproducible.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include "ptx.cuh"
#include "decode.cuh"

namespace decdec {

constexpr int kRB = 8;            // residual rows per gather work item (in flight per lane)
constexpr int kSegCols = 256;     // output columns per combine segment (128 B of 4-bit codes)
constexpr int kMaxThreads = 480;  // 1 producer + <= 12 consumer + 2 gather warps
constexpr int kCntSlots = 4096;   // arrival counters at the head of the workspace

struct LinearParams {
  const uint8_t* w;      // packed weights (W3K/W4K), [d_out][row_bytes]
  const uint16_t* ws;    // fp16 scales [d_out][G]
  const uint8_t* wz;     // u8 zeros [d_out][G]
  const uint16_t* x;     // fp16 [d_in]
  uint16_t* y;           // fp16 [d_out]
  int d_in, d_out, G, row_bytes;
  int TR, RP, RPT, NC, stages, n_tiles;
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
  int n_seg, n_rb, n_items, NGW;
};

template <int RBITS>
__device__ __forceinline__ void combine_segment(const LinearParams& p, int seg, int lane) {
  const int col0 = seg * kSegCols + lane * 8;
  if (col0 >= p.d_out) return;
  const float4 o0 = ld_cg_f4(p.ob + col0), o1 = ld_cg_f4(p.ob + col0 + 4);
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int rb = 0; rb < p.n_rb; ++rb) {  // fixed order: row blocks ascending
    const float* pp = p.part + (size_t)rb * p.d_out + col0;
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

// Publish `add` arrivals for segment `seg`; the warp whose arrival completes the segment
// combines it.  Caller: all lanes have stored their data and executed __threadfence().
template <int RBITS>
__device__ __forceinline__ void arrive_segment(const LinearParams& p, int seg, uint32_t add, int lane) {
  __syncwarp();
  uint32_t old = 0;
  if (lane == 0) old = atomicAdd(p.cnt + seg, add);
  old = __shfl_sync(0xffffffffu, old, 0);
  const int seg_cols = min(kSegCols, p.d_out - seg * kSegCols);
  if (old + add == (uint32_t)(seg_cols + p.n_rb)) {
    __threadfence();
    combine_segment<RBITS>(p, seg, lane);
    if (lane == 0) p.cnt[seg] = 0;  // ready for the next call
  }
}

template <int BITS, int RBITS>
__global__ void __launch_bounds__(kMaxThreads, 1) k_linear(const LinearParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stage0 = smem;
  float* red = reinterpret_cast<float*>(smem + (size_t)p.stages * p.stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 2 * p.TR * p.G);
  uint64_t* empty = full + p.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

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
      const uint32_t wb = (uint32_t)p.TR * p.row_bytes, sb = (uint32_t)p.TR * p.G * 2, zb = (uint32_t)p.TR * p.G;
      int it = 0;
      for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
        const int st = it % p.stages;
        if (it >= p.stages) mbar_wait(&empty[st], ((it / p.stages) & 1) ^ 1);
        uint8_t* dst = stage0 + (size_t)st * p.stage_bytes;
        mbar_arrive_expect_tx(&full[st], wb + sb + zb);
        bulk_g2s(dst, p.w + (size_t)tile * wb, wb, &full[st], pol);
        bulk_g2s(dst + p.off_s, p.ws + (size_t)tile * p.TR * p.G, sb, &full[st], pol);
        bulk_g2s(dst + p.off_z, p.wz + (size_t)tile * p.TR * p.G, zb, &full[st], pol);
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers (GEMV)
  if (warp <= p.NC) {
    constexpr int GB = 16 * BITS;  // bytes of one 128-code group
    const int ct = threadIdx.x - 32;
    const int G = p.G;
    const int g = ct % G, rp = ct / G;
    const bool active = rp < p.RP;
    const int rot = (BITS == 4) ? ((g >> 1) & 3) : 0;  // 4-bit: bank-conflict-free 16-B chunk order
    uint32_t xr[64];
    float Xs = 0.f;
    if (active) {
      const uint4* xp = reinterpret_cast<const uint4*>(p.x + (size_t)g * 128);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = (j + rot) & 3;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint4 v = __ldg(xp + 4 * c + e);
          xr[16 * j + 4 * e + 0] = v.x;
          xr[16 * j + 4 * e + 1] = v.y;
          xr[16 * j + 4 * e + 2] = v.z;
          xr[16 * j + 4 * e + 3] = v.w;
        }
      }
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        Xs += __half2float(__ushort_as_half((unsigned short)(xr[i] & 0xffffu)));
        Xs += __half2float(__ushort_as_half((unsigned short)(xr[i] >> 16)));
      }
      Xs *= 5.9604644775390625e-08f;  // 2^-24: same scale as the decoded codes
    }
    const int cw = warp - 1;
    int it = 0;
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
      const int st = it % p.stages;
      mbar_wait(&full[st], (it / p.stages) & 1);
      const uint8_t* sw = stage0 + (size_t)st * p.stage_bytes;
      const uint16_t* ss = reinterpret_cast<const uint16_t*>(sw + p.off_s);
      const uint8_t* sz = sw + p.off_z;
      float* rbuf = red + (it & 1) * p.TR * G;
      if (active) {
        for (int m = 0; m < p.RPT; ++m) {
          const int r = rp + m * p.RP;
          const uint8_t* gp = sw + (size_t)r * p.row_bytes + g * GB;
          float acc[3] = {0.f, 0.f, 0.f};
          if (BITS == 4) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint4 v = *reinterpret_cast<const uint4*>(gp + 16 * ((j + rot) & 3));
              fma_w4_word(v.x, xr + 16 * j + 0, acc);
              fma_w4_word(v.y, xr + 16 * j + 4, acc);
              fma_w4_word(v.z, xr + 16 * j + 8, acc);
              fma_w4_word(v.w, xr + 16 * j + 12, acc);
            }
          } else {
            const uint4 v0 = *reinterpret_cast<const uint4*>(gp);
            const uint4 v1 = *reinterpret_cast<const uint4*>(gp + 16);
            const uint4 v2 = *reinterpret_cast<const uint4*>(gp + 32);
            const uint32_t wv[12] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w, v2.x, v2.y, v2.z, v2.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) fma_w3_slice(wv[3 * u], wv[3 * u + 1], wv[3 * u + 2], xr + 16 * u, acc);
          }
          const float sc = __half2float(__ushort_as_half(ss[r * G + g])) * 16777216.f;  // s * 2^24
          const float zf = (float)sz[r * G + g];
          const float t = (BITS == 4) ? fmaf(acc[1], 0.0625f, acc[0])
                                      : fmaf(acc[2], 0.015625f, fmaf(acc[1], 0.125f, acc[0]));
          rbuf[r * G + g] = sc * fmaf(-zf, Xs, t);  // s * sum_(i in g) (q_i - z) x_i
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);  // stage fully read into registers
      named_bar_sync(1, p.NC * 32);
      int nrows = 0;
      for (int r = cw; r < p.TR; r += p.NC) {
        float s = 0.f;
        for (int gg = lane; gg < G; gg += 32) s += rbuf[r * G + gg];
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const int row = tile * p.TR + r;
        if (lane == 0) {
          if (p.k_sel == 0) p.y[row] = __half_as_ushort(__float2half_rn(s));
          else p.ob[row] = s;
        }
        ++nrows;
      }
      if (p.k_sel > 0 && nrows > 0) {
        __threadfence();
        arrive_segment<RBITS>(p, (tile * p.TR) / kSegCols, (uint32_t)nrows, lane);
      }
    }
    return;
  }

  // ------------------------------------------------------------------ gather warps (DEC)
  if (p.k_sel <= 0) return;
  pdl_wait();  // selector kernel complete and its writes visible
  const int gw = (warp - 1 - p.NC) + p.NGW * blockIdx.x, ngw = p.NGW * gridDim.x;
  for (int item = gw; item < p.n_items; item += ngw) {
    const int seg = item % p.n_seg, rbk = item / p.n_seg;
    const int r0 = rbk * kRB, nr = min(kRB, p.k_sel - r0);
    const int col0 = seg * kSegCols + lane * 8;
    const bool cv = col0 < p.d_out;
    int myrow = 0;
    uint32_t myxs = 0;
    if (lane < nr) {
      myrow = __ldcg(p.idx + r0 + lane);
      myxs = __ldcg(p.xs + r0 + lane);
    }
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (RBITS == 4) {
      uint32_t wv[kRB];
#pragma unroll
      for (int r = 0; r < kRB; ++r) {
        const int row = __shfl_sync(0xffffffffu, myrow, r);
        wv[r] = (r < nr && cv) ? ld_zc_u32(p.r_rows + (size_t)row * p.r_row_bytes + (col0 >> 1)) : 0u;
      }
      if (rbk == 0 && cv) {  // all scale factors are fetched every call
        const uint4 sv = ld_zc_u4(p.r_scales + col0);
        *reinterpret_cast<uint4*>(p.sdev + col0) = sv;
      }
#pragma unroll
      for (int r = 0; r < kRB; ++r) {
        const uint16_t xv = (uint16_t)__shfl_sync(0xffffffffu, myxs, r);
        if (r < nr) {
          uint32_t c[4];
          decode_rq_word(wv[r], c);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[2 * q] = fhfma_s_lo(xv, c[q], acc[2 * q]);
            acc[2 * q + 1] = fhfma_s_hi(xv, c[q], acc[2 * q + 1]);
          }
        }
      }
    } else {
      uint4 wv[kRB];
#pragma unroll
      for (int r = 0; r < kRB; ++r) {
        const int row = __shfl_sync(0xffffffffu, myrow, r);
        wv[r] = (r < nr && cv) ? ld_zc_u4(p.r_rows + (size_t)row * p.r_row_bytes + col0 * 2) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int r = 0; r < kRB; ++r) {
        const uint16_t xv = (uint16_t)__shfl_sync(0xffffffffu, myxs, r);
        if (r < nr) {
          const uint32_t h[4] = {wv[r].x, wv[r].y, wv[r].z, wv[r].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[2 * q] = fhfma_s_lo(xv, h[q], acc[2 * q]);
            acc[2 * q + 1] = fhfma_s_hi(xv, h[q], acc[2 * q + 1]);
          }
        }
      }
    }
    if (cv) {
      float* pp = p.part + (size_t)rbk * p.d_out + col0;
      *reinterpret_cast<float4*>(pp) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      *reinterpret_cast<float4*>(pp + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
    __threadfence();
    arrive_segment<RBITS>(p, seg, 1u, lane);
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
