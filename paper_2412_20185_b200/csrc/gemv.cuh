// Base GEMV o_b = W_hat x ("the base GEMV"; step a3 of SURVEY.md §8(a)) for
// sm_100a, laid out so that TWO CTAs fit on one SM (8 warps x <= 128 registers,
// <= ~110 KB shared memory each).  With programmatic dependent launch the next layer's CTA is
// then already resident while this layer computes: it fills its weight ring from HBM
// before griddepcontrol.wait, so at the layer boundary only x is still to be loaded and the
// HBM stream does not stop between layers (measured round 1: one CTA per SM left the x loads
// queued behind each new CTA's own weight burst, 1.0-1.8 us per layer).
//
//   warp 0           producer: 1-D bulk async copies (TMA engine) of a stage of TRS
//                    consecutive rows (+ their fp16 scales and u8 zeros) into a ring of
//                    `stages` smem slots, mbarrier full/empty handshake, L2 evict-first.
//   warps 1..NC      consumers (NC = 15): "teams" of T | NC warps; lane L of a team owns input group
//                    g = L % G (128 channels, x in 64 registers for the whole launch) of row
//                    L / G of the current pass (M = floor(32T / G) rows per pass), so no
//                    lane idles when G does not divide 32 (e.g. Phi-3's G = 40: T = 4, M = 3).
//                    A row is decoded in registers (decode.cuh) and accumulated with FHFMA
//                    (fp16 x fp16 -> fp32, exact products), one row at a time in a rolled
//                    loop (small code: the body stays in the L0 instruction cache).
// Rows: every GEMV CTA owns one contiguous, balanced row range (sizes differ by at most one
// row quantum), streamed in stages; reductions over a row's G lanes run in a fixed order
// (warp butterflies; for teams, smem partials summed in group order) -> deterministic.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#include "decode.cuh"
#include "ptx.cuh"

namespace decdec {

constexpr int kGemvNC = 15;                    // consumer warps per CTA (+ 1 producer warp)
constexpr int kGemvMaxRPS = 4;                 // row passes per stage
constexpr int kGemvTraceEvents = 20;           // same stride as the fused kernel's trace

struct GemvParams {
  const uint8_t* w;    // packed weights [d_out][row_bytes] (W3K / W4K)
  const uint16_t* ws;  // fp16 scales [d_out][G]
  const uint8_t* wz;   // u8 zeros [d_out][G]
  const uint16_t* x;   // fp16 [d_in]
  uint16_t* y;         // fp16 [d_out] (ob == nullptr)
  float* ob;           // fp32 o_b [d_out], self-validating relaxed stores (fused kernel's combine)
  int d_in, d_out, G, row_bytes;
  int NC, T, M, RPS, TRS, stages, Q;
  int pre;             // ring stages requested before griddepcontrol.wait (the rest after x)
  int s_row, z_row;    // bytes per row of the 2nd / 3rd stream: 2G / G (uniform s, z); 2^(b+1) / 0 (LUT)
  int team_red;        // 1: team reduction through smem partials; 0: in-warp butterflies (T == 1, G | 32)
  uint32_t stage_bytes, off_s, off_z, off_x, off_red, off_bar;
  int cta0;            // first blockIdx.x running the GEMV (fused kernel: after the DEC CTAs)
  int n_cta;           // GEMV CTAs
  int x_pf;            // prefetch x into L2 before griddepcontrol.wait
  // cross-layer L2 prefetch (decode-step executor): the NEXT layer's packed weights, scales and
  // zeros, split evenly over this launch's CTAs, requested into L2 (no smem, no completion) by
  // the producer after its own ring; the next layer's bulk copies then hit L2
  const uint8_t* pf_ptr[3];
  uint32_t pf_bytes[3];
  unsigned long long* trace;
};

#define DECDEC_GTRACE(p, ev)                                                                  \
  do {                                                                                       \
    if ((p).trace) (p).trace[blockIdx.x * kGemvTraceEvents + (ev)] = globaltimer();          \
  } while (0)

// One row's partial for input group g (this lane): s * sum_{i in g} (q_i - z) x_i.
// `gp` points at the group's packed codes in smem; xr holds the group's x as 64 half2.
template <int BITS>
__device__ __forceinline__ float row_group_dot(const uint8_t* gp, const uint32_t* xr, float Xs, float s24, float z, int rot) {
  float a[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (BITS == 4) {
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = *reinterpret_cast<const uint4*>(gp + 16 * ((j + rot) & 3));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      fma_w4_word(v[j].x, xr + 16 * j + 0, a);
      fma_w4_word(v[j].y, xr + 16 * j + 4, a);
      fma_w4_word(v[j].z, xr + 16 * j + 8, a);
      fma_w4_word(v[j].w, xr + 16 * j + 12, a);
    }
  } else {
    uint32_t w[12];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const uint4 t = *reinterpret_cast<const uint4*>(gp + 16 * j);
      w[4 * j] = t.x; w[4 * j + 1] = t.y; w[4 * j + 2] = t.z; w[4 * j + 3] = t.w;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) fma_w3_slice(w[3 * u], w[3 * u + 1], w[3 * u + 2], xr + 16 * u, a);
  }
  return s24 * fmaf(-z, Xs, combine_classes<BITS>(a));
}

// Two rows at once (12 independent FHFMA chains; x registers shared): more ILP per warp.
template <int BITS>
__device__ __forceinline__ void row_group_dot2(const uint8_t* g0, const uint8_t* g1, const uint32_t* xr, float Xs, float s0,
                                               float z0, float s1, float z1, int rot, float& v0, float& v1) {
  float a0[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, a1[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (BITS == 4) {
    uint4 u0[4], u1[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      u0[j] = *reinterpret_cast<const uint4*>(g0 + 16 * ((j + rot) & 3));
      u1[j] = *reinterpret_cast<const uint4*>(g1 + 16 * ((j + rot) & 3));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      fma_w4_word(u0[j].x, xr + 16 * j + 0, a0);
      fma_w4_word(u1[j].x, xr + 16 * j + 0, a1);
      fma_w4_word(u0[j].y, xr + 16 * j + 4, a0);
      fma_w4_word(u1[j].y, xr + 16 * j + 4, a1);
      fma_w4_word(u0[j].z, xr + 16 * j + 8, a0);
      fma_w4_word(u1[j].z, xr + 16 * j + 8, a1);
      fma_w4_word(u0[j].w, xr + 16 * j + 12, a0);
      fma_w4_word(u1[j].w, xr + 16 * j + 12, a1);
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
  v0 = s0 * fmaf(-z0, Xs, combine_classes<BITS>(a0));
  v1 = s1 * fmaf(-z1, Xs, combine_classes<BITS>(a1));
}

// This CTA's share of the next layer's bytes, into L2 (16-B aligned pieces of <= 64 KB).
__device__ __forceinline__ void l2_prefetch_share(const GemvParams& p, int c) {
#pragma unroll 1
  for (int r = 0; r < 3; ++r) {
    const uint32_t n16 = p.pf_bytes[r] >> 4;
    if (!p.pf_ptr[r] || !n16) continue;
    uint32_t a = (uint32_t)(((unsigned long long)n16 * c) / p.n_cta) << 4;
    const uint32_t b = (uint32_t)(((unsigned long long)n16 * (c + 1)) / p.n_cta) << 4;
    while (a < b) {
      const uint32_t len = min(b - a, 65536u);
      bulk_prefetch_l2(p.pf_ptr[r] + a, len);
      a += len;
    }
  }
}

// The GEMV part of one CTA (gemv CTA index c of p.n_cta).  smem: ring | x | red | barriers.
// LUTB = 0: uniform base (W3K / W4K codes, per-group s and z); LUTB = 3 | 4: non-uniform base
// with a per-row table of 2^LUTB fp16 values (codes W4K nibbles; BITS must be 4).
template <int BITS, int PAIR, int LUTB>
__device__ __forceinline__ void gemv_cta(const GemvParams& p, uint8_t* smem, int c) {
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* empty = full + p.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // balanced contiguous row range, in units of Q rows (keeps every bulk copy 16-B aligned)
  const int units = p.d_out / p.Q;
  const int r0 = (int)(((long long)c * units) / p.n_cta) * p.Q;
  const int r1 = (int)(((long long)(c + 1) * units) / p.n_cta) * p.Q;
  const int n_st = (r1 - r0 + p.TRS - 1) / p.TRS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], p.NC);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // warp 0 = producer (a dedicated warp: issuing bulk copies can stall on a full TMA queue, which
  // must not hold up consumer rows); warps 1..NC = consumers.  NC + 1 = 16 warps keeps <= 4
  // warps per SM sub-partition, so <= 128 registers per thread fit its 16K-register file.
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int first = min(p.stages, n_st), pre = min(p.pre, first);
      auto issue = [&](int i) {
        const int st = i % p.stages;
        const int ra = r0 + i * p.TRS;
        const int nr = min(p.TRS, r1 - ra);
        uint8_t* dst = ring + (size_t)st * p.stage_bytes;
        const uint32_t wb = (uint32_t)nr * p.row_bytes, sb = (uint32_t)nr * p.s_row, zb = (uint32_t)nr * p.z_row;
        mbar_arrive_expect_tx(&full[st], wb + sb + zb);
        bulk_g2s(dst, p.w + (size_t)ra * p.row_bytes, wb, &full[st], pol);
        bulk_g2s(dst + p.off_s, reinterpret_cast<const uint8_t*>(p.ws) + (size_t)ra * p.s_row, sb, &full[st], pol);
        if (zb) bulk_g2s(dst + p.off_z, p.wz + (size_t)ra * p.z_row, zb, &full[st], pol);
      };
      // only `pre` stages before griddepcontrol.wait: a deeper burst is still queued in the
      // memory system when the wait releases and delays the x loads every warp needs first
      for (int i = 0; i < pre; ++i) issue(i);
      pdl_wait();
      for (int i = pre; i < n_st; ++i) {
        if (i >= p.stages) mbar_wait(&empty[i % p.stages], ((i / p.stages) & 1) ^ 1);
        issue(i);
        if (i == first - 1) l2_prefetch_share(p, c);  // optional: the next layer's share into L2
      }
      if (first <= pre) l2_prefetch_share(p, c);
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  constexpr int GB = 16 * BITS;  // bytes of one 128-code group
  const int G = p.G, T = p.T, M = p.M;
  const int ct = threadIdx.x - 32, cw = warp - 1;
  const int team = cw / T, wi = cw % T;
  const int nteam = p.NC / T;
  const int L = wi * 32 + lane;
  const int g = L % G, rsub = L / G;
  const bool active = rsub < M;
  const bool warp_active = wi * 32 < M * G;  // some lane of this warp owns a (row, group)
  const int rot = (BITS == 4) ? ((g >> 1) & 3) : 0;
  pdl_wait();  // x is the previous layer's product
  if (ct == 0) DECDEC_GTRACE(p, 8);
  // x -> smem (coalesced 16-B loads), 16-B unit c of group gg at gg*16 + (c ^ (gg & 7))
  uint4* xsm = reinterpret_cast<uint4*>(smem + p.off_x);
  {
    const int nx = p.d_in >> 3, nct = p.NC * 32;
    const uint4* xg = reinterpret_cast<const uint4*>(p.x);
    for (int u = ct; u < nx; u += nct) {
      const uint4 v = ld_nc_u4(xg + u);
      xsm[(u & ~15) | ((u & 15) ^ ((u >> 4) & 7))] = v;
    }
    named_bar_sync(15, nct);
  }

  uint32_t xr[64];
  float Xs = 0.f;
  if (active) {
    const uint4* xp = xsm + g * 16;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = (j + rot) & 3;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint4 v = xp[(4 * cc + e) ^ (g & 7)];
        xr[16 * j + 4 * e + 0] = v.x;
        xr[16 * j + 4 * e + 1] = v.y;
        xr[16 * j + 4 * e + 2] = v.z;
        xr[16 * j + 4 * e + 3] = v.w;
      }
    }
    float xa[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const uint32_t one2 = 0x3C003C00u;  // (1.0, 1.0)
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      xa[i & 3] = fhfma_lo(one2, xr[i], xa[i & 3]);
      xa[4 + (i & 3)] = fhfma_hi(one2, xr[i], xa[4 + (i & 3)]);
    }
    Xs = (((xa[0] + xa[1]) + (xa[2] + xa[3])) + ((xa[4] + xa[5]) + (xa[6] + xa[7]))) * 5.9604644775390625e-08f;  // x 2^-24
    if (LUTB) {
#pragma unroll
      for (int w = 0; w < 16; ++w) lut_x_pairs(xr + 4 * w);  // (c, c+2) pairing of the table lookups
    }
  } else {
#pragma unroll
    for (int i = 0; i < 64; ++i) xr[i] = 0u;
  }
  if (ct == 0) DECDEC_GTRACE(p, 2);
  float* red = reinterpret_cast<float*>(smem + p.off_red);  // [2][TRS][G] team partials
  const int RPS = p.RPS, TRS = p.TRS;
  for (int i = 0; i < n_st; ++i) {
    const int st = i % p.stages;
    mbar_wait(&full[st], (i / p.stages) & 1);
    if (i == 0 && ct == 0) DECDEC_GTRACE(p, 3);
    const uint8_t* sw = ring + (size_t)st * p.stage_bytes;
    const uint16_t* ss = reinterpret_cast<const uint16_t*>(sw + p.off_s);
    const uint8_t* sz = sw + p.off_z;
    const int ra = r0 + i * TRS;
    const int nr = min(TRS, r1 - ra);
    float part[kGemvMaxRPS] = {0.f, 0.f, 0.f, 0.f};
    if (warp_active) {
      if (PAIR && !LUTB) {
#pragma unroll 1
        for (int m = 0; m < RPS; m += 2) {
          const int rr0 = (m * nteam + team) * M + rsub, rr1 = ((m + 1) * nteam + team) * M + rsub;
          const bool ok0 = active && rr0 < nr, ok1 = active && m + 1 < RPS && rr1 < nr;
          float v0 = 0.f, v1 = 0.f;
          if (ok0) {
            const int q1 = ok1 ? rr1 : rr0;
            const float s0 = __half2float(__ushort_as_half(ss[rr0 * G + g])) * 16777216.f;  // s * 2^24
            const float s1 = __half2float(__ushort_as_half(ss[q1 * G + g])) * 16777216.f;
            row_group_dot2<BITS>(sw + (size_t)rr0 * p.row_bytes + g * GB, sw + (size_t)q1 * p.row_bytes + g * GB, xr, Xs,
                                 s0, (float)sz[rr0 * G + g], s1, (float)sz[q1 * G + g], rot, v0, v1);
            if (!ok1) v1 = 0.f;
          }
          part[0] = m == 0 ? v0 : part[0];
          part[1] = m == 0 ? v1 : part[1];
          part[2] = m == 2 ? v0 : part[2];
          part[3] = m == 2 ? v1 : part[3];
        }
      } else {
#pragma unroll 1
        for (int m = 0; m < RPS; ++m) {
          const int rr = (m * nteam + team) * M + rsub;  // row within the stage
          float v = 0.f;
          if (active && rr < nr) {
            if (LUTB) {
              v = row_group_dot_lut<LUTB ? LUTB : 3>(sw + (size_t)rr * p.row_bytes + g * GB,
                                                      reinterpret_cast<const uint32_t*>(sw + p.off_s + (size_t)rr * p.s_row), xr, rot);
            } else {
              const float s24 = __half2float(__ushort_as_half(ss[rr * G + g])) * 16777216.f;  // s * 2^24
              const float z = (float)sz[rr * G + g];
              v = row_group_dot<BITS>(sw + (size_t)rr * p.row_bytes + g * GB, xr, Xs, s24, z, rot);
            }
          }
          part[0] = m == 0 ? v : part[0];
          part[1] = m == 1 ? v : part[1];
          part[2] = m == 2 ? v : part[2];
          part[3] = m == 3 ? v : part[3];
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);  // stage read (codes, scales, zeros)
    if (!p.team_red) {
      // T == 1, G | 32: the M rows of a pass sit in G-lane segments of the warp
      if (G == 32 && RPS == 4) {
        const bool hi16 = lane & 16, hi8 = lane & 8;
        float u0 = (hi16 ? part[2] : part[0]) + __shfl_xor_sync(0xffffffffu, hi16 ? part[0] : part[2], 16);
        float u1 = (hi16 ? part[3] : part[1]) + __shfl_xor_sync(0xffffffffu, hi16 ? part[1] : part[3], 16);
        float v = (hi8 ? u1 : u0) + __shfl_xor_sync(0xffffffffu, hi8 ? u0 : u1, 8);
#pragma unroll
        for (int o = 4; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((lane & 7) == 0) {
          const int m = (hi16 ? 2 : 0) + (hi8 ? 1 : 0);
          const int rr = m * nteam + team;
          if (rr < nr) {
            if (p.ob) st_relaxed_gpu_f32(p.ob + ra + rr, v);
            else p.y[ra + rr] = __half_as_ushort(__float2half_rn(v));
          }
        }
      } else if (G == 32 && RPS == 2) {
        const bool hi16 = lane & 16;
        float v = (hi16 ? part[1] : part[0]) + __shfl_xor_sync(0xffffffffu, hi16 ? part[0] : part[1], 16);
#pragma unroll
        for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((lane & 15) == 0) {
          const int rr = (hi16 ? 1 : 0) * nteam + team;
          if (rr < nr) {
            if (p.ob) st_relaxed_gpu_f32(p.ob + ra + rr, v);
            else p.y[ra + rr] = __half_as_ushort(__float2half_rn(v));
          }
        }
      } else {
#pragma unroll
        for (int m = 0; m < kGemvMaxRPS; ++m) {
          if (m >= RPS) break;
          float v = part[m];
          for (int o = G >> 1; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          const int rr = (m * nteam + team) * M + rsub;
          if (g == 0 && rr < nr) {
            if (p.ob) st_relaxed_gpu_f32(p.ob + ra + rr, v);
            else p.y[ra + rr] = __half_as_ushort(__float2half_rn(v));
          }
        }
      }
    } else {
      // team: partials to smem [row][g], one named barrier per team, then the team's warps
      // sum rows in group order (lane j: groups j, j+32, ...; then a fixed butterfly)
      float* rb = red + (size_t)(i & 1) * TRS * G;
      if (active) {
#pragma unroll
        for (int m = 0; m < kGemvMaxRPS; ++m) {
          if (m >= RPS) break;
          const int rr = (m * nteam + team) * M + rsub;
          if (rr < nr) rb[rr * G + g] = part[m];
        }
      }
      named_bar_sync(1 + team, T * 32);
      const int rows_team = RPS * M;  // rows of this team in the stage: (m * nteam + team) * M + q
      for (int q = wi; q < rows_team; q += T) {
        const int m = q / M, qs = q % M;
        const int rr = (m * nteam + team) * M + qs;
        if (rr >= nr) continue;  // warp-uniform
        float v = 0.f;
        for (int gg = lane; gg < G; gg += 32) v += rb[rr * G + gg];
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) {
          if (p.ob) st_relaxed_gpu_f32(p.ob + ra + rr, v);
          else p.y[ra + rr] = __half_as_ushort(__float2half_rn(v));
        }
      }
    }
  }
  if (ct == 0) DECDEC_GTRACE(p, 4);
}

template <int BITS, int PAIR, int LUTB>
__device__ __forceinline__ void gemv_kernel_body(const GemvParams& p) {
  extern __shared__ __align__(128) uint8_t smem[];
  // the next layer's CTAs may become resident now (two CTAs per SM): they fill their weight
  // rings while this layer computes
  pdl_launch_dependents();
  if (threadIdx.x == 0) DECDEC_GTRACE(p, 0);
  if (p.x_pf) {  // x into L2 before griddepcontrol.wait (L2 is the coherence point)
    const int lines = (p.d_in * 2 + 127) >> 7;
    const int i = (int)threadIdx.x * 8 + ((int)blockIdx.x & 7);
    if (i < lines) prefetch_l2(reinterpret_cast<const uint8_t*>(p.x) + ((size_t)i << 7));
  }
  gemv_cta<BITS, PAIR, LUTB>(p, smem, (int)blockIdx.x - p.cta0);
}

// 1 producer + 15 consumer warps, one CTA per SM.  (Measured: a two-CTAs-per-SM variant with
// 8 warps each -- the next layer's CTA resident and its ring filled before this layer ends --
// did co-reside, but 8 warps computing cost more than the overlap won: k_chunk-0 step 1.44 vs
// 1.25 ms.)
template <int BITS, int PAIR, int LUTB = 0>
__global__ void __launch_bounds__(512, 1) k_gemv16(const GemvParams p) {
  gemv_kernel_body<BITS, PAIR, LUTB>(p);
}

}  // namespace decdec
