// In-register decode of the packed layouts of include/decdec.h (DESIGN.md ledger L6).
//
// Base weights: a code q is masked in place into the mantissa field of an fp16 half,
// exponent 0, i.e. the fp16 SUBNORMAL q * 2^(pos-24) where pos = its bit offset inside
// the half.  One LOP3 extracts two codes (one per half); FHFMA multiplies them exactly
// by x.  Codes at different offsets feed different fp32 accumulators ("scale classes")
// that are recombined once per group with exact power-of-two factors.
//   W4K: class 0 = offset 0 (x 2^-24), class 1 = offset 4 (x 2^-20)
//   W3K: class 0 = offset 0 (x 2^-24), class 1 = offset 3 (x 2^-21), class 2 = offset 6 (x 2^-18)
// The group sum is  sum q*x = 2^24 * (acc0 + acc1/16)            (4-bit)
//                             2^24 * (acc0 + acc1/8 + acc2/64)    (3-bit)
// (each class accumulator is split into a low-half and a high-half chain).
#pragma once
#include <cstdint>
#include "ptx.cuh"

namespace decdec {

// ---------------------------------------------------------------- W4K
// word: channels c = 0..7 at bit 4*(c>>1) + 16*(c&1); pair p = channels (2p, 2p+1).
// m[p] holds the pair as two subnormal halves; class(p) = p & 1.
__device__ __forceinline__ void decode_w4_word(uint32_t w, uint32_t m[4]) {
  m[0] = w & 0x000F000Fu;
  m[1] = w & 0x00F000F0u;
  const uint32_t v = w >> 8;
  m[2] = v & 0x000F000Fu;
  m[3] = v & 0x00F000F0u;
}
__host__ __device__ constexpr int w4_class(int p) { return p & 1; }

// acc[2c + h] += (half h of class-c codes) . x for one 8-channel word; xr[p] = (x[2p], x[2p+1]).
// Low and high halves feed separate accumulators: 4 independent FHFMA chains per row.
__device__ __forceinline__ void fma_w4_word(uint32_t w, const uint32_t* xr, float* acc) {
  uint32_t m[4];
  decode_w4_word(w, m);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    acc[2 * w4_class(q)] = fhfma_lo(m[q], xr[q], acc[2 * w4_class(q)]);
    acc[2 * w4_class(q) + 1] = fhfma_hi(m[q], xr[q], acc[2 * w4_class(q) + 1]);
  }
}

// ---------------------------------------------------------------- W3K
// One 32-channel slice = 3 words.  Pair k = 5t + p (t = word, p = position 0..4) holds
// channels (10t + 2p, 10t + 2p + 1); pair 15 holds channels (30, 31) assembled from the
// spare bit 15 / 31 of the three words.  class: p in {0,3} -> 0, p in {1,4} -> 1, p = 2 -> 2,
// pair 15 -> 2.
__device__ __forceinline__ void decode_w3_slice(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t m[16]) {
  const uint32_t w[3] = {w0, w1, w2};
  uint32_t v[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    m[5 * t + 0] = w[t] & 0x00070007u;
    m[5 * t + 1] = w[t] & 0x00380038u;
    m[5 * t + 2] = w[t] & 0x01C001C0u;
    v[t] = w[t] >> 9;
    m[5 * t + 3] = v[t] & 0x00070007u;
    m[5 * t + 4] = v[t] & 0x00380038u;
  }
  // spare bits now at bit 6 (low half) / 22 (high half) of v[t]; code bit t -> offset 6 + t
  m[15] = (v[0] & 0x00400040u) | ((v[1] & 0x00400040u) << 1) | ((v[2] & 0x00400040u) << 2);
}
__host__ __device__ constexpr int w3_class(int k) {
  return k == 15 ? 2 : ((k % 5) == 0 || (k % 5) == 3) ? 0 : ((k % 5) == 2 ? 2 : 1);
}

// acc[2c + h] += (half h of class-c codes) . x(xr[0..15]): 6 independent FHFMA chains per row
__device__ __forceinline__ void fma_w3_slice(uint32_t w0, uint32_t w1, uint32_t w2, const uint32_t* xr, float* acc) {
  uint32_t m[16];
  decode_w3_slice(w0, w1, w2, m);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    acc[2 * w3_class(k)] = fhfma_lo(m[k], xr[k], acc[2 * w3_class(k)]);
    acc[2 * w3_class(k) + 1] = fhfma_hi(m[k], xr[k], acc[2 * w3_class(k) + 1]);
  }
}

// Group sum of (q . x) in units of 2^-24, from the split accumulators.
template <int BITS>
__device__ __forceinline__ float combine_classes(const float* a) {
  if (BITS == 4) return fmaf(a[2] + a[3], 0.0625f, a[0] + a[1]);
  return fmaf(a[4] + a[5], 0.015625f, fmaf(a[2] + a[3], 0.125f, a[0] + a[1]));
}

// ---------------------------------------------------------------- Rq (residual, 4-bit)
// word: columns c = 0..7 at bit 4*(c>>1) + 16*(c&1), nibble = code + 8.  Returns the four
// column pairs as exact fp16 integer codes in [-7, 7]: (1024 + n) via the 0x6400 exponent,
// minus 1032, both exact in fp16.
__device__ __forceinline__ void decode_rq_word(uint32_t w, uint32_t c[4]) {
  const __half2 bias = __halves2half2(__ushort_as_half(0x6408), __ushort_as_half(0x6408));  // 1032
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const uint32_t h = ((w >> (4 * p)) & 0x000F000Fu) | 0x64006400u;
    __half2 hv = *reinterpret_cast<const __half2*>(&h);
    hv = __hsub2(hv, bias);
    c[p] = *reinterpret_cast<const uint32_t*>(&hv);
  }
}

// ---------------------------------------------------------------- LUT (non-uniform base, NEXT-3)
// Codes are W4K nibbles (channel c of a word at bit 4*(c>>1) + 16*(c&1); values < 2^LB).  The
// row's table of 2^LB fp16 values is held as byte planes: tl[t] / th[t] = the low / high bytes
// of entries 4t..4t+3, so ONE `prmt` looks up four codes' low (or high) bytes at once (its
// selector nibbles are the codes: bits 2..0 pick one of 8 bytes, bit 3 must be 0).  Two more
// `prmt` interleave them into fp16 pairs (channel c, c+2) -- x is kept in the same pairing --
// and FHFMA multiplies exactly into fp32.  LB = 4 looks up the low 3 code bits in both halves of
// the table and blends by code bit 3 (byte masks built by `prmt`'s sign-replicate mode).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// table (2^LB fp16, as LB == 3 ? 4 : 8 half2 words e[]) -> byte planes tl[], th[]
template <int LB>
__device__ __forceinline__ void lut_planes(const uint32_t* e, uint32_t* tl, uint32_t* th) {
#pragma unroll
  for (int t = 0; t < (1 << LB) / 4; ++t) {
    tl[t] = prmt(e[2 * t], e[2 * t + 1], 0x6420u);
    th[t] = prmt(e[2 * t], e[2 * t + 1], 0x7531u);
  }
}

// acc[0..3] += table[codes of word w] . x for one 8-channel word; xp[0..3] = x pairs
// (0,2), (4,6), (1,3), (5,7) of the word (see lut_x_pairs).
template <int LB>
__device__ __forceinline__ void fma_lut_word(uint32_t w, const uint32_t* tl, const uint32_t* th, const uint32_t* xp,
                                             float* acc) {
  uint32_t le, he, lo, ho;
  if (LB == 3) {
    const uint32_t so = w >> 16;
    le = prmt(tl[0], tl[1], w);
    he = prmt(th[0], th[1], w);
    lo = prmt(tl[0], tl[1], so);
    ho = prmt(th[0], th[1], so);
  } else {
    const uint32_t m = w & 0x77777777u, so = m >> 16, w4 = w << 4;
    const uint32_t me = prmt(w4, w, 0xD9C8u), mo = prmt(w4, w, 0xFBEAu);  // 0xFF bytes where code bit 3 is set
    le = (prmt(tl[0], tl[1], m) & ~me) | (prmt(tl[2], tl[3], m) & me);
    he = (prmt(th[0], th[1], m) & ~me) | (prmt(th[2], th[3], m) & me);
    lo = (prmt(tl[0], tl[1], so) & ~mo) | (prmt(tl[2], tl[3], so) & mo);
    ho = (prmt(th[0], th[1], so) & ~mo) | (prmt(th[2], th[3], so) & mo);
  }
  const uint32_t v02 = prmt(le, he, 0x5140u), v46 = prmt(le, he, 0x7362u);  // (ch0, ch2), (ch4, ch6)
  const uint32_t v13 = prmt(lo, ho, 0x5140u), v57 = prmt(lo, ho, 0x7362u);  // (ch1, ch3), (ch5, ch7)
  acc[0] = fhfma_lo(v02, xp[0], acc[0]);
  acc[1] = fhfma_hi(v02, xp[0], acc[1]);
  acc[2] = fhfma_lo(v46, xp[1], acc[2]);
  acc[3] = fhfma_hi(v46, xp[1], acc[3]);
  acc[0] = fhfma_lo(v13, xp[2], acc[0]);
  acc[1] = fhfma_hi(v13, xp[2], acc[1]);
  acc[2] = fhfma_lo(v57, xp[3], acc[2]);
  acc[3] = fhfma_hi(v57, xp[3], acc[3]);
}

// x registers of one 8-channel word, (x0,x1),(x2,x3),(x4,x5),(x6,x7) -> (x0,x2),(x4,x6),(x1,x3),(x5,x7)
__device__ __forceinline__ void lut_x_pairs(uint32_t* xr4) {
  const uint32_t a = xr4[0], b = xr4[1], c = xr4[2], d = xr4[3];
  xr4[0] = prmt(a, b, 0x5410u);
  xr4[1] = prmt(c, d, 0x5410u);
  xr4[2] = prmt(a, b, 0x7632u);
  xr4[3] = prmt(c, d, 0x7632u);
}

// LUT base (NEXT-3): one row's partial sum_{i in g} lut[q_i] x_i for input group g.  gp: the
// group's 64 B of W4K nibble codes; lp: the row's table (2^LB fp16) in smem; xr: x in the
// (c, c+2) pairing of lut_x_pairs.
template <int LB>
__device__ __forceinline__ float row_group_dot_lut(const uint8_t* gp, const uint32_t* lp, const uint32_t* xr, int rot) {
  uint32_t e[1 << (LB - 1)], tl[(1 << LB) / 4], th[(1 << LB) / 4];
#pragma unroll
  for (int t = 0; t < (1 << LB) / 8; ++t) {
    const uint4 v = reinterpret_cast<const uint4*>(lp)[t];
    e[4 * t] = v.x; e[4 * t + 1] = v.y; e[4 * t + 2] = v.z; e[4 * t + 3] = v.w;
  }
  lut_planes<LB>(e, tl, th);
  float a[4] = {0.f, 0.f, 0.f, 0.f};
  uint4 v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = *reinterpret_cast<const uint4*>(gp + 16 * ((j + rot) & 3));
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    fma_lut_word<LB>(v[j].x, tl, th, xr + 16 * j + 0, a);
    fma_lut_word<LB>(v[j].y, tl, th, xr + 16 * j + 4, a);
    fma_lut_word<LB>(v[j].z, tl, th, xr + 16 * j + 8, a);
    fma_lut_word<LB>(v[j].w, tl, th, xr + 16 * j + 12, a);
  }
  return (a[0] + a[1]) + (a[2] + a[3]);
}

}  // namespace decdec
