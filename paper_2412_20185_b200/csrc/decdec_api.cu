// C-ABI entry points of libdecdec (include/decdec.h): validation, launch planning and
// launches of the sm_100a kernels in select.cuh / linear.cuh.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "decdec.h"
#include "gemv.cuh"
#include "linear.cuh"
#include "select.cuh"
#include "p2p_internal.h"
#include "tp_internal.h"

using namespace decdec;

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v, size_t a = kAlign) { return (v + a - 1) / a * a; }

int device_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
  }
  return cache[dev];
}

unsigned long long* g_trace = nullptr;  // debug timelines (decdec_debug_trace)
size_t g_trace_bytes = 0;
int* g_dbg_idx = nullptr;  // debug: every DEC CTA's own selection (decdec_debug_selections)
uint16_t* g_dbg_xs = nullptr;
int g_dbg_cap = 0, g_dbg_ctas = 0;
constexpr size_t kTraceStride = 160 * 20;  // u64 per layer in stack traces (<= 160 CTAs)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct Plan {
  int G, NKW, NSLOTS, RPS, TR, NC, stages, n_tiles, grid, n_dec;  // grid = GEMV CTAs (+ n_dec DEC CTAs)
  int n_seg, rpi, gws, nparts, one_seg;  // DEC: output segments, rows per gather item, items and partials per segment
  int early_reads, early_cap;            // DEC: read the D rows during the selection (linear.cuh)
  double r_ratio, t_hbm_us;              // PCIe / HBM roofline time of the call; HBM roofline (us)
  uint32_t stage_bytes, off_s, off_z, off_sel, off_x, off_part, off_rsc, off_stage;
  size_t smem;
};

constexpr size_t kSmemBudget = 200 * 1024;

// Launch plan: enumerate (consumer warps NC, rows per slot RPS); pick the one minimising the
// busiest CTA's bytes (ceil(tiles / SMs) x (stage bytes + a per-tile overhead equivalent)),
// ties -> more consumer warps.  DECDEC_PLAN="NC,RPS" overrides (tuning).
// Number of DEC CTAs: ~544 warps of zero-copy reads (measured on the llama3-8b stack at
// k_chunk 21, 17-warp CTAs: 4 -> 105 us/block, 8 -> 92, 16 -> 84, 32 -> 80, 64 -> 78 within
// noise, while the GEMV CTAs lose SMs); DECDEC_NDEC overrides.
int g_dec_override = 0;  // decdec_set_dec_ctas (tuner), 0 = automatic

// r = PCIe roofline time / HBM roofline time of the call.  Measured with tools/tune.py on the
// Llama-3-8B classes (profiles/r01_tuner.json, 17-warp CTAs): while the GEMV bounds the call
// (r < 1) every SM taken from it costs time and 16 DEC CTAs suffice; once PCIe dominates, more
// DEC CTAs issue the gather faster (r >= 2.5: 48 beat 32 by 1-3 %, 64 beat 48 by ~1 % on the
// k_chunk 21 step).
int dec_ctas(int warps_per_cta, double r) {
  if (g_dec_override > 0) return g_dec_override;
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("DECDEC_NDEC");
    env = e ? atoi(e) : 0;
  }
  if (env > 0) return env;
  // r >= 2.5: 48 CTAs of 17 warps since the 16-B gather and the fitted stack grids (k_chunk 21
  // -1.7 % vs 64, profiles/r02_s3_experiments.json); DECDEC_DEC_WARPS_HI overrides
  static int hi = -1;
  if (hi < 0) {
    const char* e = getenv("DECDEC_DEC_WARPS_HI");
    hi = e ? atoi(e) : 816;
    if (hi < 17) hi = 17;
  }
  static int mid = -1;  // DECDEC_DEC_WARPS_MID: gather warps for 1 <= r < 2.5
  if (mid < 0) {
    const char* e = getenv("DECDEC_DEC_WARPS_MID");
    mid = e ? atoi(e) : 544;
    if (mid < 17) mid = 17;
  }
  const int base = r < 1.0 ? 272 : (r < 2.5 ? mid : hi);  // gather warps
  int n = (base + warps_per_cta - 1) / warps_per_cta;
  return n < 2 ? 2 : (n > 64 ? 64 : n);
}

// Early D-row reads (linear.cuh dec_cta): on for calls whose PCIe/HBM roofline ratio r lies in a
// window (early_reads() below) -- first measured with the 4-B gather (k_chunk 21 -3.6 %, k_chunk
// 1-4 +2-3 %), re-measured with the 16-B gather and the fitted step graph.  DECDEC_EARLY=0|1
// forces it.
// Early reads per warp at most (DECDEC_EARLY_CAP, 0 = every D row the warp holds): an SM keeps
// few zero-copy requests in flight, so a warp with many D rows stalls in its early-read loop and
// holds up the selection's barrier 2 (d layer: D placed at ~19000 instead of ~12000 cycles).
// Measured (1x B200, Llama-3-8B k_chunk-21 step, 4 alternating runs): cap 4 -1.6 % vs no cap with
// the 4-B gather, +-0 with the 16-B gather (profiles/r02_s3_experiments.json).
int early_cap() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("DECDEC_EARLY_CAP");
    env = e ? atoi(e) : 4;
    if (env < 0) env = 0;
    const char* f = getenv("DECDEC_EARLY_SPARE_FIN");  // 1: the finisher warp issues none
    if (f && atoi(f) > 0) env |= 1 << 16;
  }
  return env;
}

int early_reads(double r) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("DECDEC_EARLY");
    env = e ? atoi(e) : -1;
  }
  if (env >= 0) return env > 0;
  // window re-measured with the 16-B gather and the fitted step graph (forced on vs this window,
  // profiles/r02_s3_experiments.json): k_chunk 8 (r ~1.3) -2.0 %, 32 (r ~5.2) -3.8 %, 48 -1.2 %,
  // 64 +-0.5 %, 82 (r ~13) +2.8 %, 4 (r ~0.6) +-0.1 %; with [1.0, 9.0] vs [1.5, 4.5]: 8 -1.8 %,
  // 32 -3.8 %, 48 -1.2 %, Phi-3 32 -3.4 %, 6 (r ~1.0) +0.5 % -> lower bound 1.1
  return r >= 1.1 && r <= 9.0;
}

// DEC CTA layout: CTA c owns segments c, c + n_dec, ...; a segment's k_sel rows are split in
// gws items of rpi rows, sized so that every warp of a DEC CTA has an item in the first round
// (items = local segments x gws >= warps) but an item never exceeds one load per row per lane.
// smem: SelectSmem + staged x | idx, xs | partials [ns][gws][256] f32 | residual scales [ns][256].
bool plan_dec(int d_out, int k_sel, int sel_len, int warps, int max_rpi, double r, Plan* p) {
  p->n_seg = (d_out + kSegCols - 1) / kSegCols;
  static int env_rpi = -1;
  if (env_rpi < 0) {
    const char* e = getenv("DECDEC_GATHER_ROWS");
    env_rpi = e ? atoi(e) : 0;
  }
  size_t sel_bytes = select_block_smem_bytes(sel_len);
  if (sel_bytes < select_split_smem_bytes(sel_len)) sel_bytes = select_split_smem_bytes(sel_len);
  const uint32_t off_sel = (uint32_t)align_up(sel_bytes, 16);
  const uint32_t off_part = (uint32_t)align_up((size_t)off_sel + (size_t)k_sel * 6, 16);
  const size_t row_b = max_rpi == kGatherRows16 ? 16 : 4;  // bytes per lane per staged row
  // A DEC CTA without a segment would only select and exit while holding an SM the GEMV
  // needs; and at least half of the SMs stay GEMV CTAs (no plan where DEC CTAs fill the GPU).
  const int nd_max = p->n_seg < device_sms() / 2 ? p->n_seg : device_sms() / 2;
  int nd_first = dec_ctas(warps, r);
  if (nd_first > nd_max) nd_first = nd_max;
  if (nd_first < 1) nd_first = 1;
  for (int nd = nd_first; nd <= nd_max; nd = (nd == nd_max ? nd_max + 1 : (2 * nd < nd_max ? 2 * nd : nd_max))) {
    const int ns = (p->n_seg + nd - 1) / nd;
    const int gws_target = (warps + ns - 1) / ns;
    // staging rows per buffer: as many as fit (<= max_rpi); fewer rows -> more, smaller items
    for (int cap = max_rpi; cap >= 2; cap /= 2) {
      int rpi = (k_sel + gws_target - 1) / gws_target;
      if (rpi > cap) rpi = cap;
      if (env_rpi > 0 && env_rpi < rpi) rpi = env_rpi;
      if (rpi < 1) rpi = 1;
      const int gws = (k_sel + rpi - 1) / rpi;
      const int one_seg = ns == 1;
      const int nparts = one_seg ? (gws < warps ? gws : warps) : gws;
      const uint32_t off_rsc = off_part + (uint32_t)ns * nparts * kSegCols * 4;
      // + 16 B: the mbarrier the residual scales' bulk copies complete on
      const uint32_t off_stage = (uint32_t)align_up((size_t)off_rsc + (size_t)ns * kSegCols * 2 + 16, 16);
      const size_t dec = off_stage + (size_t)warps * 2 * rpi * 32 * row_b;
      if (dec > kSmemBudget + 16 * 1024) continue;
      p->n_dec = nd;
      p->rpi = rpi;
      p->gws = gws;
      p->nparts = nparts;
      p->one_seg = one_seg;
      p->off_sel = off_sel;
      p->off_part = off_part;
      p->off_rsc = off_rsc;
      p->off_stage = off_stage;
      if (dec > p->smem) p->smem = dec;
      return true;
    }
  }
  return false;
}

// lut_bits = 3 | 4: non-uniform base (W4K nibble codes + a 2^lut_bits fp16 table per row in
// place of the group scales / zeros)
decdec_status make_plan(int d_in, int d_out, int bits, int k_sel, Plan* pl, int sel_len = 0, int r_bits = 4,
                        int lut_bits = 0) {
  if (sel_len == 0) sel_len = d_in;
  const int G = d_in / DECDEC_GROUP;
  const int sms = device_sms();
  const bool small_g = G <= 32 && 32 % G == 0;
  const int nkw = small_g ? 0 : (G + 31) / 32;
  if (lut_bits) bits = 4;  // codes are W4K nibbles
  const uint32_t row_bytes = (uint32_t)d_in * bits / 8;
  const uint32_t meta_row = lut_bits ? (2u << lut_bits) : (uint32_t)G * 2;  // scale / table bytes per row
  const uint32_t zero_row = lut_bits ? 0u : (uint32_t)G;
  static int env_nc = -1, env_rps = -1;
  if (env_nc < 0) {
    const char* e = getenv("DECDEC_PLAN");
    env_nc = 0;
    env_rps = 0;
    if (e) sscanf(e, "%d,%d", &env_nc, &env_rps);
  }
  // PCIe / HBM roofline time ratio with the measured link and copy bandwidths
  const double t_hbm = ((double)d_in * d_out * bits / 8 + (double)d_out * (meta_row + zero_row)) / 6455.0;
  const double t_pcie = ((double)k_sel * d_out * r_bits / 8 + 2.0 * d_out) / 51.4;
  const double r_ratio = t_pcie / t_hbm;
  Plan best{};
  double best_cost = 1e300;
  bool have = false;
  for (int nc = 1; nc <= 16; ++nc) {
    if (small_g ? (nc & (nc - 1)) != 0 : (nc % nkw || ((nc / nkw) & (nc / nkw - 1)) != 0)) continue;
    for (int rps = 1; rps <= kMaxRPS; rps *= 2) {  // rows are computed in pairs: RPS 1 halves the ILP
      if (env_nc > 0 && (nc != env_nc || rps != env_rps)) continue;
      Plan p{};
      p.G = G;
      p.NKW = nkw;
      p.NC = nc;
      p.NSLOTS = small_g ? nc * (32 / G) : nc / nkw;
      p.RPS = rps;
      p.TR = p.NSLOTS * rps;
      if (p.TR > kSegCols || kSegCols % p.TR || d_out % p.TR || (p.TR * G) % 16) continue;
      p.off_s = (uint32_t)p.TR * row_bytes;
      p.off_z = p.off_s + (uint32_t)p.TR * meta_row;
      p.stage_bytes = (uint32_t)align_up(p.off_z + (uint32_t)p.TR * zero_row, 16);
      const size_t red = (size_t)2 * p.NSLOTS * 4 * (nkw ? nkw : 1) * 4;
      const size_t xb = align_up((size_t)d_in * 2, 16);  // staged x (swizzled, see k_linear)
      const size_t avail = kSmemBudget - red - 16 * 8 - xb;
      p.stages = (int)(avail / p.stage_bytes);
      if (p.stages > 8) p.stages = 8;
      if (p.stages < 2) continue;
      // Cap the bytes in flight per SM near what Little's law needs at HBM latency: a deeper
      // ring does not add bandwidth, it only queues ~µs of traffic ahead of latency-critical
      // loads (x, selection, gather bookkeeping).
      {
        static int env_kb = -1;
        if (env_kb < 0) {
          const char* e = getenv("DECDEC_INFLIGHT_KB");
          env_kb = e ? atoi(e) : 128;
        }
        int cap = (int)(((size_t)env_kb * 1024) / p.stage_bytes);
        if (cap < 2) cap = 2;
        if (p.stages > cap) p.stages = cap;
      }
      p.n_tiles = d_out / p.TR;
      // k > 0: the DEC CTAs take the first SMs; GEMV CTAs fill the rest
      p.off_x = (uint32_t)align_up((size_t)p.stages * p.stage_bytes + red + (size_t)2 * p.stages * 8, 16);
      p.smem = p.off_x + xb;
      p.n_dec = 0;
      if (k_sel > 0 && !plan_dec(d_out, k_sel, sel_len, 1 + nc, r_bits == 16 ? kGatherRows16 : kGatherRows4, r_ratio, &p))
        continue;
      p.early_reads = k_sel > 0 && early_reads(r_ratio);
      p.r_ratio = k_sel > 0 ? r_ratio : 0.0;
      p.t_hbm_us = t_hbm / 1000.0;
      p.early_cap = early_cap();
      const int max_grid = sms - p.n_dec;
      if (max_grid <= 0) continue;
      p.grid = p.n_tiles < max_grid ? p.n_tiles : max_grid;
      if (p.smem > kSmemBudget + 16 * 1024) continue;
      const double waves = (double)((p.n_tiles + max_grid - 1) / max_grid);
      // more consumer warps hide more latency (measured: 16 warps beat 8 by 6-11% on the big layers)
      double cost = waves * ((double)p.stage_bytes + 8192.0) * (1.0 + 2.0 / nc) * (rps == 1 ? 1.5 : 1.0);
      if (k_sel > 0) cost *= 1.0 + 0.5 * (16 - nc) / 16.0;  // DEC CTAs gather with every warp of the CTA
      if (!have || cost < best_cost * 0.999 || (cost <= best_cost * 1.001 && p.NC > best.NC)) {
        best = p;
        best_cost = cost;
        have = true;
      }
    }
  }
  if (!have) return DECDEC_EUNSUPPORTED;
  *pl = best;
  return DECDEC_OK;
}

// ---------------------------------------------------------------- k_gemv plan (k = 0)
// Two CTAs per SM: <= kGemvSmemBudget dynamic smem each.  Team shape (T warps, M rows per pass)
// maximises the issuing lanes that own a (row, group): efficiency M*G / (32 * ceil(M*G/32)),
// ties -> smaller T.  RPS (passes per stage): the largest with >= 3 ring stages, else >= 2.

// DECDEC_GEMV_PAIR = 0 | 1: rows one at a time or in pairs (A/B knob)
bool gemv_pair() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("DECDEC_GEMV_PAIR");
    env = e ? (atoi(e) > 0) : 0;  // measured: pairs 1.265 vs single rows 1.251 ms (k_chunk-0 step)
  }
  return env == 1;
}
// DECDEC_PREWAIT_KB: ring bytes requested before griddepcontrol.wait (A/B knob)
int prewait_kb() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("DECDEC_PREWAIT_KB");
    env = e ? atoi(e) : 32;
  }
  return env;
}

constexpr size_t kGemvSmemBudget = 200 * 1024;  // one CTA per SM
struct GemvPlan {
  GemvParams gp;
  size_t smem;
  int grid;
};

// lut_bits = 0: uniform base (bits = 3 | 4); lut_bits = 3 | 4: LUT base (codes in W4K nibbles)
decdec_status make_gemv_plan(int d_in, int d_out, int bits, int n_cta_max, GemvPlan* out, int lut_bits = 0) {
  const int G = d_in / DECDEC_GROUP;
  GemvParams g{};
  g.d_in = d_in;
  g.d_out = d_out;
  g.G = G;
  g.row_bytes = d_in * (lut_bits ? 4 : bits) / 8;
  const int NC = kGemvNC;
  const size_t budget = kGemvSmemBudget;
  g.NC = NC;
  g.s_row = lut_bits ? 2 << lut_bits : 2 * G;  // LUT: the row's table of 2^b fp16
  g.z_row = lut_bits ? 0 : G;
  int bestT = 0, bestM = 0;
  double best_eff = -1.0;
  for (int T = 1; T <= NC; ++T) {
    if (NC % T) continue;
    const int M = 32 * T / G;
    if (M < 1) continue;
    const int lanes = M * G, warps = (lanes + 31) / 32;
    const double eff = (double)lanes / (32.0 * warps);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      bestT = T;
      bestM = M;
    }
  }
  if (!bestT) return DECDEC_EUNSUPPORTED;  // G > 256: d_in > 32768
  g.T = bestT;
  g.M = bestM;
  g.team_red = !(bestT == 1 && 32 % G == 0);
  int Q = 1;
  while (!lut_bits && (Q * G) % 16) ++Q;  // rows*G bytes of zeros (and 2x of scales) stay 16-B multiples
  g.Q = Q;
  const int nteam = NC / bestT;
  const size_t xb = align_up((size_t)d_in * 2, 16);
  bool ok = false;
  for (int need = 3; need >= 2 && !ok; --need) {
    for (int rps = kGemvMaxRPS; rps >= 1; rps /= 2) {
      const int TRS = (nteam * bestM * rps) / Q * Q;  // stage rows: a multiple of the row quantum
      if (TRS == 0) continue;
      const uint32_t off_s = (uint32_t)align_up((size_t)TRS * g.row_bytes, 16);
      const uint32_t off_z = off_s + (uint32_t)align_up((size_t)TRS * g.s_row, 16);
      const uint32_t sb = (uint32_t)align_up((size_t)off_z + (size_t)TRS * g.z_row, 128);
      const size_t red = g.team_red ? align_up((size_t)2 * TRS * G * 4, 16) : 0;
      const size_t fixed = xb + red + 16 * 8;
      if (fixed + (size_t)need * sb > budget) continue;
      int stages = (int)((budget - fixed) / sb);
      if (stages > 8) stages = 8;
      g.RPS = (TRS + nteam * bestM - 1) / (nteam * bestM);  // passes that cover TRS rows
      g.TRS = TRS;
      g.stages = stages;
      g.stage_bytes = sb;
      g.off_s = off_s;
      g.off_z = off_z;
      g.off_x = (uint32_t)((size_t)stages * sb);
      g.off_red = (uint32_t)align_up((size_t)g.off_x + xb, 16);
      g.off_bar = (uint32_t)align_up((size_t)g.off_red + red, 16);
      out->smem = (size_t)g.off_bar + 2 * (size_t)stages * 8;
      g.pre = (int)(((size_t)prewait_kb() * 1024) / sb);
      if (g.pre < 1) g.pre = 1;
      ok = true;
      break;
    }
  }
  if (!ok) return DECDEC_EUNSUPPORTED;
  const int units = d_out / Q;
  g.n_cta = units < n_cta_max ? units : n_cta_max;
  g.cta0 = 0;
  g.x_pf = 1;
  out->grid = g.n_cta;
  out->gp = g;
  return DECDEC_OK;
}

struct WsLayout {
  size_t cnt, ob, total;
};
// workspace: reserved head (16 KB), then o_b (fp32, d_out; self-validating, see ptx.cuh kObEmpty)
WsLayout ws_layout(int k, int d_out) {
  (void)k;
  WsLayout w{};
  w.cnt = 0;
  w.ob = align_up((size_t)kCntSlots * 4);
  w.total = w.ob + align_up((size_t)d_out * 4);
  return w;
}

decdec_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return DECDEC_OK;
  fprintf(stderr, "[decdec] CUDA error: %s\n", cudaGetErrorString(e));
  return DECDEC_ECUDA;
}

template <typename K>
decdec_status set_smem_attr(K kern, size_t bytes) {
  return cuda_status(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

// Kernel attributes (max dynamic smem) are per device: initialise once per device.
constexpr int kMaxDevices = 64;
std::mutex g_attr_mu;
int g_attr_done[kMaxDevices] = {0};
decdec_status g_attr_status[kMaxDevices];
decdec_status init_attrs() {
  decdec_status s = DECDEC_OK;
  const size_t lin = 226 * 1024;  // + static smem <= 227 KB
  if (s == DECDEC_OK) s = set_smem_attr(k_select, 80 * 1024);
  if (s == DECDEC_OK) s = set_smem_attr(k_linear<3, 4>, lin);
  if (s == DECDEC_OK) s = set_smem_attr(k_linear<4, 4>, lin);
  if (s == DECDEC_OK) s = set_smem_attr(k_linear<3, 16>, lin);
  if (s == DECDEC_OK) s = set_smem_attr(k_linear<4, 16>, lin);
  if (s == DECDEC_OK) s = set_smem_attr(k_linear<4, 4, 3>, lin);
  if (s == DECDEC_OK) s = set_smem_attr(k_linear<4, 4, 4>, lin);
  if (s == DECDEC_OK) s = set_smem_attr(k_linear<3, 4, 0, 1>, lin);
  if (s == DECDEC_OK) s = set_smem_attr(k_linear<4, 4, 0, 1>, lin);
  if (s == DECDEC_OK) s = set_smem_attr(k_gemv16<3, 0>, kGemvSmemBudget + 1024);
  if (s == DECDEC_OK) s = set_smem_attr(k_gemv16<4, 0>, kGemvSmemBudget + 1024);
  if (s == DECDEC_OK) s = set_smem_attr(k_gemv16<3, 1>, kGemvSmemBudget + 1024);
  if (s == DECDEC_OK) s = set_smem_attr(k_gemv16<4, 1>, kGemvSmemBudget + 1024);
  if (s == DECDEC_OK) s = set_smem_attr(k_gemv16<4, 0, 3>, kGemvSmemBudget + 1024);
  if (s == DECDEC_OK) s = set_smem_attr(k_gemv16<4, 0, 4>, kGemvSmemBudget + 1024);
  return s;
}
decdec_status ensure_attrs() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return DECDEC_ECUDA;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (!g_attr_done[dev]) {
    g_attr_status[dev] = init_attrs();
    g_attr_done[dev] = 1;
  }
  return g_attr_status[dev];
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}
bool is_host_mapped(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer != nullptr;
}

decdec_status check_layer(const decdec_layer* L, bool need_residual) {
  if (!L) return DECDEC_EINVAL;
  if (L->group_size != DECDEC_GROUP) return DECDEC_EUNSUPPORTED;
  if (L->w_bits != 3 && L->w_bits != 4) return DECDEC_EUNSUPPORTED;
  if (L->w_format != DECDEC_WFMT_UNIFORM && L->w_format != DECDEC_WFMT_LUT) return DECDEC_EUNSUPPORTED;
  if (L->d_in < 128 || L->d_in > 32768 || L->d_in % DECDEC_GROUP) return DECDEC_EINVAL;
  if (L->d_out < 32 || L->d_out % 32) return DECDEC_EINVAL;
  if (L->w_format == DECDEC_WFMT_LUT) {
    if (!L->w_packed || !L->w_lut) return DECDEC_EINVAL;
    if (!aligned16(L->w_packed) || !aligned16(L->w_lut)) return DECDEC_EALIGN;
    if (!is_device_ptr(L->w_packed) || !is_device_ptr(L->w_lut)) return DECDEC_EINVAL;
    if (need_residual && L->r_bits != 4) return DECDEC_EUNSUPPORTED;  // LUT base: r4 residual only
  } else {
    if (!L->w_packed || !L->w_scales || !L->w_zeros) return DECDEC_EINVAL;
    if (!aligned16(L->w_packed) || !aligned16(L->w_scales) || !aligned16(L->w_zeros)) return DECDEC_EALIGN;
    if (!is_device_ptr(L->w_packed) || !is_device_ptr(L->w_scales) || !is_device_ptr(L->w_zeros)) return DECDEC_EINVAL;
  }
  if (need_residual) {
    if (L->r_bits != 4 && L->r_bits != 16) return DECDEC_EUNSUPPORTED;
    if (!L->r_rows || (L->r_bits == 4 && !L->r_scales)) return DECDEC_EINVAL;
    if (!aligned16(L->r_rows) || (L->r_bits == 4 && !aligned16(L->r_scales))) return DECDEC_EALIGN;
    if (!is_host_mapped(L->r_rows) || (L->r_bits == 4 && !is_host_mapped(L->r_scales))) return DECDEC_ENOTMAPPED;
  }
  return DECDEC_OK;
}

int n_selected(int d_in, int k, int chunk) {
  if (k < 0 || d_in <= 0) return -1;
  if (chunk == 0) return k <= d_in ? k : -1;
  if (chunk < 32 || chunk > 32768 || chunk % 8 || k > chunk) return -1;
  const int full = d_in / chunk, rem = d_in % chunk;
  return full * k + (rem < k ? rem : k);
}

decdec_status launch_select(const uint16_t* x, int d_in, int k, int chunk, int* idx, uint16_t* xs, int* sel,
                            cudaStream_t st) {
  const int n = chunk ? (chunk < d_in ? chunk : d_in) : d_in;
  const int nseg = chunk ? (d_in + chunk - 1) / chunk : 1;
  int nt = (n / 8 + 31) / 32 * 32;
  if (nt > 1024) nt = 1024;
  k_select<<<nseg, nt, select_block_smem_bytes(n), st>>>(x, d_in, k, chunk, idx, xs, sel);
  return cuda_status(cudaGetLastError());
}

// Liveness: a compensated launch's DEC CTAs wait for o_b entries written by GEMV CTAs of the
// same grid, so all of its CTAs must be co-resident.  The grid is <= one CTA per SM, and it is
// launched COOPERATIVELY: the runtime then co-schedules the whole grid or fails the launch (it
// never leaves a partially resident grid spinning), also when other streams hold SMs.  Measured
// with PDL inside graphs (csrc/probe/probe_coop.cu, profiles/r02_probe_coop.json): legal, and a
// cooperative grid still starts early when it fits beside the previous kernel.  DECDEC_COOP=0
// disables it (A/B only).
bool coop_launch() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("DECDEC_COOP");
    env = e ? (atoi(e) > 0) : 1;
  }
  return env == 1;
}

template <int BITS, int RBITS, int LUTB = 0, int MLF = 0>
decdec_status launch_linear_t(const LinearParams& p, const Plan& pl, bool pdl, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(32 * (1 + pl.NC));
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  // cooperative: DEC CTAs wait for GEMV CTAs of the same grid; the fused P2P all-gather's
  // leader waits for the other CTAs' signals
  if ((p.k_sel > 0 && coop_launch()) || (p.pp.active && p.pp.wait_self)) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cuda_status(cudaLaunchKernelEx(&cfg, k_linear<BITS, RBITS, LUTB, MLF>, p));
}

decdec_status launch_linear(const LinearParams& p, const Plan& pl, int bits, int rbits, bool pdl, cudaStream_t st,
                            int lut_bits = 0) {
  if (p.share_n > 1) {  // multi-link residual fetch (uniform base, r4 residual)
    if (lut_bits || rbits != 4) return DECDEC_EUNSUPPORTED;
    return bits == 3 ? launch_linear_t<3, 4, 0, 1>(p, pl, pdl, st) : launch_linear_t<4, 4, 0, 1>(p, pl, pdl, st);
  }
  if (lut_bits == 3) return launch_linear_t<4, 4, 3>(p, pl, pdl, st);  // LUT base: W4K nibbles, r4 residual
  if (lut_bits == 4) return launch_linear_t<4, 4, 4>(p, pl, pdl, st);
  if (bits == 3) return rbits == 16 ? launch_linear_t<3, 16>(p, pl, pdl, st) : launch_linear_t<3, 4>(p, pl, pdl, st);
  return rbits == 16 ? launch_linear_t<4, 16>(p, pl, pdl, st) : launch_linear_t<4, 4>(p, pl, pdl, st);
}

decdec_status launch_gemv(const GemvPlan& pl, int bits, bool pdl, cudaStream_t st, int lut_bits = 0) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(32 * (1 + pl.gp.NC));
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  const bool pair = gemv_pair();
  cudaError_t e;
  if (lut_bits) e = lut_bits == 3 ? cudaLaunchKernelEx(&cfg, k_gemv16<4, 0, 3>, pl.gp) : cudaLaunchKernelEx(&cfg, k_gemv16<4, 0, 4>, pl.gp);
  else if (pair) e = bits == 3 ? cudaLaunchKernelEx(&cfg, k_gemv16<3, 1>, pl.gp) : cudaLaunchKernelEx(&cfg, k_gemv16<4, 1>, pl.gp);
  else e = bits == 3 ? cudaLaunchKernelEx(&cfg, k_gemv16<3, 0>, pl.gp) : cudaLaunchKernelEx(&cfg, k_gemv16<4, 0>, pl.gp);
  return cuda_status(e);
}

// DECDEC_STACK_FIT: 0 = off, else the least % of a compensated layer's planned GEMV CTAs kept when
// its grid is shrunk to fit beside the previous layer's DEC CTAs (stack_create)
int stack_fit() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("DECDEC_STACK_FIT");
    env = e ? atoi(e) : 50;
    if (env < 0) env = 0;
  }
  return env;
}

// DECDEC_STACK_FIT_RMIN (x100): the least PCIe/HBM roofline ratio of a call the fit applies to
double stack_fit_rmin() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("DECDEC_STACK_FIT_RMIN");
    env = e ? atoi(e) : 0;  // measured: 0 (the time model alone) vs 2.0: k_chunk 1 -2.6 %, 4 -2.2 %,
    if (env < 0) env = 0;   // 8 -1.6 %, 12/21 +-0.6 % (the small layers' GEMV hides under the
  }                         // compensation latency at any k)
  return env / 100.0;
}

// DECDEC_L2PF_NEXT=1 enables the stack executor's cross-layer L2 prefetch (A/B only)
bool l2_next_prefetch() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("DECDEC_L2PF_NEXT");
    env = e ? (atoi(e) > 0) : 0;  // measured: no gain (k_chunk 0 step 1.327 -> 1.384 ms with it)
  }
  return env == 1;
}

// Uniform-weight k = 0 calls run the fused kernel's GEMV CTAs (k_linear with no DEC CTAs) by
// default; DECDEC_NEW_GEMV=1 routes them through gemv.cuh's k_gemv16 instead.  Measured (1x B200,
// Llama-3-8B 3-bit k_chunk-0 step, profiles/r02_gemv_ab.json): k_linear 1.078 ms; k_gemv16
// 1.25-1.32 ms (dedicated or in-warp producer, single rows or pairs, 16-96 KB before the wait),
// two-CTAs-per-SM k_gemv 1.44-1.51 ms.  LUT (non-uniform) layers always use k_gemv16.
// LUT-base k = 0 calls: the fused kernel's GEMV CTAs or k_gemv16.  Measured (Llama-3-8B k_chunk-0
// step, 1x B200, profiles/r02_experiments.json): 3-bit tables 1.443 ms fused vs 1.586 ms k_gemv16;
// 4-bit tables 2.252 vs 2.118 (k_linear<4,4,4> spills its table planes).  DECDEC_LUT_GEMV16=0|1
// forces one kernel for both widths.
bool lut_gemv16(int lutb) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("DECDEC_LUT_GEMV16");
    env = e ? (atoi(e) > 0) : -1;
  }
  return env >= 0 ? env == 1 : lutb == 4;
}

bool use_gemv_kernel() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("DECDEC_NEW_GEMV");
    env = (e && atoi(e) > 0) ? 1 : 0;
  }
  return env == 1;
}

LinearParams base_params(const decdec_layer* L, const uint16_t* x, uint16_t* y, const Plan& pl) {
  LinearParams p{};
  const bool lut = L->w_format == DECDEC_WFMT_LUT;
  p.w = static_cast<const uint8_t*>(L->w_packed);
  p.ws = lut ? L->w_lut : L->w_scales;  // LUT base: the rows' tables travel in the scales' place
  p.wz = lut ? nullptr : L->w_zeros;
  p.x = x;
  p.y = y;
  p.d_in = L->d_in;
  p.d_out = L->d_out;
  p.G = pl.G;
  p.row_bytes = L->d_in * (lut ? 4 : L->w_bits) / 8;
  p.TR = pl.TR;
  p.NKW = pl.NKW;
  p.NSLOTS = pl.NSLOTS;
  p.RPS = pl.RPS;
  p.NC = pl.NC;
  p.stages = pl.stages;
  p.n_tiles = pl.n_tiles;
  p.stage_bytes = pl.stage_bytes;
  p.off_s = pl.off_s;
  p.off_z = pl.off_z;
  p.n_dec = pl.n_dec;
  p.off_sel = pl.off_sel;
  p.off_part = pl.off_part;
  p.off_rsc = pl.off_rsc;
  p.off_stage = pl.off_stage;
  p.off_x = pl.off_x;
  p.trace = g_trace ? g_trace + 2 : nullptr;
  p.dbg_idx = g_dbg_idx;
  p.dbg_xs = g_dbg_xs;
  p.dbg_cap = g_dbg_cap;
  p.dbg_ctas = g_dbg_ctas;
  static int env_prefetch = -1;
  if (env_prefetch < 0) {
    const char* e = getenv("DECDEC_PREFETCH");
    env_prefetch = e ? atoi(e) : 8;
  }
  p.prefetch = env_prefetch;
  static int env_l2pf = -1;
  if (env_l2pf < 0) {
    const char* e = getenv("DECDEC_L2PF");
    env_l2pf = e ? atoi(e) : 0;
  }
  p.l2pf = env_l2pf;
  static int env_xpf = -1;
  if (env_xpf < 0) {
    const char* e = getenv("DECDEC_XPF");
    env_xpf = e ? atoi(e) : 1;
  }
  p.x_pf = env_xpf;
  return p;
}

}  // namespace

extern "C" {

size_t decdec_workspace_bytes(int32_t max_k, int32_t max_d_out) {
  if (max_k < 0 || max_d_out < 0) return 0;
  return ws_layout(max_k, max_d_out).total;
}

decdec_status decdec_workspace_init(void* ws, size_t ws_bytes, decdec_stream_t stream) {
  const size_t head = ws_layout(0, 0).ob;
  if (!ws || ws_bytes < head) return DECDEC_EINVAL;
  cudaError_t e = cudaMemsetAsync(ws, 0, head, (cudaStream_t)stream);
  if (e == cudaSuccess && ws_bytes > head)  // o_b entries = kObEmpty (0xFFFFFFFF)
    e = cudaMemsetAsync(static_cast<uint8_t*>(ws) + head, 0xFF, ws_bytes - head, (cudaStream_t)stream);
  return cuda_status(e);
}

int32_t decdec_num_selected(int32_t d_in, int32_t k, int32_t chunk) { return n_selected(d_in, k, chunk); }

decdec_status decdec_select(const uint16_t* x, int32_t d_in, int32_t k, int32_t chunk, int32_t* idx, uint16_t* xs,
                            decdec_stream_t stream) {
  if (!x || !idx || !xs) return DECDEC_EINVAL;
  if (d_in <= 0 || d_in > 32768 || d_in % 8) return DECDEC_EINVAL;  // the selector reads x as 16-B chunks
  if (n_selected(d_in, k, chunk) < 0) return DECDEC_EINVAL;
  if (!aligned16(x) || (reinterpret_cast<uintptr_t>(idx) & 3u) || (reinterpret_cast<uintptr_t>(xs) & 1u))
    return DECDEC_EALIGN;
  decdec_status s = ensure_attrs();
  if (s != DECDEC_OK) return s;
  if (k == 0) return DECDEC_OK;
  return launch_select(x, d_in, k, chunk, idx, xs, nullptr, (cudaStream_t)stream);
}

decdec_status decdec_gemv(const decdec_layer* L, const uint16_t* x, uint16_t* y, void* ws, size_t ws_bytes,
                          decdec_stream_t stream) {
  (void)ws;
  (void)ws_bytes;
  decdec_status s = check_layer(L, false);
  if (s != DECDEC_OK) return s;
  if (!x || !y) return DECDEC_EINVAL;
  if (!aligned16(x) || !aligned16(y)) return DECDEC_EALIGN;
  if ((s = ensure_attrs()) != DECDEC_OK) return s;
  const int lutb = L->w_format == DECDEC_WFMT_LUT ? L->w_bits : 0;
  if (use_gemv_kernel() || (lutb && lut_gemv16(lutb))) {
    GemvPlan gpl;
    if ((s = make_gemv_plan(L->d_in, L->d_out, L->w_bits, device_sms(), &gpl, lutb)) != DECDEC_OK) return s;
    gpl.gp.w = static_cast<const uint8_t*>(L->w_packed);
    gpl.gp.ws = lutb ? L->w_lut : L->w_scales;
    gpl.gp.wz = lutb ? nullptr : L->w_zeros;
    gpl.gp.x = x;
    gpl.gp.y = y;
    gpl.gp.trace = g_trace ? g_trace + 2 : nullptr;
    return launch_gemv(gpl, L->w_bits, false, (cudaStream_t)stream, lutb);
  }
  Plan pl;
  if ((s = make_plan(L->d_in, L->d_out, L->w_bits, 0, &pl, 0, 4, lutb)) != DECDEC_OK) return s;
  LinearParams p = base_params(L, x, y, pl);
  return launch_linear(p, pl, L->w_bits, 4, false, (cudaStream_t)stream, lutb);
}

}  // extern "C"

namespace {

// Validated, planned launch of one layer (no CUDA API calls except the launches), so it
// can run inside stream capture.
struct Prepared {
  LinearParams p;
  Plan pl;
  bool gemv;  // k = 0: the base GEMV kernel (gemv.cuh)
  int lut_bits;
  GemvPlan gpl;
  int k, chunk, bits, rbits;
  const uint16_t* x;
  int32_t* sel;
};

decdec_status prepare_linear(const decdec_layer* L, const uint16_t* x, int32_t k, int32_t chunk, uint16_t* y,
                             int32_t* sel, void* ws, size_t ws_bytes, Prepared* out) {
  decdec_status s = check_layer(L, k > 0);
  if (s != DECDEC_OK) return s;
  if (!x || !y) return DECDEC_EINVAL;
  if (!aligned16(x) || !aligned16(y)) return DECDEC_EALIGN;
  const int k_sel = n_selected(L->d_in, k, chunk);
  if (k_sel < 0) return DECDEC_EINVAL;
  if ((s = ensure_attrs()) != DECDEC_OK) return s;
  Prepared P{};
  const int lutb = L->w_format == DECDEC_WFMT_LUT ? L->w_bits : 0;
  if (k_sel == 0 && (use_gemv_kernel() || (lutb && lut_gemv16(lutb)))) {
    if ((s = make_gemv_plan(L->d_in, L->d_out, L->w_bits, device_sms(), &P.gpl, lutb)) != DECDEC_OK) return s;
    GemvParams& g = P.gpl.gp;
    g.w = static_cast<const uint8_t*>(L->w_packed);
    g.ws = lutb ? L->w_lut : L->w_scales;
    g.wz = lutb ? nullptr : L->w_zeros;
    P.lut_bits = lutb;
    g.x = x;
    g.y = y;
    g.ob = nullptr;
    g.trace = g_trace ? g_trace + 2 : nullptr;
    P.gemv = true;
    P.k = k;
    P.chunk = chunk;
    P.bits = L->w_bits;
    P.rbits = L->r_bits;
    P.x = x;
    P.sel = sel;
    *out = P;
    return DECDEC_OK;
  }
  const int sel_len = chunk ? (chunk < L->d_in ? chunk : L->d_in) : L->d_in;
  if ((s = make_plan(L->d_in, L->d_out, L->w_bits, k_sel, &P.pl, sel_len, L->r_bits, lutb)) != DECDEC_OK)
    return s;
  P.p = base_params(L, x, y, P.pl);
  P.lut_bits = lutb;
  P.k = k;
  P.chunk = chunk;
  P.bits = L->w_bits;
  P.rbits = L->r_bits;
  P.x = x;
  P.sel = sel;
  if (k_sel > 0) {
    if (!ws) return DECDEC_EINVAL;
    const WsLayout wl = ws_layout(k_sel, L->d_out);
    if (wl.total > ws_bytes) return DECDEC_ESPACE;
    if (!aligned16(ws)) return DECDEC_EALIGN;
    uint8_t* base = static_cast<uint8_t*>(ws);
    LinearParams& p = P.p;
    p.k_sel = k_sel;
    p.r_rows = static_cast<const uint8_t*>(L->r_rows);
    p.r_scales = L->r_scales;
    p.r_row_bytes = L->d_out * L->r_bits / 8;
    p.ob = reinterpret_cast<float*>(base + wl.ob);
    p.k_req = k;
    p.chunk = chunk;
    p.sel_out = sel;
    p.n_seg = P.pl.n_seg;
    p.rpi = P.pl.rpi;
    p.gws = P.pl.gws;
    p.nparts = P.pl.nparts;
    p.one_seg = P.pl.one_seg;
    p.early_reads = P.pl.early_reads;
    p.early_cap = P.pl.early_cap;
  }
  *out = P;
  return DECDEC_OK;
}

decdec_status enqueue_linear(const Prepared& P, cudaStream_t st, bool chained = false) {
  if (P.gemv) return launch_gemv(P.gpl, P.bits, chained, st, P.lut_bits);
  Plan pl = P.pl;
  pl.grid += P.pl.n_dec;  // DEC CTAs first
  return launch_linear(P.p, pl, P.bits, P.p.k_sel ? P.rbits : 4, chained, st, P.lut_bits);
}

// This rank's shard pointer inside the user area of its peer region (decdec_linear_p2p).
uint16_t* p2p_shard(const decdec_peers* pe, int q, size_t y_off, int d_out) {
  return reinterpret_cast<uint16_t*>(static_cast<uint8_t*>(pe->base[q]) + decdec::kFlagBytes + y_off) +
         (size_t)pe->rank * d_out;
}

decdec_status check_p2p(const decdec_layer* L, const decdec_peers* pe, size_t y_off, int slot) {
  if (!L || !pe || pe->nranks < 1) return DECDEC_EINVAL;
  if (slot < 0 || slot >= decdec::kFlagSlots || (y_off & 15)) return DECDEC_EINVAL;
  if (y_off + (size_t)pe->nranks * L->d_out * 2 > pe->user_bytes) return DECDEC_ESPACE;
  return DECDEC_OK;
}

// Fused all-gather parameters of a prepared layer call (p2p.cuh).
decdec_status fill_p2p(Prepared* P, const decdec_layer* L, const decdec_peers* pe, size_t y_off, int slot) {
  if (P->gemv) return DECDEC_EUNSUPPORTED;  // LUT base / DECDEC_NEW_GEMV: k_gemv16 has no exchange epilogue
  decdec::P2PParams& pp = P->p.pp;
  pp.active = 1;
  pp.nranks = pe->nranks;
  pp.n_writers = P->p.k_sel > 0 ? P->pl.n_dec : P->pl.grid;  // DEC CTAs (combine) or GEMV CTAs write y
  pp.leader = 0;
  pp.wait_self = 1;  // standalone call: returns with y_full complete (stacks defer all but the last)
  pp.prev_flag = nullptr;
  for (int q = 0; q < pe->nranks; ++q) {
    pp.peer_y[q] = p2p_shard(pe, q, y_off, L->d_out);
    pp.peer_flag[q] = static_cast<unsigned int*>(pe->base[q]) + (size_t)slot * decdec::kFlagStrideWords;
  }
  pp.my_flag = pp.peer_flag[pe->rank];
  return DECDEC_OK;
}

}  // namespace

struct decdec_stack {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int n_layers = 0, n_kernels = 0;
};

extern "C" {

decdec_status decdec_linear(const decdec_layer* L, const uint16_t* x, int32_t k, int32_t chunk, uint16_t* y,
                            int32_t* sel, void* ws, size_t ws_bytes, decdec_stream_t stream) {
  Prepared P;
  decdec_status s = prepare_linear(L, x, k, chunk, y, sel, ws, ws_bytes, &P);
  if (s != DECDEC_OK) return s;
  return enqueue_linear(P, (cudaStream_t)stream);
}

}  // extern "C"

namespace {

// comm == nullptr: single-GPU stack; otherwise layer i writes y[i] + rank*d_out_r and is
// followed by the in-place all-gather of y[i].
decdec_status stack_create(const decdec_layer* layers, int32_t n_layers, const int32_t* k, int32_t chunk,
                           const uint16_t* const* x, uint16_t* const* y, void* ws, size_t ws_bytes,
                           decdec_comm* comm, decdec_stack** out, decdec_peers* peers = nullptr,
                           const size_t* y_off = nullptr) {
  if (!layers || n_layers <= 0 || !k || !x || !out) return DECDEC_EINVAL;
  if (peers ? (!y_off || n_layers > decdec::kFlagSlots || peers->nranks < 1) : !y) return DECDEC_EINVAL;
  *out = nullptr;
  if (g_trace && g_trace_bytes < (2 + (size_t)n_layers * kTraceStride) * 8) return DECDEC_ESPACE;
  const int rank = comm ? tp_rank(comm) : 0;
  const bool gather = comm && decdec_comm_nranks(comm) > 1;
  Prepared* P = new Prepared[n_layers];
  decdec_status s = DECDEC_OK;
  int n_kernels = 0;
  for (int i = 0; i < n_layers && s == DECDEC_OK; ++i) {
    if (peers) {  // fused all-gather: layer i writes every rank's y_full at y_off[i], slot i
      s = check_p2p(&layers[i], peers, y_off[i], i);
      if (s == DECDEC_OK)
        s = prepare_linear(&layers[i], x[i], k[i], chunk, p2p_shard(peers, peers->rank, y_off[i], layers[i].d_out),
                           nullptr, ws, ws_bytes, &P[i]);
      if (s == DECDEC_OK) s = fill_p2p(&P[i], &layers[i], peers, y_off[i], i);
      if (s == DECDEC_OK) {  // only the last layer returns with its y_full complete; layer i > 0
        decdec::P2PParams& pp = P[i].p.pp;  // first waits for layer i - 1's (deferred wait)
        pp.wait_self = i == n_layers - 1;
        if (i > 0) pp.prev_flag = static_cast<unsigned int*>(peers->base[peers->rank]) + (size_t)(i - 1) * decdec::kFlagStrideWords;
      }
    } else {
      uint16_t* yi = y[i] ? y[i] + (size_t)rank * layers[i].d_out : nullptr;
      s = prepare_linear(&layers[i], x[i], k[i], chunk, yi, nullptr, ws, ws_bytes, &P[i]);
    }
    // debug timelines: one trace region per layer (decdec_debug_trace buffer must hold them)
    if (g_trace) {
      P[i].p.trace = g_trace + 2 + (size_t)i * kTraceStride;
      P[i].gpl.gp.trace = g_trace + 2 + (size_t)i * kTraceStride;
    }
    n_kernels += 1;
  }
  if (s != DECDEC_OK) {
    delete[] P;
    return s;
  }
  // A compensated layer's launch is cooperative: the whole grid must be resident at once, so a
  // 148-CTA grid waits until the previous layer's DEC CTAs (still combining) have left.  Shrinking
  // its GEMV CTAs to fit beside them lets it launch -- and run its prologue -- while the previous
  // layer finishes.  Only where the GEMV has slack (time model below), and not below stack_fit()
  // % of the planned GEMV CTAs.  Measured (1x B200, alternating runs): Llama-3-8B k_chunk 21
  // -7 %, 12 -6 %, 4 -2 % vs no fit (profiles/r02_s3_experiments.json).  DECDEC_STACK_FIT=0
  // turns it off (A/B).
  if (stack_fit() > 0 && n_layers > 1) {
    const int sms = device_sms();
    for (int i = 0; i < n_layers; ++i) {
      Prepared& Q = P[i];
      if (Q.gemv || Q.p.k_sel == 0 || Q.pl.r_ratio < stack_fit_rmin()) continue;
      const Prepared& Pv = P[(i + n_layers - 1) % n_layers];  // the graph replays cyclically
      const int prev_dec = (Pv.gemv || Pv.p.k_sel == 0) ? 0 : Pv.pl.n_dec;
      const int cap = sms - prev_dec - Q.pl.n_dec;
      if (Q.pl.grid <= cap || cap * 100 < stack_fit() * Q.pl.grid) continue;
      // and only if the shrunk GEMV still hides under the compensation: GEMV time modelled from
      // the HBM roofline at ~60 % efficiency x the lanes a row team uses (3-bit decode is issue
      // bound; G = 40 teams idle 24 of 64 lanes), compensation time from the PCIe roofline at
      // ~75 % + ~4 us fixed (§6c); keep 20 % margin.  Phi-3's gate/up layer (G = 40) fails it:
      // fitted, it turned the Phi-3 k_chunk-21 step 11 % slower.
      const double lane_eff = Q.pl.NKW ? (double)Q.pl.G / (32.0 * Q.pl.NKW) : 1.0;
      const double t_gemv = Q.pl.t_hbm_us / (0.6 * lane_eff * cap / sms);
      const double t_dec = Q.pl.t_hbm_us * Q.pl.r_ratio / 0.75 + 4.0;
      if (t_gemv <= 0.8 * t_dec) Q.pl.grid = cap;
    }
  }
  if (l2_next_prefetch() && n_layers > 1) {
    for (int i = 0; i < n_layers; ++i) {
      if (!P[i].gemv) continue;
      const decdec_layer& Ln = layers[(i + 1) % n_layers];
      if (Ln.w_format != DECDEC_WFMT_UNIFORM) continue;
      const int Gn = Ln.d_in / DECDEC_GROUP;
      GemvParams& g = P[i].gpl.gp;
      g.pf_ptr[0] = static_cast<const uint8_t*>(Ln.w_packed);
      g.pf_bytes[0] = (uint32_t)((size_t)Ln.d_out * Ln.d_in * Ln.w_bits / 8);
      g.pf_ptr[1] = reinterpret_cast<const uint8_t*>(Ln.w_scales);
      g.pf_bytes[1] = (uint32_t)((size_t)Ln.d_out * Gn * 2);
      g.pf_ptr[2] = Ln.w_zeros;
      g.pf_bytes[2] = (uint32_t)((size_t)Ln.d_out * Gn);
    }
  }
  cudaStream_t st = nullptr;
  cudaError_t e0 = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e0 != cudaSuccess) {
    delete[] P;
    return cuda_status(e0);
  }
  if (gather) {
    // NCCL sets up connections / algorithm buffers lazily on a communicator's first
    // collectives: run each layer's all-gather once outside the capture (in place on y_full,
    // whose contents are overwritten by every replay anyway)
    for (int i = 0; i < n_layers && s == DECDEC_OK; ++i) s = tp_allgather(comm, y[i], layers[i].d_out, st);
    if (s == DECDEC_OK) s = cuda_status(cudaStreamSynchronize(st));
    if (s != DECDEC_OK) {
      cudaStreamDestroy(st);
      delete[] P;
      return s;
    }
  }
  decdec_stack* g = new decdec_stack();
  cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < n_layers && e == cudaSuccess && s == DECDEC_OK; ++i) {
    // PDL edges only between consecutive layer kernels (not across a collective)
    s = enqueue_linear(P[i], st, i > 0 && !gather);
    if (s == DECDEC_OK && gather) s = tp_allgather(comm, y[i], layers[i].d_out, st);
  }
  cudaGraph_t graph = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(st, &graph);
  cudaStreamDestroy(st);
  delete[] P;
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess && s == DECDEC_OK) e = cudaGraphInstantiate(&g->exec, graph, 0);
  g->graph = graph;
  g->n_layers = n_layers;
  g->n_kernels = n_kernels;
  if (e != cudaSuccess || s != DECDEC_OK) {
    decdec_stack_destroy(g);
    return s != DECDEC_OK ? s : cuda_status(e);
  }
  *out = g;
  return DECDEC_OK;
}

}  // namespace

extern "C" {

decdec_status decdec_stack_create(const decdec_layer* layers, int32_t n_layers, const int32_t* k, int32_t chunk,
                                  const uint16_t* const* x, uint16_t* const* y, void* ws, size_t ws_bytes,
                                  decdec_stream_t stream, decdec_stack** out) {
  (void)stream;  // capture runs on a private stream (the legacy NULL stream cannot capture)
  return stack_create(layers, n_layers, k, chunk, x, y, ws, ws_bytes, nullptr, out);
}

decdec_status decdec_stack_create_tp(const decdec_layer* layers, int32_t n_layers, const int32_t* k, int32_t chunk,
                                     const uint16_t* const* x, uint16_t* const* y_full, void* ws, size_t ws_bytes,
                                     decdec_comm* comm, decdec_stream_t stream, decdec_stack** out) {
  (void)stream;
  if (!comm) return DECDEC_EINVAL;
  return stack_create(layers, n_layers, k, chunk, x, y_full, ws, ws_bytes, comm, out);
}

decdec_status decdec_stack_create_p2p(const decdec_layer* layers, int32_t n_layers, const int32_t* k, int32_t chunk,
                                      const uint16_t* const* x, const size_t* y_off, void* ws, size_t ws_bytes,
                                      decdec_peers* peers, decdec_stream_t stream, decdec_stack** out) {
  (void)stream;
  if (!peers) return DECDEC_EINVAL;
  return stack_create(layers, n_layers, k, chunk, x, nullptr, ws, ws_bytes, nullptr, out, peers, y_off);
}

decdec_status decdec_linear_p2p(const decdec_layer* L, const uint16_t* x, int32_t k, int32_t chunk, size_t y_off,
                                int32_t slot, int32_t* sel, void* ws, size_t ws_bytes, decdec_peers* peers,
                                decdec_stream_t stream) {
  decdec_status s = check_p2p(L, peers, y_off, slot);
  if (s != DECDEC_OK) return s;
  Prepared P;
  s = prepare_linear(L, x, k, chunk, p2p_shard(peers, peers->rank, y_off, L->d_out), sel, ws, ws_bytes, &P);
  if (s != DECDEC_OK) return s;
  if ((s = fill_p2p(&P, L, peers, y_off, slot)) != DECDEC_OK) return s;
  return enqueue_linear(P, (cudaStream_t)stream);
}

size_t decdec_ml_bytes(int32_t d_out, int32_t nranks) {
  if (d_out <= 0 || nranks < 1) return 0;
  return align_up(512 + (size_t)(nranks - 1) * d_out * 4, 256);
}

decdec_status decdec_linear_ml(const decdec_layer* L, const uint16_t* x, int32_t k, int32_t chunk, uint16_t* y,
                               int32_t* sel, void* ws, size_t ws_bytes, decdec_peers* peers, size_t ml_off,
                               decdec_stream_t stream) {
  if (!L || !peers || peers->nranks < 1) return DECDEC_EINVAL;
  const int rank = peers->rank, P = peers->nranks;
  if (ml_off & 15) return DECDEC_EINVAL;
  if (ml_off + decdec_ml_bytes(L->d_out, P) > peers->user_bytes) return DECDEC_ESPACE;
  if (P == 1 || rank == 0) {
    if (!y) return DECDEC_EINVAL;
  }
  Prepared Pp;
  // a helper has no output of its own: its (never written) y is the workspace head
  decdec_status s = prepare_linear(L, x, k, chunk, rank == 0 ? y : static_cast<uint16_t*>(ws), rank == 0 ? sel : nullptr,
                                   ws, ws_bytes, &Pp);
  if (s != DECDEC_OK) return s;
  if (P == 1 || Pp.gemv || Pp.p.k_sel == 0) {  // nothing to split: the main rank alone, as decdec_linear
    return rank == 0 ? enqueue_linear(Pp, (cudaStream_t)stream) : DECDEC_OK;
  }
  if (Pp.pl.n_dec > 64) return DECDEC_EUNSUPPORTED;  // 64 flag / ack words per layer
  if (Pp.lut_bits || Pp.rbits != 4) return DECDEC_EUNSUPPORTED;  // built for the uniform base + r4
  auto user = [&](int q) { return static_cast<uint8_t*>(peers->base[q]) + decdec::kFlagBytes + ml_off; };
  LinearParams& p = Pp.p;
  p.share_n = P;
  p.share_r = rank;
  if (rank == 0) {
    p.ml_flag = reinterpret_cast<unsigned int*>(user(0));
    p.ml_in = reinterpret_cast<const float*>(user(0) + 512);
    for (int h = 1; h < P; ++h) p.ml_peer_ack[h - 1] = reinterpret_cast<unsigned int*>(user(h) + 256);
  } else {
    p.ml_out = reinterpret_cast<float*>(user(0) + 512) + (size_t)(rank - 1) * L->d_out;
    p.ml_out_flag = reinterpret_cast<unsigned int*>(user(0));
    p.ml_ack = reinterpret_cast<unsigned int*>(user(rank) + 256);
    Pp.pl.grid = 0;  // DEC CTAs only: no base GEMV on a helper
  }
  return enqueue_linear(Pp, (cudaStream_t)stream);
}

decdec_status decdec_stack_launch(decdec_stack* g, decdec_stream_t stream) {
  if (!g || !g->exec) return DECDEC_EINVAL;
  return cuda_status(cudaGraphLaunch(g->exec, (cudaStream_t)stream));
}

int32_t decdec_stack_kernels(const decdec_stack* g) { return g ? g->n_kernels : -1; }

void decdec_stack_destroy(decdec_stack* g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
}

decdec_status decdec_debug_unpack_weights(const decdec_layer* L, uint8_t* q_out, decdec_stream_t stream) {
  decdec_status s = check_layer(L, false);
  if (s != DECDEC_OK) return s;
  if (!q_out) return DECDEC_EINVAL;
  const int blocks = 4 * device_sms();
  if (L->w_bits == 3 && L->w_format != DECDEC_WFMT_LUT)  // LUT codes are W4K nibbles
    k_debug_unpack<3><<<blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<const uint8_t*>(L->w_packed), L->d_in, L->d_out, q_out);
  else
    k_debug_unpack<4><<<blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<const uint8_t*>(L->w_packed), L->d_in, L->d_out, q_out);
  return cuda_status(cudaGetLastError());
}

decdec_status decdec_plan_string(const decdec_layer* L, int32_t k, char* buf, size_t buf_bytes) {
  if (!L || !buf) return DECDEC_EINVAL;
  const int k_sel = k;  // caller passes the selected count
  const int lutb = L->w_format == DECDEC_WFMT_LUT ? L->w_bits : 0;
  if (k_sel == 0 && (use_gemv_kernel() || (lutb && lut_gemv16(lutb)))) {
    GemvPlan g;
    decdec_status s = make_gemv_plan(L->d_in, L->d_out, L->w_bits, device_sms(), &g, lutb);
    if (s != DECDEC_OK) return s;
    snprintf(buf, buf_bytes,
             "{\"kernel\": \"k_gemv\", \"G\": %d, \"T\": %d, \"M\": %d, \"team_red\": %d, \"RPS\": %d, \"TRS\": %d, "
             "\"Q\": %d, \"NC\": %d, \"stages\": %d, \"stage_bytes\": %u, \"grid\": %d, \"threads\": %d, \"smem\": %zu}",
             g.gp.G, g.gp.T, g.gp.M, g.gp.team_red, g.gp.RPS, g.gp.TRS, g.gp.Q, g.gp.NC, g.gp.stages, g.gp.stage_bytes,
             g.grid, 32 * (1 + g.gp.NC), g.smem);
    return DECDEC_OK;
  }
  Plan pl;
  decdec_status s = make_plan(L->d_in, L->d_out, L->w_bits, k_sel, &pl, 0, L->r_bits ? L->r_bits : 4, lutb);
  if (s != DECDEC_OK) return s;
  snprintf(buf, buf_bytes,
           "{\"G\": %d, \"NKW\": %d, \"NSLOTS\": %d, \"RPS\": %d, \"TR\": %d, \"NC\": %d, \"n_dec\": %d, "
           "\"stages\": %d, \"stage_bytes\": %u, \"n_tiles\": %d, \"grid\": %d, \"threads\": %d, \"smem\": %zu}",
           pl.G, pl.NKW, pl.NSLOTS, pl.RPS, pl.TR, pl.NC, pl.n_dec, pl.stages, pl.stage_bytes, pl.n_tiles, pl.grid,
           32 * (1 + pl.NC), pl.smem);
  return DECDEC_OK;
}

decdec_status decdec_set_dec_ctas(int32_t n) {
  if (n < 0 || n > 64) return DECDEC_EINVAL;
  g_dec_override = n;
  return DECDEC_OK;
}

int32_t decdec_launches_per_call(int32_t k) {
  (void)k;
  return 1;  // DEC CTAs (select + gather + combine) and GEMV CTAs run in one kernel
}

decdec_status decdec_debug_trace(void* buf, size_t bytes) {
  if (buf && bytes < (size_t)(2 + 1024 * kTraceEvents) * 8) return DECDEC_ESPACE;
  g_trace = static_cast<unsigned long long*>(buf);
  g_trace_bytes = buf ? bytes : 0;
  return DECDEC_OK;
}

decdec_status decdec_debug_selections(int32_t* idx, uint16_t* xs, int32_t cap, int32_t max_ctas) {
  if (!idx || !xs) {
    g_dbg_idx = nullptr;
    g_dbg_xs = nullptr;
    g_dbg_cap = g_dbg_ctas = 0;
    return DECDEC_OK;
  }
  if (cap <= 0 || max_ctas <= 0) return DECDEC_EINVAL;
  g_dbg_idx = idx;
  g_dbg_xs = xs;
  g_dbg_cap = cap;
  g_dbg_ctas = max_ctas;
  return DECDEC_OK;
}

}  // extern "C"
