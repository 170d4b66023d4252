// Fused P2P-store all-gather (BASELINE.json north_star "output
// assembled with an NCCL all-gather over NVLink" -- here the layer kernel itself does the
// exchange).  Every rank holds a symmetric device region (decdec_peers, p2p.cu): a flag area
// and a user area holding y_full buffers.  The layer kernel stores each fp16 output of its
// shard straight into EVERY rank's y_full (peer pointers opened through CUDA IPC: NVLink
// stores on a multi-GPU node).  Per layer slot three words: `flag` (incremented once per use by
// every rank, monotonic), `count` (this rank's CTAs counting in, reset per use) and `uses` (this
// rank's completed publications of the slot, monotonic).  The writing CTAs count in with a
// gpu-scope release; the rank's publication -- one system-scope fence, `uses` + 1 and an
// increment of every rank's flag -- is done by the last arriver, or by the leader CTA when the
// kernel itself must return with y_full complete (standalone calls, the last layer of a
// stack); that leader then acquires flag >= uses * nranks.  The other layers of a stack return
// at once and the NEXT layer's CTAs acquire the previous slot's flag before reading anything
// (deferred wait: the hand-off overlaps the next layer's launch and weight prefetch).  Counts
// never need resetting across uses, so no epoch or reset protocol is involved.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace decdec {

constexpr int kMaxPeers = 8;
constexpr int kFlagSlots = 1024;       // per-layer completion counters of a peer region
constexpr int kFlagStrideWords = 32;   // 128 B per slot
constexpr size_t kFlagBytes = (size_t)kFlagSlots * kFlagStrideWords * 4;

struct P2PParams {
  int active;                       // the call belongs to a peer group (any nranks)
  int nranks;                       // 1 = no remote stores (plain y store)
  int n_writers;                    // CTAs of this kernel that store outputs (same on every rank)
  int leader;                       // blockIdx.x of the leader CTA
  int wait_self;                    // 1: the kernel returns with y_full complete (leader waits)
  uint16_t* peer_y[kMaxPeers];      // this rank's shard in rank q's y_full (peer_y[rank] = local)
  unsigned int* peer_flag[kMaxPeers];  // rank q's flag of this layer's slot
  unsigned int* my_flag;            // this rank's slot: [0] flag, [1] count, [2] uses
  unsigned int* prev_flag;          // deferred wait: the previous layer's slot (or null)
};

__device__ __forceinline__ void p2p_store_u16(const P2PParams& P, uint16_t* y_local, int i, uint16_t v) {
  if (P.nranks <= 1) {
    y_local[i] = v;
    return;
  }
#pragma unroll 1
  for (int q = 0; q < P.nranks; ++q) P.peer_y[q][i] = v;
}

__device__ __forceinline__ void p2p_store_u4(const P2PParams& P, uint16_t* y_local, int i, uint4 v) {
  if (P.nranks <= 1) {
    *reinterpret_cast<uint4*>(y_local + i) = v;
    return;
  }
#pragma unroll 1
  for (int q = 0; q < P.nranks; ++q) *reinterpret_cast<uint4*>(P.peer_y[q] + i) = v;
}

// this rank's publication of the slot: one system-scope fence, uses + 1, every rank's flag + 1
__device__ __forceinline__ void p2p_publish(const P2PParams& P) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  P.my_flag[1] = 0u;                // count re-armed (this rank's next arrivals: a later kernel)
  P.my_flag[2] = P.my_flag[2] + 1u;  // uses
  for (int q = 0; q < P.nranks; ++q)
    asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(P.peer_flag[q]) : "memory");
}

__device__ __forceinline__ void p2p_wait_flag(const unsigned int* slot, unsigned target) {
  const unsigned long long t0 = globaltimer();
  unsigned v = 0;
  while (true) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(slot) : "memory");
    if ((int)(v - target) >= 0) break;  // monotonic (wrap-safe)
    __nanosleep(64);
    if (globaltimer() - t0 > 20000000000ull) __trap();  // a peer never arrived: fail, do not hang
  }
}

// One thread of a writing CTA, after a barrier that orders all of the CTA's y stores before it:
// count in (gpu-scope release, cumulative over the barrier-ordered stores of the CTA's other
// threads); without wait_self the last arriver publishes, with it the leader does -- after it
// has seen every local arrival -- and then waits for every rank.  Causality is transitive, so
// all of a rank's peer stores are visible to a rank that acquires its flag.  (One system-scope
// fence per rank per layer: a per-CTA system release cost ~5 us per layer at k = 0.)
__device__ __forceinline__ void p2p_signal(const P2PParams& P) {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  const unsigned old = atomicAdd(P.my_flag + 1, 1u);
  if (!P.wait_self) {
    if (old + 1u == (unsigned)P.n_writers) p2p_publish(P);
    return;
  }
  if ((int)blockIdx.x != P.leader) return;
  const unsigned long long t0 = globaltimer();
  while (*reinterpret_cast<volatile unsigned*>(P.my_flag + 1) != (unsigned)P.n_writers) {  // every local CTA
    __nanosleep(32);
    if (globaltimer() - t0 > 20000000000ull) __trap();
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  const unsigned uses = P.my_flag[2] + 1u;
  p2p_publish(P);
  p2p_wait_flag(P.my_flag, uses * (unsigned)P.nranks);
}

// Deferred wait, one thread per CTA of the next layer (after griddepcontrol.wait: the previous
// kernel, and its publication's `uses`, are complete on this rank).
__device__ __forceinline__ void p2p_wait_prev(const P2PParams& P) {
  if (!P.prev_flag) return;
  p2p_wait_flag(P.prev_flag, P.prev_flag[2] * (unsigned)P.nranks);
}

}  // namespace decdec
