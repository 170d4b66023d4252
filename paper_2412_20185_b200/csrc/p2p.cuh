// Fused P2P-store all-gather (BASELINE.json north_star "output
// assembled with an NCCL all-gather over NVLink" -- here the layer kernel itself does the
// exchange).  Every rank holds a symmetric device region (decdec_peers, p2p.cu): a flag area
// and a user area holding y_full buffers.  The layer kernel stores each fp16 output of its
// shard straight into EVERY rank's y_full (peer pointers opened through CUDA IPC: NVLink
// stores on a multi-GPU node); the writing CTAs of a rank count in locally and the last one
// releases one increment to every rank's per-layer flag; one leader CTA per rank waits
// (acquire, system scope) until its flag holds nranks increments -- i.e. every rank's shard has
// landed in its y_full -- resets it, and only then does the kernel complete.  No separate collective launch, no NCCL.
//
// Reset safety: a rank signals slot s of the next use only after finishing the layer before
// it, which needs every rank's signals for that layer, which this rank sends only after its
// own kernel for slot s completed (leader's reset included).  Slots are per layer of a stack.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace decdec {

constexpr int kMaxPeers = 8;
constexpr int kFlagSlots = 1024;       // per-layer completion counters of a peer region
constexpr int kFlagStrideWords = 32;   // 128 B per slot
constexpr size_t kFlagBytes = (size_t)kFlagSlots * kFlagStrideWords * 4;

struct P2PParams {
  int active;                       // the call belongs to a peer group: signal + leader wait (any nranks)
  int nranks;                       // 1 = no remote stores (plain y store)
  int n_writers;                    // CTAs of this kernel that store outputs (same on every rank)
  int leader;                       // blockIdx.x of the CTA that waits for the whole y_full
  uint16_t* peer_y[kMaxPeers];      // this rank's shard in rank q's y_full (peer_y[rank] = local)
  unsigned int* peer_flag[kMaxPeers];  // rank q's flag of this layer's slot
  unsigned int* my_flag;            // this rank's flag of the slot
  unsigned int* my_count;           // this rank's local arrival counter of the slot (next word)
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

// One thread of a writing CTA, after a barrier that orders all of the CTA's y stores before it.
// The CTAs of this rank count in on a local counter (gpu-scope release: cumulative over the
// barrier-ordered stores of the CTA's other threads); the LAST one (acquire) publishes the whole
// shard with ONE system-scope release to every rank's flag -- causality is transitive, so the
// other CTAs' peer stores are visible to a rank that acquires the flag.  One system-scope fence
// per rank per layer instead of one per CTA (measured: a per-CTA system release cost ~5 us per
// layer at k = 0 on 148 CTAs).
__device__ __forceinline__ void p2p_signal(const P2PParams& P) {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  const unsigned old = atomicAdd(P.my_count, 1u);
  if (old + 1u != (unsigned)P.n_writers) return;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  *P.my_count = 0u;  // re-armed: this rank's next arrivals on the slot come after this kernel
  for (int q = 0; q < P.nranks; ++q)
    asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(P.peer_flag[q]) : "memory");
}

// Leader CTA, one thread: every rank's shard has landed in this rank's y_full.  A peer that
// never signals (a rank died, mismatched call sequences) traps after ~20 s instead of hanging
// the GPU.
__device__ __forceinline__ void p2p_wait_all(const P2PParams& P) {

  const unsigned target = (unsigned)P.nranks;  // one release per rank
  unsigned v = 0;
  const unsigned long long t0 = globaltimer();
  while (true) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(P.my_flag) : "memory");
    if (v >= target) break;
    __nanosleep(64);
    if (globaltimer() - t0 > 20000000000ull) __trap();
  }
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(P.my_flag), "r"(0u) : "memory");
}

}  // namespace decdec
