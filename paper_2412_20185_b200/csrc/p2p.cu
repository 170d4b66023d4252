// Symmetric peer regions for the fused P2P-store all-gather (p2p.cuh, include/decdec.h
// "decdec_peers"): one device allocation per rank = [flag area | user area], exported with
// cudaIpcGetMemHandle and opened by every other rank (cudaIpcOpenMemHandle; NVLink peer
// mappings on a multi-GPU node, a second mapping of the same memory when ranks share a GPU).
// The handles travel over the caller's process group (plumbing); no NCCL.
#include <cuda_runtime.h>

#include <cstring>

#include "decdec.h"
#include "p2p.cuh"
#include "p2p_internal.h"

using decdec::kFlagBytes;
using decdec::kMaxPeers;

extern "C" {

decdec_status decdec_peers_create(size_t user_bytes, void* handle_out, decdec_peers** out) {
  if (!handle_out || !out) return DECDEC_EINVAL;
  *out = nullptr;
  decdec_peers* p = new decdec_peers();
  p->user_bytes = (user_bytes + 255) / 256 * 256;
  cudaError_t e = cudaMalloc(&p->base[0], kFlagBytes + p->user_bytes);
  if (e == cudaSuccess) e = cudaMemset(p->base[0], 0, kFlagBytes + p->user_bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p->base[0]);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (p->base[0]) cudaFree(p->base[0]);
    delete p;
    cudaGetLastError();
    return DECDEC_ECUDA;
  }
  p->local = p->base[0];
  std::memcpy(handle_out, &h, sizeof(h));
  *out = p;
  return DECDEC_OK;
}

decdec_status decdec_peers_connect(decdec_peers* p, int32_t rank, int32_t nranks, const void* handles) {
  if (!p || !handles || nranks < 1 || nranks > kMaxPeers || rank < 0 || rank >= nranks) return DECDEC_EINVAL;
  if (p->nranks) return DECDEC_EINVAL;  // connect once
  void* mapped[kMaxPeers] = {nullptr};
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) {
      mapped[q] = p->local;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const uint8_t*>(handles) + (size_t)q * DECDEC_IPC_HANDLE_BYTES, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(&mapped[q], h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int r = 0; r < q; ++r)
        if (r != rank && mapped[r]) cudaIpcCloseMemHandle(mapped[r]);
      cudaGetLastError();
      return DECDEC_ECUDA;
    }
  }
  for (int q = 0; q < nranks; ++q) p->base[q] = mapped[q];
  p->rank = rank;
  p->nranks = nranks;
  return DECDEC_OK;
}

void* decdec_peers_buffer(const decdec_peers* p) {
  return p ? static_cast<uint8_t*>(p->local) + kFlagBytes : nullptr;
}

size_t decdec_peers_buffer_bytes(const decdec_peers* p) { return p ? p->user_bytes : 0; }

void decdec_peers_destroy(decdec_peers* p) {
  if (!p) return;
  for (int q = 0; q < p->nranks; ++q)
    if (q != p->rank && p->base[q]) cudaIpcCloseMemHandle(p->base[q]);
  if (p->local) cudaFree(p->local);
  delete p;
}

}  // extern "C"
