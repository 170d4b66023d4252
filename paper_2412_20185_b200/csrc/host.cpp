// Offline host-side pieces of libdecdec: weight / residual packers (layouts of
// include/decdec.h, DESIGN.md ledger L6), the pinned + mapped residual host store
// (zero-copy source), status strings.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "decdec.h"

namespace {

// bit offset of channel c (0..7) inside an interleaved 8 x 4-bit word
constexpr int kW4Pos[8] = {0, 16, 4, 20, 8, 24, 12, 28};

// W3K table: for slice channel c -> (word, bit) of each of its 3 code bits.
struct W3Bit {
  unsigned char word, bit;
};
struct W3Table {
  W3Bit b[32][3];
  W3Table() {
    for (int c = 0; c < 32; ++c) {
      if (c < 30) {
        const int t = c / 10, r = c % 10, pos = 16 * (r & 1) + 3 * (r >> 1);
        for (int k = 0; k < 3; ++k) b[c][k] = {(unsigned char)t, (unsigned char)(pos + k)};
      } else {
        const int bit = 15 + 16 * (c - 30);
        for (int k = 0; k < 3; ++k) b[c][k] = {(unsigned char)k, (unsigned char)bit};
      }
    }
  }
};
const W3Table& w3_table() {
  static const W3Table t;
  return t;
}

std::mutex g_alloc_mu;
std::unordered_map<void*, std::pair<size_t, bool>> g_allocs;  // ptr -> (bytes, registered-mmap)

}  // namespace

extern "C" {

decdec_status decdec_pack_weights(const uint8_t* q, int32_t d_in, int32_t d_out, int32_t bits, void* out,
                                  size_t out_bytes) {
  if (!q || !out) return DECDEC_EINVAL;
  if (bits != 3 && bits != 4) return DECDEC_EUNSUPPORTED;
  if (d_in <= 0 || d_out <= 0 || d_in % 32) return DECDEC_EINVAL;
  const size_t row_words = (size_t)d_in * bits / 32;
  if (out_bytes < row_words * 4 * (size_t)d_out) return DECDEC_ESPACE;
  uint32_t* o = static_cast<uint32_t*>(out);
  const uint8_t qmax = (uint8_t)((1 << bits) - 1);
  for (int32_t j = 0; j < d_out; ++j) {
    uint32_t* row = o + (size_t)j * row_words;
    std::memset(row, 0, row_words * 4);
    for (int32_t i = 0; i < d_in; ++i) {
      const uint32_t v = q[(size_t)i * d_out + j];
      if (v > qmax) return DECDEC_EINVAL;
      if (bits == 4) {
        row[i >> 3] |= v << kW4Pos[i & 7];
      } else {
        const W3Bit* tb = w3_table().b[i & 31];
        uint32_t* sl = row + 3 * (i >> 5);
        for (int k = 0; k < 3; ++k) sl[tb[k].word] |= ((v >> k) & 1u) << tb[k].bit;
      }
    }
  }
  return DECDEC_OK;
}

decdec_status decdec_pack_residual(const int8_t* c, int32_t d_in, int32_t d_out, void* out, size_t out_bytes) {
  if (!c || !out) return DECDEC_EINVAL;
  if (d_in <= 0 || d_out <= 0 || d_out % 8) return DECDEC_EINVAL;
  const size_t row_words = (size_t)d_out / 8;
  if (out_bytes < row_words * 4 * (size_t)d_in) return DECDEC_ESPACE;
  uint32_t* o = static_cast<uint32_t*>(out);
  for (int32_t i = 0; i < d_in; ++i) {
    const int8_t* src = c + (size_t)i * d_out;
    uint32_t* row = o + (size_t)i * row_words;
    for (size_t w = 0; w < row_words; ++w) {
      uint32_t acc = 0;
      for (int e = 0; e < 8; ++e) {
        const int v = src[w * 8 + e];
        if (v < -7 || v > 7) return DECDEC_EINVAL;
        acc |= (uint32_t)(v + 8) << kW4Pos[e];
      }
      row[w] = acc;
    }
  }
  return DECDEC_OK;
}

decdec_status decdec_host_alloc(size_t bytes, int32_t numa_node, int32_t write_combined, void** p) {
  if (!p || bytes == 0) return DECDEC_EINVAL;
  *p = nullptr;
  if (numa_node < 0) {
    unsigned flags = cudaHostAllocMapped | cudaHostAllocPortable;
    if (write_combined) flags |= cudaHostAllocWriteCombined;
    void* h = nullptr;
    cudaError_t e = cudaHostAlloc(&h, bytes, flags);
    if (e != cudaSuccess) {
      fprintf(stderr, "[decdec] cudaHostAlloc(%zu): %s\n", bytes, cudaGetErrorString(e));
      return DECDEC_ECUDA;
    }
    std::lock_guard<std::mutex> g(g_alloc_mu);
    g_allocs[h] = {bytes, false};
    *p = h;
    return DECDEC_OK;
  }
  // NUMA-bound: mmap, mbind to the node, touch, then pin + map for the GPU.
  const size_t pg = (size_t)sysconf(_SC_PAGESIZE);
  const size_t len = (bytes + pg - 1) / pg * pg;
  void* h = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (h == MAP_FAILED) return DECDEC_ECUDA;
  if (numa_node < 64) {
    unsigned long mask = 1ul << numa_node;
    // MPOL_BIND = 2; failure (single-node kernels without NUMA) is not fatal.
    syscall(SYS_mbind, h, len, 2, &mask, 64, 0);
  }
  std::memset(h, 0, len);
  cudaError_t e = cudaHostRegister(h, len, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    munmap(h, len);
    fprintf(stderr, "[decdec] cudaHostRegister(%zu): %s\n", len, cudaGetErrorString(e));
    return DECDEC_ECUDA;
  }
  std::lock_guard<std::mutex> g(g_alloc_mu);
  g_allocs[h] = {len, true};
  *p = h;
  return DECDEC_OK;
}

void decdec_host_free(void* p) {
  if (!p) return;
  std::pair<size_t, bool> info{0, false};
  {
    std::lock_guard<std::mutex> g(g_alloc_mu);
    auto it = g_allocs.find(p);
    if (it == g_allocs.end()) return;
    info = it->second;
    g_allocs.erase(it);
  }
  if (info.second) {
    cudaHostUnregister(p);
    munmap(p, info.first);
  } else {
    cudaFreeHost(p);
  }
}

const char* decdec_status_string(decdec_status s) {
  switch (s) {
    case DECDEC_OK: return "ok";
    case DECDEC_EINVAL: return "invalid argument";
    case DECDEC_EALIGN: return "pointer not 16-byte aligned";
    case DECDEC_ENOTMAPPED: return "residual pointer is not host-mapped memory";
    case DECDEC_EUNSUPPORTED: return "unsupported configuration";
    case DECDEC_ECUDA: return "CUDA runtime error";
    case DECDEC_ENCCL: return "NCCL error";
    case DECDEC_ESPACE: return "buffer too small";
  }
  return "unknown status";
}

const char* decdec_version(void) { return "decdec-b200 0.2 (sm_100a)"; }

int32_t decdec_device_numa_node(int32_t device) {
  char bdf[32] = {0};
  if (cudaDeviceGetPCIBusId(bdf, (int)sizeof bdf, device) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  for (char* c = bdf; *c; ++c)  // sysfs uses lower-case hex ("0000:e5:00.0")
    if (*c >= 'A' && *c <= 'F') *c = (char)(*c - 'A' + 'a');
  char path[96];
  snprintf(path, sizeof path, "/sys/bus/pci/devices/%s/numa_node", bdf);
  FILE* f = fopen(path, "r");
  if (!f) return -1;
  int node = -1;
  if (fscanf(f, "%d", &node) != 1) node = -1;
  fclose(f);
  return node >= 0 ? node : -1;
}

}  // extern "C"
