// Output-feature tensor parallelism: the one exchange step of the sharded path (SURVEY.md
// §8(e)).  Every rank runs decdec_linear on its column shard (identical S on
// every rank: x is replicated and the selector is exact and deterministic, ledger L11), then
// the fp16 shards are assembled by an in-place NCCL all-gather on the same stream.
//
// NCCL is resolved at run time (dlopen) so libdecdec.so has no link-time NCCL dependency and
// shares the process's already-loaded libnccl (PyTorch's) when there is one.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "decdec.h"
#include "tp_internal.h"

struct decdec_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
};

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  bool ok = false;
};

NcclApi g_nccl;
std::once_flag g_nccl_once;

void load_nccl() {
  // Prefer a libnccl already in the process (PyTorch's bundled one), else the system's.
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return;
  g_nccl.get_unique_id = reinterpret_cast<decltype(g_nccl.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  g_nccl.comm_init_rank = reinterpret_cast<decltype(g_nccl.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  g_nccl.comm_destroy = reinterpret_cast<decltype(g_nccl.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  g_nccl.all_gather = reinterpret_cast<decltype(g_nccl.all_gather)>(dlsym(h, "ncclAllGather"));
  g_nccl.get_version = reinterpret_cast<decltype(g_nccl.get_version)>(dlsym(h, "ncclGetVersion"));
  g_nccl.ok = g_nccl.get_unique_id && g_nccl.comm_init_rank && g_nccl.comm_destroy && g_nccl.all_gather;
}

bool nccl() {
  std::call_once(g_nccl_once, load_nccl);
  return g_nccl.ok;
}

}  // namespace

// In-place all-gather of this rank's d_out_r fp16 outputs, which sit at
// y_full + rank * d_out_r, into y_full[nranks * d_out_r] (stream-ordered; capturable).
decdec_status tp_allgather(decdec_comm* c, uint16_t* y_full, int32_t d_out_r, cudaStream_t st) {
  if (!c || !c->comm || !nccl()) return DECDEC_ENCCL;
  if (c->nranks == 1) return DECDEC_OK;
  const uint16_t* mine = y_full + (size_t)c->rank * d_out_r;
  return g_nccl.all_gather(mine, y_full, (size_t)d_out_r, ncclFloat16, c->comm, st) == ncclSuccess ? DECDEC_OK
                                                                                                   : DECDEC_ENCCL;
}

int32_t tp_rank(const decdec_comm* c) { return c ? c->rank : -1; }

extern "C" {

int32_t decdec_nccl_version(void) {
  int v = -1;
  if (!nccl() || !g_nccl.get_version || g_nccl.get_version(&v) != ncclSuccess) return -1;
  return v;
}

decdec_status decdec_nccl_unique_id(void* id_out) {
  if (!id_out) return DECDEC_EINVAL;
  if (!nccl()) return DECDEC_ENCCL;
  ncclUniqueId id;
  if (g_nccl.get_unique_id(&id) != ncclSuccess) return DECDEC_ENCCL;
  std::memcpy(id_out, &id, sizeof(id));
  return DECDEC_OK;
}

decdec_status decdec_comm_init(const void* id, int32_t rank, int32_t nranks, decdec_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return DECDEC_EINVAL;
  *out = nullptr;
  if (!nccl()) return DECDEC_ENCCL;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  decdec_comm* c = new decdec_comm();
  c->rank = rank;
  c->nranks = nranks;
  if (g_nccl.comm_init_rank(&c->comm, nranks, uid, rank) != ncclSuccess) {
    delete c;
    return DECDEC_ENCCL;
  }
  *out = c;
  return DECDEC_OK;
}

void decdec_comm_destroy(decdec_comm* c) {
  if (!c) return;
  if (c->comm && nccl()) g_nccl.comm_destroy(c->comm);
  delete c;
}

int32_t decdec_comm_rank(const decdec_comm* c) { return c ? c->rank : -1; }
int32_t decdec_comm_nranks(const decdec_comm* c) { return c ? c->nranks : -1; }

decdec_status decdec_linear_tp(const decdec_layer* L, const uint16_t* x, int32_t k, int32_t chunk,
                               uint16_t* y_full, int32_t* sel, void* ws, size_t ws_bytes, decdec_comm* comm,
                               decdec_stream_t stream) {
  if (!L || !comm || !y_full) return DECDEC_EINVAL;
  uint16_t* mine = y_full + (size_t)comm->rank * L->d_out;
  decdec_status s = decdec_linear(L, x, k, chunk, mine, sel, ws, ws_bytes, stream);
  if (s != DECDEC_OK) return s;
  return tp_allgather(comm, y_full, L->d_out, (cudaStream_t)stream);
}

}  // extern "C"
