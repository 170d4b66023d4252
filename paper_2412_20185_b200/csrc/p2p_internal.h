// Internal (not part of the C ABI): the peer group behind decdec_peers (p2p.cu), read by the
// layer planner (decdec_api.cu) to fill p2p.cuh's P2PParams.
#pragma once
#include <cstddef>

#include "decdec.h"

struct decdec_peers {
  int rank = 0, nranks = 0;   // nranks = 0 until decdec_peers_connect
  size_t user_bytes = 0;
  void* local = nullptr;      // this rank's region: [flag area | user area]
  void* base[8] = {nullptr};  // every rank's region as mapped in this process (base[rank] = local)
};
