// Neighbour plane exchanges over NVLink peer memory (CUDA IPC mail slots, flag/ack protocol);
// see peer.cu. Used by the z-slab exchanges of semlab_space_s when every rank supports it.
#pragma once

#include <cstdint>

#include "common.hpp"

struct semlab_ctx_s;

namespace sb {

constexpr int kPeerMaxPlanes = 4;  // planes per direction per exchange
constexpr int kPeerSlots = 4;      // in-flight exchanges per direction

struct PeerSide {  // one direction (0 = rank-1, 1 = rank+1) of an exchange
  bool active = false;  // the neighbour exists
  int nsend = 0;
  const double* src[kPeerMaxPlanes] = {};
  int nrecv = 0;
  double* dst[kPeerMaxPlanes] = {};
  int op[kPeerMaxPlanes] = {};  // 0 copy, 1 dst = received + dst (neighbour = lower partial), 2 dst = dst + received
};

struct PeerLinks {
  struct Impl;
  Impl* impl = nullptr;
  int64_t capacity = 0;  // doubles per slot
  ~PeerLinks();
  static bool supported(semlab_ctx_s* c);
  bool init(semlab_ctx_s* c, int64_t slot_doubles);  // collective
  void release();
  void check(semlab_ctx_s* c) const;  // throws if a wait timed out
  // one exchange of planes of P doubles in both directions (sends, then receives): 2 launches
  int64_t exchange(semlab_ctx_s* c, const PeerSide* sides, int64_t P, cudaStream_t s);
};

}  // namespace sb
