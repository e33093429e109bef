// Neighbour plane exchanges of the z-slab path over NVLink peer memory (no NCCL on this path).
//
// Every rank owns one "mail" allocation, mapped into its z-neighbours' address spaces with CUDA
// IPC: an inbox of K slots per neighbour, one flag per slot and one acknowledgement counter per
// neighbour, all written by that neighbour with system-scope release stores. An exchange is two
// kernels on the rank's stream:
//   send: wait until the neighbour has consumed the exchange K sends ago (ack), store the planes
//         into the neighbour's inbox slot over NVLink, fence, then release the slot's flag = seq;
//   recv: wait (acquire) until the flag of this exchange's slot holds seq, copy or add the planes
//         from the local inbox (lower rank's partial first), then release the ack to the sender.
// Sequence numbers live in device memory and are advanced by the kernels, so the exchanges can be
// captured in the V-cycle's CUDA graph and replayed. Ranks run the same exchange sequence, and a
// send never waits on a receive of the same exchange, so the protocol cannot deadlock. Spins are
// bounded (about 10 s): a timeout sets an error word the host checks at its next synchronisation.
#include <nccl.h>

#include <cstring>

#include "device.cuh"
#include "objects.hpp"
#include "peer.hpp"

namespace sb {

namespace {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// spin until *p >= v (acquire); false on timeout
__device__ bool wait_geq(const unsigned long long* p, unsigned long long v, unsigned* err) {
  if (ld_acquire_sys(p) >= v) return true;
  const long long t0 = clock64();
  for (unsigned it = 0;; ++it) {
    if (ld_acquire_sys(p) >= v) return true;
    if (it > 4096) __nanosleep(64);
    if (clock64() - t0 > (long long)20000000000LL) {  // ~10 s at 2 GHz
      atomicExch(err, 1u);
      return false;
    }
  }
}
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

struct Side {                   // one direction of one exchange
  int active;                   // neighbour exists
  int n;                        // planes
  const double* src[kPeerMaxPlanes];
  double* dst[kPeerMaxPlanes];
  int op[kPeerMaxPlanes];       // recv: 0 copy, 1 dst = in + dst, 2 dst = dst + in
  double* slot_base;            // send: neighbour's inbox (slots); recv: my inbox
  unsigned long long* flags;    // send: neighbour's flags; recv: my flags
  unsigned long long* ack;      // send: my ack counter (written by the neighbour); recv: the neighbour's
  unsigned long long* seq;      // my device counter of this side
  unsigned* done;               // block-completion counter of this side
};

// blocks [0, G) serve side 0 (below), [G, 2G) side 1 (above)
__global__ void k_peer_send(Side s0, Side s1, int64_t P, int64_t slot_doubles, int K, unsigned* err) {
  const int G = gridDim.x / 2;
  const Side& s = blockIdx.x < unsigned(G) ? s0 : s1;
  if (!s.active) return;
  const int b = blockIdx.x % G;
  __shared__ unsigned long long seq;
  __shared__ bool ok;
  if (threadIdx.x == 0) {
    seq = *s.seq + 1;
    ok = seq <= (unsigned long long)K || wait_geq(s.ack, seq - K, err);  // slot reuse: consumed K sends ago
  }
  __syncthreads();
  if (!ok) return;
  double* slot = s.slot_base + ((seq - 1) % K) * slot_doubles;
  for (int k = 0; k < s.n; ++k)
    for (int64_t t = int64_t(b) * blockDim.x + threadIdx.x; t < P; t += int64_t(G) * blockDim.x)
      slot[k * P + t] = s.src[k][t];
  // the block's stores -> (barrier) -> thread 0's acq_rel counter -> the last block's system-scope
  // release of the flag: cumulative, so the neighbour's acquire of the flag sees every store
  __syncthreads();
  if (threadIdx.x == 0 && atom_add_acq_rel_gpu(s.done, 1u) == unsigned(G) - 1) {
    *s.done = 0;
    *s.seq = seq;
    __threadfence_system();
    st_release_sys(s.flags + (seq - 1) % K, seq);
  }
}

__global__ void k_peer_recv(Side s0, Side s1, int64_t P, int64_t slot_doubles, int K, unsigned* err) {
  const int G = gridDim.x / 2;
  const Side& s = blockIdx.x < unsigned(G) ? s0 : s1;
  if (!s.active) return;
  const int b = blockIdx.x % G;
  __shared__ unsigned long long seq;
  __shared__ bool ok;
  if (threadIdx.x == 0) {
    seq = *s.seq + 1;
    ok = wait_geq(s.flags + (seq - 1) % K, seq, err);
  }
  __syncthreads();
  if (!ok) return;
  const double* slot = s.slot_base + ((seq - 1) % K) * slot_doubles;
  for (int k = 0; k < s.n; ++k) {
    const int op = s.op[k];
    double* d = s.dst[k];
    for (int64_t t = int64_t(b) * blockDim.x + threadIdx.x; t < P; t += int64_t(G) * blockDim.x) {
      const double in = __ldcv(slot + k * P + t);
      d[t] = op == 0 ? in : (op == 1 ? in + d[t] : d[t] + in);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && atom_add_acq_rel_gpu(s.done, 1u) == unsigned(G) - 1) {
    *s.done = 0;
    *s.seq = seq;
    st_release_sys(s.ack, seq);  // the sender may reuse the slot
  }
}

// layout of one rank's mail allocation (doubles / u64 words)
struct MailLayout {
  int64_t slot_doubles;
  int K;
  size_t inbox(int d) const { return size_t(d) * K * slot_doubles; }              // from below / above
  size_t words() const { return size_t(2) * K * slot_doubles; }                    // first control word
  size_t flag(int d) const { return words() + size_t(d) * K; }
  size_t ack(int d) const { return words() + size_t(2 * K) + size_t(d); }          // acks of MY sends
  size_t bytes() const { return (words() + size_t(2 * K) + 2) * 8; }
};

}  // namespace

struct PeerLinks::Impl {
  MailLayout L{};
  void* mail = nullptr;            // mine
  void* peer_mail[2] = {nullptr, nullptr};
  unsigned long long* ctl = nullptr;  // local: seq send[2], seq recv[2]; done counters after
  unsigned* err = nullptr;
};

PeerLinks::~PeerLinks() { release(); }

// The rank's own mail is never freed while the process lives: a neighbour that is still finishing
// its last receive may store an acknowledgement into it after this rank has moved on (a few MB).
void PeerLinks::release() {
  if (!impl) return;
  for (auto& p : impl->peer_mail)
    if (p) cudaIpcCloseMemHandle(p);
  delete impl;
  impl = nullptr;
}

bool PeerLinks::supported(semlab_ctx c) {
  if (c->nranks < 2) return false;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return false;
  // one process per GPU on one node: rank r drives device r (torchrun LOCAL_RANK = device)
  for (int d : {c->device - 1, c->device + 1}) {
    if (d < 0 || d >= n) continue;
    int ok = 0;
    if (cudaDeviceCanAccessPeer(&ok, c->device, d) != cudaSuccess || !ok) return false;
  }
  return true;
}

// Collective (all ranks): allocate the mail with slots of `slot_doubles`, exchange IPC handles
// (NCCL all-gather of the 64-byte handles) and map the z-neighbours' mail. The peer path is used
// only if every rank can (NCCL min-reduction of the local verdicts); otherwise false (NCCL path).
bool PeerLinks::init(semlab_ctx c, int64_t slot_doubles) {
  if (impl) {  // growth: every rank's earlier exchanges have drained (barrier) before the switch
    DevBuf<double> one(1);
    one.zero(c->stream);
    SB_NCCL(ncclAllReduce(one.p, one.p, 1, ncclDouble, ncclSum, static_cast<ncclComm_t>(c->nccl), c->stream));
    SB_CUDA(cudaStreamSynchronize(c->stream));
  }
  release();
  {
    DevBuf<double> ok(1);
    const double mine = supported(c) ? 1.0 : 0.0;
    ok.upload(&mine, 1, c->stream);
    SB_NCCL(ncclAllReduce(ok.p, ok.p, 1, ncclDouble, ncclMin, static_cast<ncclComm_t>(c->nccl), c->stream));
    double all = 0.0;
    SB_CUDA(cudaMemcpyAsync(&all, ok.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    SB_CUDA(cudaStreamSynchronize(c->stream));
    if (all < 1.0) return false;
  }
  impl = new Impl();
  impl->L.slot_doubles = slot_doubles;
  impl->L.K = kPeerSlots;
  cudaStream_t s = c->stream;
  SB_CUDA(cudaMalloc(&impl->mail, impl->L.bytes()));
  SB_CUDA(cudaMemsetAsync(impl->mail, 0, impl->L.bytes(), s));
  SB_CUDA(cudaMalloc(&impl->ctl, 16 * sizeof(unsigned long long)));
  SB_CUDA(cudaMemsetAsync(impl->ctl, 0, 16 * sizeof(unsigned long long), s));
  impl->err = reinterpret_cast<unsigned*>(impl->ctl + 12);
  cudaIpcMemHandle_t h;
  SB_CUDA(cudaIpcGetMemHandle(&h, impl->mail));
  const int R = c->nranks;
  DevBuf<unsigned char> dh(sizeof(h)), all(sizeof(h) * size_t(R));
  dh.upload(reinterpret_cast<const unsigned char*>(&h), sizeof(h), s);
  SB_NCCL(ncclAllGather(dh.p, all.p, sizeof(h), ncclUint8, static_cast<ncclComm_t>(c->nccl), s));
  std::vector<cudaIpcMemHandle_t> hs(static_cast<size_t>(R));
  SB_CUDA(cudaMemcpyAsync(hs.data(), all.p, sizeof(h) * size_t(R), cudaMemcpyDeviceToHost, s));
  SB_CUDA(cudaStreamSynchronize(s));
  for (int d = 0; d < 2; ++d) {
    const int nb = c->rank + (d == 0 ? -1 : 1);
    if (nb < 0 || nb >= R) continue;
    SB_CUDA(cudaIpcOpenMemHandle(&impl->peer_mail[d], hs[size_t(nb)], cudaIpcMemLazyEnablePeerAccess));
  }
  // every rank's mail is zeroed before anyone can send into it
  DevBuf<double> one(1);
  one.zero(s);
  SB_NCCL(ncclAllReduce(one.p, one.p, 1, ncclDouble, ncclSum, static_cast<ncclComm_t>(c->nccl), s));
  SB_CUDA(cudaStreamSynchronize(s));
  capacity = slot_doubles;
  return true;
}

void PeerLinks::check(semlab_ctx) const {
  if (!impl) return;
  unsigned e = 0;
  SB_CUDA(cudaMemcpy(&e, impl->err, sizeof(e), cudaMemcpyDeviceToHost));
  if (e) numeric("peer exchange: a z-neighbour did not answer within ~10 s (ranks out of step?)");
}

int64_t PeerLinks::exchange(semlab_ctx c, const PeerSide* sides, int64_t P, cudaStream_t s) {
  const int K = impl->L.K;
  const int64_t SD = impl->L.slot_doubles;
  Side snd[2], rcv[2];
  for (int d = 0; d < 2; ++d) {
    const PeerSide& ps = sides[d];
    auto* mine = static_cast<double*>(impl->mail);
    auto* mine_w = reinterpret_cast<unsigned long long*>(impl->mail);
    auto* peer = static_cast<double*>(impl->peer_mail[d]);
    auto* peer_w = reinterpret_cast<unsigned long long*>(impl->peer_mail[d]);
    const int od = 1 - d;  // I am the neighbour's direction od
    Side& a = snd[d];
    a = Side{};
    a.active = ps.active && ps.nsend > 0;
    a.n = ps.nsend;
    for (int k = 0; k < ps.nsend; ++k) a.src[k] = ps.src[k];
    if (a.active) {
      a.slot_base = peer + impl->L.inbox(od);
      a.flags = peer_w + impl->L.flag(od);
      a.ack = mine_w + impl->L.ack(d);
    }
    a.seq = impl->ctl + d;
    a.done = reinterpret_cast<unsigned*>(impl->ctl + 4) + d;
    Side& b = rcv[d];
    b = Side{};
    b.active = ps.active && ps.nrecv > 0;
    b.n = ps.nrecv;
    for (int k = 0; k < ps.nrecv; ++k) {
      b.dst[k] = ps.dst[k];
      b.op[k] = ps.op[k];
    }
    if (b.active) {
      b.slot_base = mine + impl->L.inbox(d);
      b.flags = mine_w + impl->L.flag(d);
      b.ack = peer_w + impl->L.ack(od);
    }
    b.seq = impl->ctl + 2 + d;
    b.done = reinterpret_cast<unsigned*>(impl->ctl + 4) + 2 + d;
  }
  const int G = int(std::min<int64_t>(64, std::max<int64_t>(1, (P + 1023) / 1024)));
  k_peer_send<<<2 * G, 256, 0, s>>>(snd[0], snd[1], P, SD, K, impl->err);
  SB_LAUNCH_CHECK();
  k_peer_recv<<<2 * G, 256, 0, s>>>(rcv[0], rcv[1], P, SD, K, impl->err);
  SB_LAUNCH_CHECK();
  (void)c;
  return 2;
}

}  // namespace sb
