// Host-side objects behind the opaque C handles of include/semlab_b200.h.
#pragma once

#include <array>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../../include/semlab_b200.h"
#include "common.hpp"
#include "kernels.hpp"
#include "peer.hpp"

struct semlab_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int rank = 0, nranks = 1;
  void* nccl = nullptr;  // ncclComm_t
  int64_t launches = 0;
  sb::DevBuf<double> dot_partial;
  sb::DevBuf<unsigned> dot_counter;
  sb::DevBuf<double> dot_out;
  double* host_pinned = nullptr;  // 64 doubles
  // Krylov workspace kept across solves (grow-only): cudaMalloc/cudaFree of the ~2 GB GMRES basis
  // per solve costs a device sync and tens to hundreds of ms. A nested solve allocates its own.
  sb::DevBuf<double> krylov_ws;
  bool krylov_ws_busy = false;
  // z-slab neighbour exchanges: NCCL send/recv (exchange_mode 0, the default: measured faster), or
  // NVLink peer memory (sb::PeerLinks, exchange_mode 1) when every rank supports it.
  sb::PeerLinks peer;
  int exchange_mode = 0, peer_state = -1;  // peer_state: -1 undecided, 0 NCCL, 1 peer
  bool use_peer(int64_t slot_doubles);     // collective on first use / growth (never inside a capture)
  sb::DotScratch dots() const { return {dot_partial.p, dot_counter.p}; }
  void count(int64_t n) { launches += n; }
  // Global sum over ranks of K host doubles (NCCL allreduce on device values when nranks>1).
  void allreduce_device(double* d_vals, int K);
  void sync() { SB_CUDA(cudaStreamSynchronize(stream)); }
  // Deterministic dots of K vector pairs over [off, off+len) summed over ranks; host result.
  void dots(int K, const double* const* a, const double* const* b, int64_t off, int64_t len, double* host_out,
            bool global = true);
};

struct semlab_mesh_s {
  semlab_ctx ctx = nullptr;
  std::array<int, 3> dims{};
  std::function<std::array<double, 3>(double, double, double)> map;
  double kershaw_eps = 0.0;  // > 0 for generate_kershaw meshes
  // lattice coordinates of global planes [z0, z0+nz) at an order, (x,y,z) triples x-fastest
  std::vector<double> lattice_planes(int order, int64_t z0, int64_t nz) const;
  // 1-D unit coordinates of the global GLL lattice per axis (mesh.cpp:104-123)
  std::array<std::vector<double>, 3> lattice_axes(int order) const;
};

struct semlab_space_s {
  semlab_ctx ctx = nullptr;
  semlab_mesh mesh = nullptr;
  int order = 0, bc = SEMLAB_BC_DIRICHLET;
  sb::Slab sl{};
  int64_t n = 0, E = 0, nloc = 0;
  std::vector<double> coords;  // host lattice coords of the local planes (3 per point)
  sb::DevBuf<double> geom, massw, mass_diag, inv_diag, dep, scratch_e, plane_lo, plane_hi;
  sb::DevBuf<double> ones;  // Neumann mean removal (sem_space.cpp:207): the all-ones vector
  sb::DevBuf<unsigned> flags, ticket;
  sb::DevBuf<float> geom32;  // FP32-rounded geometric factors (the smoother's operator, order 7)
  bool has_inv_diag = false;
  bool full = false;  // whole mesh on this rank even under a distributed context (coarse solve)
  bool distributed() const { return !full && ctx->nranks > 1; }
  void halo_exchange(double* v);
  void owner_copy_up(double* v);
  void interface_sum_halo(double* v);              // interface_sum + halo_exchange, one NCCL group
  void owner_copy_up_n(double* const* vs, int k);  // owner_copy_up of k vectors, one NCCL group

  void build();
  sb::AxSync sync() const { return {dep.p, flags.p, ticket.p}; }
  // A with an epilogue; handles the slab interface sum when distributed. g32: use the
  // FP32-rounded geometric factors (only where has_geom32()).
  void apply_A(const double* in, double* out, bool g32 = false);
  void ax(const double* in, sb::Epi epi, const sb::EpiArgs& a, bool g32 = false);
  bool enable_geom32();  // builds geom32 if the order supports it; false otherwise
  bool has_geom32() const { return geom32.p != nullptr; }
  const double* jacobi_inv();
  void stiffness_diag(double* out);
  int64_t own_off() const { return sl.lidx(0, 0, sl.own_z0()); }
  int64_t own_len() const { return sl.Nx * sl.Ny * (sl.own_z1() - sl.own_z0()); }
  double dot(const double* a, const double* b);
  // Sum partial values on the slab interface planes across ranks (after a Q^T-type op).
  void interface_sum(double* v);
};

struct semlab_schwarz_s;
struct semlab_pmg_s;
struct semlab_semfem_s;
void semfem_apply(semlab_semfem_s* p, const double* r, double* z);

struct semlab_op_s {
  enum Kind { kA, kJacobi, kSchwarz, kPmg, kCallback, kSemfem } kind = kA;
  semlab_ctx ctx = nullptr;
  int64_t n = 0;
  semlab_space space = nullptr;
  semlab_schwarz_s* sch = nullptr;
  semlab_pmg_s* pmg = nullptr;
  semlab_semfem_s* semfem = nullptr;
  semlab_apply_fn fn = nullptr;
  void* user = nullptr;
  bool geom32 = false;  // kA: apply with the FP32-rounded geometric factors (smoother operator)
  void apply(const double* in, double* out);
};

// Thread-local last-error text.
void sb_set_error(const std::string& msg);
