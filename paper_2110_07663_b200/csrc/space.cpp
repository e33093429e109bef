// Context, mesh and SemSpace host logic (setup on the host/device, every apply on the device).
#include <cstdlib>
#include <nccl.h>
#include <omp.h>

#include <algorithm>
#include <cmath>

#include "host_math.hpp"
#include "objects.hpp"
#include "pmg.hpp"
#include "schwarz.hpp"

using namespace sb;


// ------------------------------------------------------------------------------ context
void semlab_ctx_s::allreduce_device(double* d_vals, int K) {
  if (nranks <= 1) return;
  SB_NCCL(ncclAllReduce(d_vals, d_vals, size_t(K), ncclDouble, ncclSum, static_cast<ncclComm_t>(nccl), stream));
}

bool semlab_ctx_s::use_peer(int64_t slot_doubles) {
  if (nranks < 2 || exchange_mode == 0 || peer_state == 0) return false;
  if (peer_state == 1 && peer.capacity >= slot_doubles) return true;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  SB_CUDA(cudaStreamIsCapturing(stream, &cs));
  if (cs != cudaStreamCaptureStatusNone)
    numeric("peer exchange: mail slots must grow during a CUDA-graph capture (run the operation eagerly first)");
  // all ranks reach this point for the same exchange (same global plane sizes): collective setup
  peer_state = peer.init(this, std::max<int64_t>(slot_doubles, peer.capacity)) ? 1 : 0;
  return peer_state == 1;
}

void semlab_ctx_s::dots(int K, const double* const* a, const double* const* b, int64_t off, int64_t len,
                        double* host_out, bool global) {
  const double* aa[4];
  const double* bb[4];
  for (int k = 0; k < K; ++k) {
    aa[k] = a[k] + off;
    bb[k] = b[k] + off;
  }
  count(launch_dots(K, aa, bb, len, dot_out.p, dots(), stream));
  if (global) allreduce_device(dot_out.p, K);
  SB_CUDA(cudaMemcpyAsync(host_pinned, dot_out.p, sizeof(double) * K, cudaMemcpyDeviceToHost, stream));
  sync();
  if (peer_state == 1) peer.check(this);
  for (int k = 0; k < K; ++k) host_out[k] = host_pinned[k];
}

// ------------------------------------------------------------------------------ mesh
// Global GLL-lattice coordinates (mesh.cpp:104-136) for planes [z0, z0+nz) only.
std::array<std::vector<double>, 3> semlab_mesh_s::lattice_axes(int order) const {
  const Gll& g = gll(order);
  std::array<std::vector<double>, 3> axis;
  for (int d = 0; d < 3; ++d) {
    const int64_t npts = int64_t(dims[d]) * order + 1;
    axis[d].resize(size_t(npts));
    for (int64_t gi = 0; gi < npts; ++gi) {
      int64_t e = gi / order, i = gi % order;
      if (e == dims[d]) {
        e -= 1;
        i = order;
      }
      axis[d][size_t(gi)] = (double(e) + 0.5 * (g.nodes[size_t(i)] + 1.0)) / dims[d];
    }
  }
  return axis;
}

std::vector<double> semlab_mesh_s::lattice_planes(int order, int64_t z0, int64_t nz) const {
  const auto axis = lattice_axes(order);
  const int64_t nx = int64_t(dims[0]) * order + 1, ny = int64_t(dims[1]) * order + 1;
  std::vector<double> out(size_t(nx * ny * nz) * 3);
  auto fill = [&](int64_t kk) {
    const int64_t k = z0 + kk;
    size_t idx = size_t(kk * nx * ny) * 3;
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        const auto p = map(axis[0][size_t(i)], axis[1][size_t(j)], axis[2][size_t(k)]);
        out[idx++] = p[0];
        out[idx++] = p[1];
        out[idx++] = p[2];
      }
  };
  if (kershaw_eps > 0.0) {  // pure C++ map: safe to evaluate in parallel
#pragma omp parallel for schedule(static)
    for (int64_t kk = 0; kk < nz; ++kk) fill(kk);
  } else {
    for (int64_t kk = 0; kk < nz; ++kk) fill(kk);
  }
  return out;
}

// ------------------------------------------------------------------------------ space
void semlab_space_s::build() {
  if (order < 1 || order > 9) invalid("SemSpace: order must be in [1,9] for the device kernels, got " + std::to_string(order));
  const int rk = full ? 0 : ctx->rank, nr = full ? 1 : ctx->nranks;
  if (nr > mesh->dims[2])
    invalid("SemSpace: more ranks (" + std::to_string(nr) + ") than element layers in z (" +
            std::to_string(mesh->dims[2]) + ")");
  sl = make_slab(order, mesh->dims[0], mesh->dims[1], mesh->dims[2], rk, nr, bc == SEMLAB_BC_DIRICHLET);
  const int nd = order + 1;
  nloc = int64_t(nd) * nd * nd;
  E = sl.elems();
  n = sl.n_local();
  cudaStream_t s = ctx->stream;
  coords = mesh->lattice_planes(order, sl.zlo, sl.nzl);
  DevBuf<double> X(coords.size());
  X.upload(coords.data(), coords.size(), s);
  geom.alloc(size_t(E * nloc * 6));
  massw.alloc(size_t(E * nloc));
  DevBuf<unsigned long long> bad(1);
  SB_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), s));
  ctx->count(launch_geom(sl, X.p, geom.p, massw.p, bad.p, s));
  unsigned long long hb = 0;
  SB_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(hb), cudaMemcpyDeviceToHost, s));
  ctx->sync();
  if (hb != ~0ull) numeric("SemSpace: non-positive Jacobian in element " + std::to_string(hb));
  mass_diag.alloc(size_t(n));
  mass_diag.zero(s);
  ctx->count(launch_gather(sl, massw.p, mass_diag.p, s));
  interface_sum(mass_diag.p);
  dep.alloc(size_t(E * nloc));
  flags.alloc(size_t(std::max<int64_t>(E, 1)));
  flags.zero(s);
  ticket.alloc(1);
  ticket.zero(s);
  ctx->sync();
}

// ---- slab exchanges over NCCL (grouped send/recv between z-neighbour ranks) ---------------
// Interface planes z = ez0 q (shared with rank-1) and z = ez1 q (shared with rank+1) hold this
// rank's partial Q^T sums after a gather-type operation; both ranks add lower + upper partial in
// that order, so the duplicated planes stay bitwise identical on the two ranks.

// The same exchanges over NVLink peer memory (peer.cu): planes are stored into the neighbour's
// mail slot and combined there in the same order as below (lower rank's partial first).
namespace {
PeerSide side(bool active) {
  PeerSide p;
  p.active = active;
  return p;
}
}  // namespace

void semlab_space_s::interface_sum(double* v) {
  if (!distributed()) return;
  const int64_t P = sl.Nx * sl.Ny;
  if (ctx->use_peer(4 * P)) {
    double* vb = v + sl.lidx(0, 0, int64_t(sl.ez0) * sl.q);
    double* vt = v + sl.lidx(0, 0, int64_t(sl.ez1) * sl.q);
    PeerSide sd[2] = {side(sl.nranks_below), side(sl.nranks_above)};
    sd[0].nsend = sd[0].nrecv = 1;
    sd[0].src[0] = vb;
    sd[0].dst[0] = vb;
    sd[0].op[0] = 1;  // lower partial + mine
    sd[1].nsend = sd[1].nrecv = 1;
    sd[1].src[0] = vt;
    sd[1].dst[0] = vt;
    sd[1].op[0] = 2;  // mine + upper partial
    ctx->count(ctx->peer.exchange(ctx, sd, P, ctx->stream));
    return;
  }
  if (plane_lo.n < size_t(P)) {
    plane_lo.alloc(size_t(P));
    plane_hi.alloc(size_t(P));
  }
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl);
  cudaStream_t s = ctx->stream;
  const int r = ctx->rank;
  double* vb = v + sl.lidx(0, 0, int64_t(sl.ez0) * sl.q);
  double* vt = v + sl.lidx(0, 0, int64_t(sl.ez1) * sl.q);
  SB_NCCL(ncclGroupStart());
  if (sl.nranks_below) {
    SB_NCCL(ncclSend(vb, size_t(P), ncclDouble, r - 1, comm, s));
    SB_NCCL(ncclRecv(plane_lo.p, size_t(P), ncclDouble, r - 1, comm, s));
  }
  if (sl.nranks_above) {
    SB_NCCL(ncclSend(vt, size_t(P), ncclDouble, r + 1, comm, s));
    SB_NCCL(ncclRecv(plane_hi.p, size_t(P), ncclDouble, r + 1, comm, s));
  }
  SB_NCCL(ncclGroupEnd());
  if (sl.nranks_below) ctx->count(launch_add_planes(vb, plane_lo.p, vb, P, s));  // lower partial first
  if (sl.nranks_above) ctx->count(launch_add_planes(vt, vt, plane_hi.p, P, s));
}

// interface_sum followed by halo_exchange in ONE grouped NCCL call: right after a Q^T-type
// operator the planes next to the interface are already final on their owner, so the partial
// interface planes and the Schwarz ghost planes travel together (one latency instead of two).
void semlab_space_s::interface_sum_halo(double* v) {
  if (!distributed()) return;
  const int64_t P = sl.Nx * sl.Ny;
  if (ctx->use_peer(4 * P)) {
    const int64_t zb = int64_t(sl.ez0) * sl.q, zt = int64_t(sl.ez1) * sl.q;
    auto pl = [&](int64_t z) { return v + sl.lidx(0, 0, z); };
    PeerSide sd[2] = {side(sl.nranks_below), side(sl.nranks_above)};
    sd[0].nsend = sd[0].nrecv = 2;
    sd[0].src[0] = pl(zb);
    sd[0].src[1] = pl(zb + 1);
    sd[0].dst[0] = pl(zb);
    sd[0].op[0] = 1;
    sd[0].dst[1] = pl(zb - 1);  // the ghost plane
    sd[0].op[1] = 0;
    sd[1].nsend = sd[1].nrecv = 2;
    sd[1].src[0] = pl(zt);
    sd[1].src[1] = pl(zt - 1);
    sd[1].dst[0] = pl(zt);
    sd[1].op[0] = 2;
    sd[1].dst[1] = pl(zt + 1);
    sd[1].op[1] = 0;
    ctx->count(ctx->peer.exchange(ctx, sd, P, ctx->stream));
    return;
  }
  if (plane_lo.n < size_t(P)) {
    plane_lo.alloc(size_t(P));
    plane_hi.alloc(size_t(P));
  }
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl);
  cudaStream_t s = ctx->stream;
  const int r = ctx->rank;
  const int64_t zb = int64_t(sl.ez0) * sl.q, zt = int64_t(sl.ez1) * sl.q;
  double* vb = v + sl.lidx(0, 0, zb);
  double* vt = v + sl.lidx(0, 0, zt);
  SB_NCCL(ncclGroupStart());
  if (sl.nranks_below) {
    SB_NCCL(ncclSend(vb, size_t(P), ncclDouble, r - 1, comm, s));
    SB_NCCL(ncclSend(v + sl.lidx(0, 0, zb + 1), size_t(P), ncclDouble, r - 1, comm, s));
    SB_NCCL(ncclRecv(plane_lo.p, size_t(P), ncclDouble, r - 1, comm, s));
    SB_NCCL(ncclRecv(v + sl.lidx(0, 0, zb - 1), size_t(P), ncclDouble, r - 1, comm, s));
  }
  if (sl.nranks_above) {
    SB_NCCL(ncclSend(vt, size_t(P), ncclDouble, r + 1, comm, s));
    SB_NCCL(ncclSend(v + sl.lidx(0, 0, zt - 1), size_t(P), ncclDouble, r + 1, comm, s));
    SB_NCCL(ncclRecv(plane_hi.p, size_t(P), ncclDouble, r + 1, comm, s));
    SB_NCCL(ncclRecv(v + sl.lidx(0, 0, zt + 1), size_t(P), ncclDouble, r + 1, comm, s));
  }
  SB_NCCL(ncclGroupEnd());
  if (sl.nranks_below) ctx->count(launch_add_planes(vb, plane_lo.p, vb, P, s));  // lower partial first
  if (sl.nranks_above) ctx->count(launch_add_planes(vt, vt, plane_hi.p, P, s));
}

// owner_copy_up of up to three vectors in one grouped call.
void semlab_space_s::owner_copy_up_n(double* const* vs, int k) {
  if (!distributed()) return;
  const int64_t P = sl.Nx * sl.Ny;
  if (ctx->use_peer(4 * P)) {
    PeerSide sd[2] = {side(sl.nranks_below), side(sl.nranks_above)};
    sd[0].nrecv = k;
    sd[1].nsend = k;
    for (int i = 0; i < k; ++i) {
      sd[0].dst[i] = vs[i] + sl.lidx(0, 0, int64_t(sl.ez0) * sl.q);
      sd[0].op[i] = 0;
      sd[1].src[i] = vs[i] + sl.lidx(0, 0, int64_t(sl.ez1) * sl.q);
    }
    ctx->count(ctx->peer.exchange(ctx, sd, P, ctx->stream));
    return;
  }
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl);
  cudaStream_t s = ctx->stream;
  const int r = ctx->rank;
  SB_NCCL(ncclGroupStart());
  for (int i = 0; i < k; ++i) {
    double* v = vs[i];
    if (sl.nranks_above)
      SB_NCCL(ncclSend(v + sl.lidx(0, 0, int64_t(sl.ez1) * sl.q), size_t(P), ncclDouble, r + 1, comm, s));
    if (sl.nranks_below)
      SB_NCCL(ncclRecv(v + sl.lidx(0, 0, int64_t(sl.ez0) * sl.q), size_t(P), ncclDouble, r - 1, comm, s));
  }
  SB_NCCL(ncclGroupEnd());
}

// Ghost planes z = ez0 q - 1 and z = ez1 q + 1 (the Schwarz halo, schwarz.cpp:159-168).
void semlab_space_s::halo_exchange(double* v) {
  if (!distributed()) return;
  const int64_t P = sl.Nx * sl.Ny;
  if (ctx->use_peer(4 * P)) {
    const int64_t zb = int64_t(sl.ez0) * sl.q, zt = int64_t(sl.ez1) * sl.q;
    PeerSide sd[2] = {side(sl.nranks_below), side(sl.nranks_above)};
    sd[0].nsend = sd[0].nrecv = 1;
    sd[0].src[0] = v + sl.lidx(0, 0, zb + 1);
    sd[0].dst[0] = v + sl.lidx(0, 0, zb - 1);
    sd[1].nsend = sd[1].nrecv = 1;
    sd[1].src[0] = v + sl.lidx(0, 0, zt - 1);
    sd[1].dst[0] = v + sl.lidx(0, 0, zt + 1);
    ctx->count(ctx->peer.exchange(ctx, sd, P, ctx->stream));
    return;
  }
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl);
  cudaStream_t s = ctx->stream;
  const int r = ctx->rank;
  const int64_t zb = int64_t(sl.ez0) * sl.q, zt = int64_t(sl.ez1) * sl.q;
  SB_NCCL(ncclGroupStart());
  if (sl.nranks_below) {
    SB_NCCL(ncclSend(v + sl.lidx(0, 0, zb + 1), size_t(P), ncclDouble, r - 1, comm, s));
    SB_NCCL(ncclRecv(v + sl.lidx(0, 0, zb - 1), size_t(P), ncclDouble, r - 1, comm, s));
  }
  if (sl.nranks_above) {
    SB_NCCL(ncclSend(v + sl.lidx(0, 0, zt - 1), size_t(P), ncclDouble, r + 1, comm, s));
    SB_NCCL(ncclRecv(v + sl.lidx(0, 0, zt + 1), size_t(P), ncclDouble, r + 1, comm, s));
  }
  SB_NCCL(ncclGroupEnd());
}

// The interface plane z = ez1 q is owned by the lower rank for owner-write operators (RAS):
// copy it up so both ranks hold the owner's value.
void semlab_space_s::owner_copy_up(double* v) {
  if (!distributed()) return;
  const int64_t P = sl.Nx * sl.Ny;
  if (ctx->use_peer(4 * P)) {
    double* vs[1] = {v};
    owner_copy_up_n(vs, 1);
    return;
  }
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl);
  cudaStream_t s = ctx->stream;
  const int r = ctx->rank;
  SB_NCCL(ncclGroupStart());
  if (sl.nranks_above) SB_NCCL(ncclSend(v + sl.lidx(0, 0, int64_t(sl.ez1) * sl.q), size_t(P), ncclDouble, r + 1, comm, s));
  if (sl.nranks_below) SB_NCCL(ncclRecv(v + sl.lidx(0, 0, int64_t(sl.ez0) * sl.q), size_t(P), ncclDouble, r - 1, comm, s));
  SB_NCCL(ncclGroupEnd());
}

void semlab_space_s::ax(const double* in, Epi epi, const EpiArgs& a, bool g32) {
  if (g32 && has_geom32())
    ctx->count(launch_ax_g32(sl, in, geom32.p, sync(), epi, a, ctx->stream));
  else
    ctx->count(launch_ax(sl, in, geom.p, sync(), epi, a, ctx->stream));
}

bool semlab_space_s::enable_geom32() {
  if (!ax_g32_supported(order)) return false;
  if (!has_geom32()) {
    geom32.alloc(size_t(E) * 6 * size_t(nloc));
    ctx->count(launch_to_f32(geom.p, geom32.p, E * 6 * nloc, ctx->stream));
  }
  return true;
}

void semlab_space_s::apply_A(const double* in, double* out, bool g32) {
  if (in == out) invalid("apply_A: in and out must not alias");
  EpiArgs a;
  a.w = out;
  ax(in, Epi::Write, a, g32);
  interface_sum(out);
  if (bc == SEMLAB_BC_NEUMANN) {  // r -= mean(r) (sem_space.cpp:207)
    if (ones.n < size_t(n)) {
      ones.alloc(size_t(n));
      ctx->count(launch_fill(ones.p, n, 1.0, ctx->stream));
    }
    const double* av[1] = {out};
    const double* bv[1] = {ones.p};
    double sum = 0.0;
    ctx->dots(1, av, bv, own_off(), own_len(), &sum, distributed());
    const double mean = sum / double(sl.Nx * sl.Ny * sl.Nz);
    ctx->count(launch_axpby(out, -mean, ones.p, 1.0, n, ctx->stream));
  }
}

const double* semlab_space_s::jacobi_inv() {
  if (!has_inv_diag) {
    DevBuf<double> d(static_cast<size_t>(n));
    stiffness_diag(d.p);
    inv_diag.alloc(size_t(n));
    ctx->count(launch_invert_masked(sl, d.p, inv_diag.p, ctx->stream));
    has_inv_diag = true;
  }
  return inv_diag.p;
}

void semlab_space_s::stiffness_diag(double* out) {
  DevBuf<double> loc(static_cast<size_t>(E * nloc));
  ctx->count(launch_local_diag(sl, geom.p, loc.p, ctx->stream));
  ctx->count(launch_fill(out, n, 0.0, ctx->stream));
  ctx->count(launch_gather(sl, loc.p, out, ctx->stream));
  interface_sum(out);
  ctx->count(launch_mask(sl, out, ctx->stream));
  ctx->sync();  // loc is freed on return
}

double semlab_space_s::dot(const double* a, const double* b) {
  const double* av[1] = {a};
  const double* bv[1] = {b};
  double r = 0.0;
  ctx->dots(1, av, bv, own_off(), own_len(), &r, distributed());
  return r;
}

// ------------------------------------------------------------------------------ operators
void semlab_op_s::apply(const double* in, double* out) {
  switch (kind) {
    case kA: space->apply_A(in, out, geom32); break;
    case kJacobi: ctx->count(launch_mul(out, space->jacobi_inv(), in, n, ctx->stream)); break;
    case kSchwarz: sch->apply(in, out); break;
    case kPmg: pmg->vcycle(in, out); break;
    case kSemfem: semfem_apply(semfem, in, out); break;
    case kCallback: fn(user, in, out); break;
    default: invalid("semlab_op: operator kind not available");
  }
}
