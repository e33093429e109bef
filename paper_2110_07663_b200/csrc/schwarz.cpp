#include <nccl.h>
// SchwarzSmoother: host setup restated from schwarz.cpp:46-214 (box lengths, extended 1-D
// operators, generalised eigendecomposition), device apply in k_fdm.cu.
#include "schwarz.hpp"

#include <cmath>
#include <cstring>

#include "capi_util.hpp"
#include "host_math.hpp"

using namespace sb;

namespace {

// Mean of the four edge arc lengths of element (ijk) along d, by the level's GLL rule
// (schwarz.cpp:53-86). Coordinates come from the mesh map on the global lattice axes, i.e. the
// same values HexMesh::lattice_coords produces (mesh.cpp:104-136).
double edge_length(const semlab_mesh_s& m, const Gll& g, const std::array<std::vector<double>, 3>& axis, int q,
                   const int ijk[3], int d) {
  double total = 0.0;
  std::vector<std::array<double, 3>> edge(size_t(q) + 1);
  const int nd = q + 1;
  for (int ca = 0; ca <= 1; ++ca)
    for (int cb = 0; cb <= 1; ++cb) {
      for (int mm = 0; mm <= q; ++mm) {
        int64_t idx[3];
        idx[d] = int64_t(ijk[d]) * q + mm;
        idx[(d + 1) % 3] = int64_t(ijk[(d + 1) % 3]) * q + ca * q;
        idx[(d + 2) % 3] = int64_t(ijk[(d + 2) % 3]) * q + cb * q;
        edge[size_t(mm)] = m.map(axis[0][size_t(idx[0])], axis[1][size_t(idx[1])], axis[2][size_t(idx[2])]);
      }
      double len = 0.0;
      for (int mm = 0; mm <= q; ++mm) {
        double t[3] = {0.0, 0.0, 0.0};
        for (int l = 0; l <= q; ++l) {
          const double dml = g.diff[size_t(mm + nd * l)];
          for (int c = 0; c < 3; ++c) t[c] += dml * edge[size_t(l)][c];
        }
        len += g.weights[size_t(mm)] * std::sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
      }
      total += len;
    }
  return total / 4.0;
}

}  // namespace

void semlab_schwarz_s::build() {
  semlab_space_s& sp = *space;
  const semlab_mesh_s& mesh = *sp.mesh;
  const int q = sp.order;
  if (q < 2) invalid("SchwarzSmoother: order must be >= 2");
  P = q + 3;
  const Slab& sl = sp.sl;
  const Gll& g = gll(q);
  const auto axis = mesh.lattice_axes(q);
  const int Ex = sl.Ex, Ey = sl.Ey, Ez = sl.Ez;
  // lengths for the slab plus one element layer on each side (ghost gaps of z-neighbours)
  const int lz0 = std::max(0, sl.ez0 - 1), lz1 = std::min(Ez, sl.ez1 + 1);
  const int64_t nlay = int64_t(Ex) * Ey;
  std::vector<double> len(size_t(nlay * (lz1 - lz0)) * 3);
  const bool par = mesh.kershaw_eps != 0.0;
  std::string err;
#pragma omp parallel for schedule(static) if (par)
  for (int64_t t = 0; t < nlay * (lz1 - lz0); ++t) {
    const int ijk[3] = {int(t % Ex), int((t / Ex) % Ey), lz0 + int(t / nlay)};
    for (int d = 0; d < 3; ++d) len[size_t(t) * 3 + d] = edge_length(mesh, g, axis, q, ijk, d);
  }
  for (size_t t = 0; t < len.size(); ++t)
    if (!(len[t] > 0.0)) numeric("SchwarzSmoother: degenerate element " + std::to_string(int64_t(t / 3) + lz0 * nlay));
  auto L_of = [&](int ex, int ey, int ez, int d) {
    return len[size_t((ex + int64_t(Ex) * (ey + int64_t(Ey) * (ez - lz0))) * 3 + d)];
  };
  const double gap01 = 0.5 * (g.nodes[1] - g.nodes[0]);
  const int nd = q + 1;
  std::vector<double> khat(size_t(nd) * nd);
  for (int i = 0; i < nd; ++i)
    for (int j = 0; j < nd; ++j) {
      double acc = 0.0;
      for (int m = 0; m < nd; ++m) acc += g.weights[size_t(m)] * g.diff[size_t(m + nd * i)] * g.diff[size_t(m + nd * j)];
      khat[size_t(i + nd * j)] = acc;
    }
  const int64_t E = sp.E;
  const bool dirichlet = sp.bc == SEMLAB_BC_DIRICHLET;
  hlen.assign(size_t(E) * 3, 0.0);
  hlam.assign(size_t(E) * 3 * P, 1.0);
  hn.assign(size_t(E) * 3, 0);
  std::vector<double> hS(size_t(E) * 3 * P * P, 0.0);
  int64_t bad = -1;
#pragma omp parallel for schedule(static)
  for (int64_t el = 0; el < E; ++el) {
    const int e3[3] = {int(el % Ex), int((el / Ex) % Ey), sl.ez0 + int(el / nlay)};
    const int Ed[3] = {Ex, Ey, Ez};
    std::vector<double> A(size_t(P) * P), B(size_t(P) * P), S(size_t(P) * P), lam(static_cast<size_t>(P));
    for (int d = 0; d < 3; ++d) {  // build_direction, schwarz.cpp:133-214
      const double L = L_of(e3[0], e3[1], e3[2], d);
      hlen[size_t(el) * 3 + d] = L;
      int nb_lo[3] = {e3[0], e3[1], e3[2]}, nb_hi[3] = {e3[0], e3[1], e3[2]};
      nb_lo[d] -= 1;
      nb_hi[d] += 1;
      const bool left_int = e3[d] > 0, right_int = e3[d] < Ed[d] - 1;
      const double gl_gap = left_int ? L_of(nb_lo[0], nb_lo[1], nb_lo[2], d) * gap01 : 0.0;
      const double gr_gap = right_int ? L_of(nb_hi[0], nb_hi[1], nb_hi[2], d) * gap01 : 0.0;
      const int i0 = (!left_int && dirichlet) ? 1 : 0;
      const int i1 = (!right_int && dirichlet) ? q - 1 : q;
      const int gl = left_int ? 1 : 0, gr = right_int ? 1 : 0;
      const int n = (i1 - i0 + 1) + gl + gr;
      hn[size_t(el) * 3 + d] = n;
      std::fill(A.begin(), A.end(), 0.0);
      std::fill(B.begin(), B.end(), 0.0);
      auto Am = [&](int a, int b) -> double& { return A[size_t(a + n * b)]; };
      auto Bm = [&](int a, int b) -> double& { return B[size_t(a + n * b)]; };
      for (int i = i0; i <= i1; ++i) {
        const int a = i - i0 + gl;
        Bm(a, a) += 0.5 * L * g.weights[size_t(i)];
        for (int j = i0; j <= i1; ++j) Am(a, j - i0 + gl) += (2.0 / L) * khat[size_t(i + nd * j)];
      }
      if (gl) {
        const double h = gl_gap;
        Am(0, 0) += 2.0 / h;
        Am(0, 1) += -1.0 / h;
        Am(1, 0) += -1.0 / h;
        Am(1, 1) += 1.0 / h;
        Bm(0, 0) += h;
        Bm(1, 1) += 0.5 * h;
      }
      if (gr) {
        const double h = gr_gap;
        const int last = n - 1;
        Am(last, last) += 2.0 / h;
        Am(last, last - 1) += -1.0 / h;
        Am(last - 1, last) += -1.0 / h;
        Am(last - 1, last - 1) += 1.0 / h;
        Bm(last, last) += h;
        Bm(last - 1, last - 1) += 0.5 * h;
      }
      if (!gen_sym_eig(n, A.data(), B.data(), lam.data(), S.data())) {
#pragma omp critical
        bad = bad < 0 ? el : std::min(bad, el);
        continue;
      }
      double* Sd = hS.data() + (size_t(el) * 3 + d) * P * P;
      for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) Sd[a * P + b] = S[size_t(a + n * b)];
      for (int a = 0; a < n; ++a) hlam[(size_t(el) * 3 + d) * P + a] = lam[size_t(a)];
    }
  }
  if (bad >= 0) numeric("SchwarzSmoother: eigensolve failed in element " + std::to_string(bad + int64_t(sl.ez0) * nlay));
  for (int64_t el = 0; el < E; ++el) {  // combined diagonal must be positive (schwarz.cpp:100-104)
    const double s0 = hlam[size_t(el) * 3 * P] + hlam[(size_t(el) * 3 + 1) * P] + hlam[(size_t(el) * 3 + 2) * P];
    if (!(s0 > 0.0))
      numeric("SchwarzSmoother: non-positive diagonal entry in element " + std::to_string(el + int64_t(sl.ez0) * nlay));
  }
  cudaStream_t s = sp.ctx->stream;
  const size_t nS = hS.size(), nL = hlam.size();
  if (precision == 32) {
    std::vector<float> fS(hS.begin(), hS.end()), fL(hlam.begin(), hlam.end());
    S.alloc(nS * sizeof(float));
    L.alloc(nL * sizeof(float));
    S.upload(reinterpret_cast<const unsigned char*>(fS.data()), nS * sizeof(float), s);
    L.upload(reinterpret_cast<const unsigned char*>(fL.data()), nL * sizeof(float), s);
    sp.ctx->sync();
  } else {
    S.alloc(nS * sizeof(double));
    L.alloc(nL * sizeof(double));
    S.upload(reinterpret_cast<const unsigned char*>(hS.data()), nS * sizeof(double), s);
    L.upload(reinterpret_cast<const unsigned char*>(hlam.data()), nL * sizeof(double), s);
    sp.ctx->sync();
  }
  if (mode == SEMLAB_SCHWARZ_ASM) boxes.alloc(size_t(E) * P * P * P * (precision == 32 ? 4 : 8));
}

void semlab_schwarz_s::ras(const double* r, int emode, const RasEpi& e) {
  space->ctx->count(launch_ras(space->sl, precision, S.p, L.p, r, emode, e, space->ctx->stream));
}

void semlab_schwarz_s::apply(const double* r, double* z) {
  if (r == z) invalid("SchwarzSmoother::apply: in and out must not alias");
  semlab_space_s& sp = *space;
  SB_CUDA(cudaMemsetAsync(z, 0, size_t(sp.n) * sizeof(double), sp.ctx->stream));
  if (sp.distributed()) {
    if (mode == SEMLAB_SCHWARZ_ASM && sp.sl.q < 3 && sp.sl.ez1 - sp.sl.ez0 < 2)
      invalid("SchwarzSmoother: ASM on slabs needs order >= 3 or >= 2 element layers per rank");
    // the ghost planes of a slab vector are scratch: fill them with the neighbours' planes
    sp.halo_exchange(const_cast<double*>(r));
  }
  if (mode == SEMLAB_SCHWARZ_RAS) {
    RasEpi e;
    e.out = z;
    ras(r, 0, e);
    sp.owner_copy_up(z);
  } else {
    const int64_t P2 = sp.sl.Nx * sp.sl.Ny;
    if (cnt.n < size_t(6 * P2)) cnt.alloc(size_t(6 * P2));
    sp.ctx->count(launch_asm(sp.sl, precision, S.p, L.p, r, boxes.p, z, cnt.p, sp.ctx->stream));
    if (sp.distributed()) asm_exchange(z);
  }
}

// ASM on z-slabs (schwarz.cpp:269-287 across ranks): the boxes of an element layer next to an
// internal boundary reach one lattice plane into the neighbour slab, so the neighbour's boxes add
// to this rank's planes zb, zb+1 (from below) and zt-1, zt (from above). Each rank sends its raw
// sums and counts on the planes its boxes share with a neighbour (zb-1, zb down; zt, zt+1 up),
// receives the neighbour's, and forms (lower sum + upper sum) / (lower count + upper count), the
// lower rank's (lower element ids) partial first; the ghost planes are zeroed.
void semlab_schwarz_s::asm_exchange(double* z) {
  semlab_space_s& sp = *space;
  const Slab& sl = sp.sl;
  const int64_t P2 = sl.Nx * sl.Ny;
  if (xch.n < size_t(8 * P2)) xch.alloc(size_t(8 * P2));
  ncclComm_t comm = static_cast<ncclComm_t>(sp.ctx->nccl);
  cudaStream_t s = sp.ctx->stream;
  const int r = sp.ctx->rank;
  const int64_t zb = int64_t(sl.ez0) * sl.q, zt = int64_t(sl.ez1) * sl.q;
  auto plane = [&](int64_t zz) { return z + sl.lidx(0, 0, zz); };
  auto cplane = [&](int k) { return cnt.p + k * P2; };
  auto rplane = [&](int k) { return xch.p + k * P2; };  // 0..3 from below, 4..7 from above
  SB_NCCL(ncclGroupStart());
  if (sl.nranks_below) {  // my (zb-1, zb) -> its (zt'-1, zt'); its (zt', zt'+1) -> my (zb, zb+1)
    SB_NCCL(ncclSend(plane(zb - 1), size_t(P2), ncclDouble, r - 1, comm, s));
    SB_NCCL(ncclSend(plane(zb), size_t(P2), ncclDouble, r - 1, comm, s));
    SB_NCCL(ncclSend(cplane(0), size_t(P2), ncclDouble, r - 1, comm, s));
    SB_NCCL(ncclSend(cplane(1), size_t(P2), ncclDouble, r - 1, comm, s));
    for (int k = 0; k < 4; ++k) SB_NCCL(ncclRecv(rplane(k), size_t(P2), ncclDouble, r - 1, comm, s));
  }
  if (sl.nranks_above) {  // my (zt, zt+1) -> its (zb', zb'+1); its (zb'-1, zb') -> my (zt-1, zt)
    SB_NCCL(ncclSend(plane(zt), size_t(P2), ncclDouble, r + 1, comm, s));
    SB_NCCL(ncclSend(plane(zt + 1), size_t(P2), ncclDouble, r + 1, comm, s));
    SB_NCCL(ncclSend(cplane(4), size_t(P2), ncclDouble, r + 1, comm, s));
    SB_NCCL(ncclSend(cplane(5), size_t(P2), ncclDouble, r + 1, comm, s));
    for (int k = 0; k < 4; ++k) SB_NCCL(ncclRecv(rplane(4 + k), size_t(P2), ncclDouble, r + 1, comm, s));
  }
  SB_NCCL(ncclGroupEnd());
  // from below the order is (sum zt', sum zt'+1, cnt zt', cnt zt'+1) = my (zb, zb+1)
  if (sl.nranks_below) {
    sp.ctx->count(launch_asm_combine(plane(zb), rplane(0), rplane(2), plane(zb), cplane(1), P2, s));
    sp.ctx->count(launch_asm_combine(plane(zb + 1), rplane(1), rplane(3), plane(zb + 1), cplane(2), P2, s));
    SB_CUDA(cudaMemsetAsync(plane(zb - 1), 0, size_t(P2) * sizeof(double), s));
  }
  // from above: (sum zb'-1, sum zb', cnt zb'-1, cnt zb') = my (zt-1, zt); mine first (lower ids)
  if (sl.nranks_above) {
    sp.ctx->count(launch_asm_combine(plane(zt - 1), plane(zt - 1), cplane(3), rplane(4), rplane(6), P2, s));
    sp.ctx->count(launch_asm_combine(plane(zt), plane(zt), cplane(4), rplane(5), rplane(7), P2, s));
    SB_CUDA(cudaMemsetAsync(plane(zt + 1), 0, size_t(P2) * sizeof(double), s));
  }
}

extern "C" {

int semlab_schwarz_create(semlab_space s, int mode, int precision, semlab_schwarz* out) {
  return guard([&] {
    need(s, "SchwarzSmoother: space");
    need(out, "SchwarzSmoother: out");
    if (mode != SEMLAB_SCHWARZ_ASM && mode != SEMLAB_SCHWARZ_RAS) invalid("SchwarzSmoother: unknown mode");
    if (precision != 32 && precision != 64) invalid("SchwarzSmoother: precision must be 32 or 64");
    auto sch = std::make_unique<semlab_schwarz_s>();
    sch->space = s;
    sch->mode = mode;
    sch->precision = precision;
    sch->build();
    *out = sch.release();
  });
}

int semlab_schwarz_destroy(semlab_schwarz sch) {
  return guard([&] {
    if (sch) cudaStreamSynchronize(sch->space->ctx->stream);
    delete sch;
  });
}

int semlab_schwarz_apply(semlab_schwarz sch, const double* r, double* z) {
  return guard([&] {
    need(sch, "SchwarzSmoother::apply: smoother");
    sch->apply(r, z);
  });
}

int semlab_schwarz_fdm_solve_all(semlab_schwarz sch, const double* in, double* out) {
  return guard([&] {
    need(sch, "fdm_solve: smoother");
    semlab_space_s& sp = *sch->space;
    sp.ctx->count(launch_fdm_boxes(sp.sl, sch->precision, sch->S.p, sch->L.p, in, out, sp.ctx->stream));
  });
}

int semlab_schwarz_element_info(semlab_schwarz sch, int e, double lengths[3], int n[3], double* lambda) {
  return guard([&] {
    need(sch, "element_info: smoother");
    if (e < 0 || e >= sch->space->E) invalid("element_info: element out of range");
    for (int d = 0; d < 3; ++d) {
      lengths[d] = sch->hlen[size_t(e) * 3 + d];
      n[d] = sch->hn[size_t(e) * 3 + d];
    }
    if (lambda) std::memcpy(lambda, sch->hlam.data() + size_t(e) * 3 * sch->P, sizeof(double) * 3 * sch->P);
  });
}

int semlab_op_schwarz(semlab_schwarz sch, semlab_op* out) {
  return guard([&] {
    need(sch, "semlab_op_schwarz: smoother");
    auto o = std::make_unique<semlab_op_s>();
    o->kind = semlab_op_s::kSchwarz;
    o->ctx = sch->space->ctx;
    o->n = sch->space->n;
    o->space = sch->space;
    o->sch = sch;
    *out = o.release();
  });
}

}  // extern "C"
