// p-multigrid: hierarchy setup, transfers, coarse solvers and the V-cycle (Alg. 1).
#include "pmg.hpp"

#include <cusolverDn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>

#include "capi_util.hpp"
#include "host_math.hpp"

using namespace sb;

namespace sb {

double HostCsr::coeff(int64_t i, int64_t j) const {
  const int* b = idx.data() + ptr[size_t(i)];
  const int* e = idx.data() + ptr[size_t(i) + 1];
  const int* it = std::lower_bound(b, e, int(j));
  return (it != e && *it == int(j)) ? val[size_t(it - idx.data())] : 0.0;
}

// Geometric factors of every element computed on the host exactly as the reference does
// (sem_space.cpp:58-97: J by D-contractions of the nodal coordinates, det and inverse by 3x3
// cofactors, G = (w det) (J^-1 J^-T) formed like Eigen's eager product), in plain IEEE double
// without FMA contraction. The coarse matrix is then bitwise the reference's, and so is its AMG
// hierarchy: aggregation breaks ties on exact comparisons (|a_ij| >= theta max, w > best,
// amg.cpp:17-52), so ulp-level differences in the entries (e.g. from the device k_geom, which
// fuses multiply-adds) would change aggregates. Layout as the device geometry: SoA per element.
static std::vector<double> host_geometry(semlab_space sp) {
  const int q = sp->order, nd = q + 1, nl = nd * nd * nd;
  const int64_t E = sp->E;
  const Slab& sl = sp->sl;
  const Gll& g = gll(q);
  const double* D = g.diff.data();  // D(i, m) = D[i + nd m]
  const double* W = g.weights.data();
  std::vector<double> geom(size_t(E) * 6 * nl);
  for (int64_t el = 0; el < E; ++el) {
    const int ex = int(el % sl.Ex), ey = int((el / sl.Ex) % sl.Ey), ez = sl.ez0 + int(el / (int64_t(sl.Ex) * sl.Ey));
    auto X = [&](int i, int j, int k, int c) {
      const int64_t gl = sl.lidx(int64_t(ex) * q + i, int64_t(ey) * q + j, int64_t(ez) * q + k);
      return sp->coords[size_t(gl) * 3 + size_t(c)];
    };
    for (int k = 0; k < nd; ++k)
      for (int j = 0; j < nd; ++j)
        for (int i = 0; i < nd; ++i) {
          double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
          for (int m = 0; m < nd; ++m)
            for (int c = 0; c < 3; ++c) {
              J[c][0] += D[i + nd * m] * X(m, j, k, c);
              J[c][1] += D[j + nd * m] * X(i, m, k, c);
              J[c][2] += D[k + nd * m] * X(i, j, m, c);
            }
          const double det = J[0][0] * (J[1][1] * J[2][2] - J[2][1] * J[1][2]) -
                             J[1][0] * (J[0][1] * J[2][2] - J[2][1] * J[0][2]) +
                             J[2][0] * (J[0][1] * J[1][2] - J[1][1] * J[0][2]);
          if (!(det > 0.0)) numeric("SemSpace: non-positive Jacobian in element " + std::to_string(el));
          const double w = W[i] * W[j] * W[k];
          const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1], c10 = J[1][2] * J[2][0] - J[1][0] * J[2][2],
                       c20 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
          const double idet = 1.0 / (J[0][0] * c00 + J[0][1] * c10 + J[0][2] * c20);
          double Ji[3][3];
          Ji[0][0] = c00 * idet;
          Ji[1][0] = c10 * idet;
          Ji[2][0] = c20 * idet;
          Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * idet;
          Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * idet;
          Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * idet;
          Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * idet;
          Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * idet;
          Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * idet;
          // P = Ji Ji^T column by column, l ascending, zero factors skipped (the eager product)
          double P[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
          for (int cj = 0; cj < 3; ++cj)
            for (int l = 0; l < 3; ++l) {
              const double b = Ji[cj][l];
              if (b == 0.0) continue;
              for (int r = 0; r < 3; ++r) P[r][cj] += Ji[r][l] * b;
            }
          const double s = w * det;
          const int node = i + nd * (j + nd * k);
          double* ge = geom.data() + size_t(el) * 6 * nl + node;
          ge[0 * nl] = s * P[0][0];
          ge[1 * nl] = s * P[0][1];
          ge[2 * nl] = s * P[0][2];
          ge[3 * nl] = s * P[1][1];
          ge[4 * nl] = s * P[1][2];
          ge[5 * nl] = s * P[2][2];
        }
  }
  return geom;
}

// Element matrices from the reference kernel applied to unit vectors (sem_space.cpp:127-175),
// assembled like setFromTriplets (duplicates summed in insertion order: ascending element).
HostCsr assemble_free_matrix(semlab_space sp) {
  if (sp->distributed()) invalid("coarse solve: assemble on a whole-mesh space");
  const int q = sp->order, nd = q + 1, nl = nd * nd * nd, nd2 = nd * nd;
  const int64_t E = sp->E;
  const Gll& g = gll(q);
  const double* D = g.diff.data();
  const Slab& sl = sp->sl;
  std::vector<double> geom = host_geometry(sp);
  const int64_t mb = sl.dirichlet ? 1 : 0;  // Dirichlet: the lattice boundary is masked out
  const int64_t fx = sl.Nx - 2 * mb, fy = sl.Ny - 2 * mb, fz = sl.Nz - 2 * mb;
  const int64_t nfree = fx * fy * fz;
  std::vector<std::vector<std::pair<int, double>>> rows(static_cast<size_t>(nfree));
  std::vector<double> in(static_cast<size_t>(nl)), out(static_cast<size_t>(nl)), ur(static_cast<size_t>(nl)), us(static_cast<size_t>(nl)), ut(static_cast<size_t>(nl));
  std::vector<double> Ae(size_t(nl) * nl);
  std::vector<int64_t> fidx(static_cast<size_t>(nl));
  for (int64_t el = 0; el < E; ++el) {
    const double* G = geom.data() + size_t(el) * 6 * nl;
    for (int c = 0; c < nl; ++c) {
      std::fill(in.begin(), in.end(), 0.0);
      in[size_t(c)] = 1.0;
      for (int k = 0; k < nd; ++k)
        for (int j = 0; j < nd; ++j)
          for (int i = 0; i < nd; ++i) {
            double dr = 0, ds = 0, dt = 0;
            for (int m = 0; m < nd; ++m) {
              dr += D[i + nd * m] * in[size_t(m + nd * j + nd2 * k)];
              ds += D[j + nd * m] * in[size_t(i + nd * m + nd2 * k)];
              dt += D[k + nd * m] * in[size_t(i + nd * j + nd2 * m)];
            }
            const int idx = i + nd * j + nd2 * k;
            ur[size_t(idx)] = dr;
            us[size_t(idx)] = ds;
            ut[size_t(idx)] = dt;
          }
      for (int idx = 0; idx < nl; ++idx) {
        const double r = ur[size_t(idx)], s = us[size_t(idx)], t = ut[size_t(idx)];
        const double g0 = G[0 * nl + idx], g1 = G[1 * nl + idx], g2 = G[2 * nl + idx];
        const double g3 = G[3 * nl + idx], g4 = G[4 * nl + idx], g5 = G[5 * nl + idx];
        ur[size_t(idx)] = g0 * r + g1 * s + g2 * t;
        us[size_t(idx)] = g1 * r + g3 * s + g4 * t;
        ut[size_t(idx)] = g2 * r + g4 * s + g5 * t;
      }
      for (int k = 0; k < nd; ++k)
        for (int j = 0; j < nd; ++j)
          for (int i = 0; i < nd; ++i) {
            double acc = 0;
            for (int m = 0; m < nd; ++m) {
              acc += D[m + nd * i] * ur[size_t(m + nd * j + nd2 * k)];
              acc += D[m + nd * j] * us[size_t(i + nd * m + nd2 * k)];
              acc += D[m + nd * k] * ut[size_t(i + nd * j + nd2 * m)];
            }
            Ae[size_t(i + nd * j + nd2 * k) + size_t(nl) * c] = acc;
          }
    }
    const int ex = int(el % sl.Ex), ey = int((el / sl.Ex) % sl.Ey), ez = int(el / (int64_t(sl.Ex) * sl.Ey));
    for (int k = 0; k < nd; ++k)
      for (int j = 0; j < nd; ++j)
        for (int i = 0; i < nd; ++i) {
          const int64_t x = int64_t(ex) * q + i, y = int64_t(ey) * q + j, z = int64_t(ez) * q + k;
          fidx[size_t(i + nd * j + nd2 * k)] =
              sl.masked(x, y, z) ? -1 : (x - mb) + fx * ((y - mb) + fy * (z - mb));
        }
    for (int c = 0; c < nl; ++c) {
      if (fidx[size_t(c)] < 0) continue;
      for (int r = 0; r < nl; ++r) {
        if (fidx[size_t(r)] < 0) continue;
        rows[size_t(fidx[size_t(r)])].push_back({int(fidx[size_t(c)]), Ae[size_t(r) + size_t(nl) * c]});
      }
    }
  }
  HostCsr A;
  A.n = A.m = nfree;
  A.ptr.assign(size_t(nfree) + 1, 0);
  for (int64_t i = 0; i < nfree; ++i) {
    auto& row = rows[size_t(i)];
    std::stable_sort(row.begin(), row.end(), [](auto& a, auto& b) { return a.first < b.first; });
    int last = -1;
    for (auto& kv : row) {
      if (kv.first == last) {
        A.val.back() += kv.second;
      } else {
        A.idx.push_back(kv.first);
        A.val.push_back(kv.second);
        last = kv.first;
      }
    }
    A.ptr[size_t(i) + 1] = int64_t(A.idx.size());
    std::vector<std::pair<int, double>>().swap(row);
  }
  return A;
}

// amg.cpp:12-65
std::vector<int> amg_aggregate(const HostCsr& A, double theta, int& n_agg) {
  const int64_t n = A.n;
  std::vector<std::vector<int>> strong(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    double row_max = 0.0;
    for (int64_t k = A.ptr[size_t(i)]; k < A.ptr[size_t(i) + 1]; ++k)
      if (A.idx[size_t(k)] != i) row_max = std::max(row_max, std::abs(A.val[size_t(k)]));
    if (row_max == 0.0) continue;
    const double cutoff = theta * row_max;
    for (int64_t k = A.ptr[size_t(i)]; k < A.ptr[size_t(i) + 1]; ++k) {
      const int j = A.idx[size_t(k)];
      if (j != i && std::abs(A.val[size_t(k)]) >= cutoff) strong[size_t(i)].push_back(j);
    }
  }
  std::vector<int> agg(size_t(n), -1);
  n_agg = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (agg[size_t(i)] >= 0) continue;
    bool clean = true;
    for (int j : strong[size_t(i)])
      if (agg[size_t(j)] >= 0) { clean = false; break; }
    if (!clean || strong[size_t(i)].empty()) continue;
    agg[size_t(i)] = n_agg;
    for (int j : strong[size_t(i)]) agg[size_t(j)] = n_agg;
    ++n_agg;
  }
  for (int64_t i = 0; i < n; ++i) {
    if (agg[size_t(i)] >= 0) continue;
    double best = 0.0;
    int best_agg = -1;
    for (int j : strong[size_t(i)]) {
      if (agg[size_t(j)] < 0) continue;
      const double w = std::abs(A.coeff(i, j));
      if (w > best) { best = w; best_agg = agg[size_t(j)]; }
    }
    if (best_agg >= 0) agg[size_t(i)] = best_agg;
  }
  for (int64_t i = 0; i < n; ++i)
    if (agg[size_t(i)] < 0) agg[size_t(i)] = n_agg++;
  return agg;
}

// Galerkin P^T A P for piecewise-constant P (amg.cpp:100-108): (P^T A)(I, j) = sum_{i in I} a_ij,
// then sum over j in J, both ascending.
static HostCsr galerkin(const HostCsr& A, const std::vector<int>& agg, int n_agg) {
  std::vector<std::vector<int>> members(static_cast<size_t>(n_agg));
  for (int64_t i = 0; i < A.n; ++i) members[size_t(agg[size_t(i)])].push_back(int(i));
  HostCsr C;
  C.n = C.m = n_agg;
  C.ptr.assign(size_t(n_agg) + 1, 0);
  std::map<int, double> rowj;
  std::map<int, double> rowJ;
  for (int I = 0; I < n_agg; ++I) {
    rowj.clear();
    rowJ.clear();
    for (int i : members[size_t(I)])
      for (int64_t k = A.ptr[size_t(i)]; k < A.ptr[size_t(i) + 1]; ++k) rowj[A.idx[size_t(k)]] += A.val[size_t(k)];
    for (auto& kv : rowj) rowJ[agg[size_t(kv.first)]] += kv.second;
    for (auto& kv : rowJ) {
      C.idx.push_back(kv.first);
      C.val.push_back(kv.second);
    }
    C.ptr[size_t(I) + 1] = int64_t(C.idx.size());
  }
  return C;
}

std::vector<AmgLevelHost> amg_build(const HostCsr& A0, double theta, int max_levels, int max_coarse_size) {
  std::vector<AmgLevelHost> levels;
  HostCsr current = A0;
  auto invd = [](const HostCsr& A, bool check) {
    std::vector<double> d(size_t(A.n));
    for (int64_t i = 0; i < A.n; ++i) {
      const double a = A.coeff(i, i);
      if (check && a == 0.0) numeric("AmgHierarchy: zero diagonal at row " + std::to_string(i));
      d[size_t(i)] = 1.0 / a;
    }
    return d;
  };
  bool stopped_uncoarsenable = false;
  while (int(levels.size()) < max_levels - 1 && current.n > max_coarse_size) {
    AmgLevelHost lvl;
    lvl.inv_diag = invd(current, true);
    int n_agg = 0;
    lvl.agg = amg_aggregate(current, theta, n_agg);
    lvl.n_agg = n_agg;
    if (n_agg >= current.n) {  // no coarsening possible: this level is the coarsest
      lvl.agg.clear();
      lvl.A = current;
      levels.push_back(std::move(lvl));
      stopped_uncoarsenable = true;
      break;
    }
    HostCsr coarse = galerkin(current, lvl.agg, n_agg);
    lvl.A = std::move(current);
    levels.push_back(std::move(lvl));
    current = std::move(coarse);
  }
  if (!stopped_uncoarsenable) {
    AmgLevelHost lvl;
    lvl.inv_diag = invd(current, false);
    lvl.A = std::move(current);
    levels.push_back(std::move(lvl));
  }
  return levels;
}

// Inverse of a dense SPD matrix (host column-major M) into a device buffer: cuSOLVER Cholesky
// (potrf) and a solve against the identity (potrs). Returns the factorization's info (0 = ok).
int device_spd_inverse(semlab_ctx ctx, int64_t n, const std::vector<double>& M, DevBuf<double>& inv) {
  cudaStream_t s = ctx->stream;
  std::vector<double> I(size_t(n) * n, 0.0);
  for (int64_t i = 0; i < n; ++i) I[size_t(i) + size_t(n) * i] = 1.0;
  DevBuf<double> dM(M.size());
  inv.alloc(I.size());
  dM.upload(M.data(), M.size(), s);
  inv.upload(I.data(), I.size(), s);
  cusolverDnHandle_t h;
  if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) fail(kCuda, "cusolverDnCreate failed");
  cusolverDnSetStream(h, s);
  int lwork = 0;
  cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, int(n), dM.p, int(n), &lwork);
  DevBuf<double> work(size_t(std::max(lwork, 1)));
  DevBuf<int> info(1);
  cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, int(n), dM.p, int(n), work.p, lwork, info.p);
  cusolverDnDpotrs(h, CUBLAS_FILL_MODE_LOWER, int(n), int(n), dM.p, int(n), inv.p, int(n), info.p);
  int hinfo = 0;
  SB_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  ctx->sync();
  cusolverDnDestroy(h);
  return hinfo;
}

bool dense_spd_inverse(int64_t n, std::vector<double>& M) {
  // Cholesky M = L L^T (lower, column-major), then inverse by solving for the identity.
  std::vector<double> L(M);
  for (int64_t j = 0; j < n; ++j) {
    double d = L[size_t(j + n * j)];
    for (int64_t k = 0; k < j; ++k) d -= L[size_t(j + n * k)] * L[size_t(j + n * k)];
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    L[size_t(j + n * j)] = d;
    for (int64_t i = j + 1; i < n; ++i) {
      double s = L[size_t(i + n * j)];
      for (int64_t k = 0; k < j; ++k) s -= L[size_t(i + n * k)] * L[size_t(j + n * k)];
      L[size_t(i + n * j)] = s / d;
    }
  }
  for (int64_t c = 0; c < n; ++c) {
    std::vector<double> y(size_t(n), 0.0);
    for (int64_t i = 0; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int64_t k = 0; k < i; ++k) s -= L[size_t(i + n * k)] * y[size_t(k)];
      y[size_t(i)] = s / L[size_t(i + n * i)];
    }
    for (int64_t i = n - 1; i >= 0; --i) {
      double s = y[size_t(i)];
      for (int64_t k = i + 1; k < n; ++k) s -= L[size_t(k + n * i)] * M[size_t(k + n * c)];
      M[size_t(i + n * c)] = s / L[size_t(i + n * i)];
    }
  }
  return true;
}

// ------------------------------------------------------------------------ coarse solver
void CoarseSolver::build(semlab_space space, int m) {
  sp = space;
  mode = m;
  HostCsr A = assemble_free_matrix(sp);
  nfree = A.n;
  cudaStream_t s = sp->ctx->stream;
  rf.alloc(size_t(nfree));
  zf.alloc(size_t(nfree));
  neumann = sp->bc == SEMLAB_BC_NEUMANN;
  if (neumann && mode != SEMLAB_COARSE_DIRECT)
    invalid("pmg: the Neumann coarse problem is singular; it needs SEMLAB_COARSE_DIRECT (nullspace projection)");
  if (mode == SEMLAB_COARSE_DIRECT) {
    if (nfree > 20000)
      invalid("coarse direct solve is limited to 20000 free dofs (got " + std::to_string(nfree) +
              "); use SEMLAB_COARSE_AMG");
    std::vector<double> M(size_t(nfree) * nfree, 0.0);
    for (int64_t i = 0; i < nfree; ++i)
      for (int64_t k = A.ptr[size_t(i)]; k < A.ptr[size_t(i) + 1]; ++k) M[size_t(i) + size_t(nfree) * A.idx[size_t(k)]] = A.val[size_t(k)];
    // Neumann: A has the constants as its nullspace. A + 1 1^T / n is SPD and,
    // on zero-mean right-hand sides, has the zero-mean solution of A e = r.
    if (neumann)
      for (auto& v : M) v += 1.0 / double(nfree);
    const int hinfo = device_spd_inverse(sp->ctx, nfree, M, Minv);
    if (hinfo != 0) numeric("coarse solve: factorization failed (info " + std::to_string(hinfo) + ")");
    if (neumann) {  // e = Pi M^-1 Pi r with Pi = I - 1 1^T / n: the mean of e is 0
      std::vector<double> H(M.size());
      Minv.download(H.data(), H.size(), s);
      sp->ctx->sync();
      const int64_t nn = nfree;
      std::vector<double> rm(size_t(nn), 0.0), cm(size_t(nn), 0.0);
      double tm = 0.0;
      for (int64_t j = 0; j < nn; ++j)
        for (int64_t i = 0; i < nn; ++i) {
          const double v = H[size_t(i + nn * j)];
          rm[size_t(i)] += v;
          cm[size_t(j)] += v;
          tm += v;
        }
      for (int64_t j = 0; j < nn; ++j)
        for (int64_t i = 0; i < nn; ++i)
          H[size_t(i + nn * j)] += -rm[size_t(i)] / double(nn) - cm[size_t(j)] / double(nn) + tm / double(nn * nn);
      Minv.upload(H.data(), H.size(), s);
      sp->ctx->sync();
    }
    return;
  }
  build_amg(space, A);
}

// AMG (amg.cpp:69-129) of a host matrix: host setup, device V-cycle; the coarsest level's dense
// LDLT (amg.cpp:124-126) becomes a dense inverse (cuSOLVER) applied by one symmetric GEMV.
void CoarseSolver::build_amg(semlab_space space, const HostCsr& A) {
  sp = space;
  mode = SEMLAB_COARSE_AMG;
  nfree = A.n;
  cudaStream_t s = sp->ctx->stream;
  if (rf.n < size_t(nfree)) {
    rf.alloc(size_t(nfree));
    zf.alloc(size_t(nfree));
  }
  auto hl = amg_build(A);
  lev.resize(hl.size());
  for (size_t l = 0; l < hl.size(); ++l) {
    Lev& L = lev[l];
    const AmgLevelHost& H = hl[l];
    L.n = H.A.n;
    L.ptr.alloc(H.A.ptr.size());
    L.ptr.upload(H.A.ptr.data(), H.A.ptr.size(), s);
    L.idx.alloc(std::max<size_t>(H.A.idx.size(), 1));
    if (!H.A.idx.empty()) L.idx.upload(H.A.idx.data(), H.A.idx.size(), s);
    L.val.alloc(std::max<size_t>(H.A.val.size(), 1));
    if (!H.A.val.empty()) L.val.upload(H.A.val.data(), H.A.val.size(), s);
    L.inv_diag.alloc(size_t(L.n));
    L.inv_diag.upload(H.inv_diag.data(), size_t(L.n), s);
    L.r.alloc(size_t(L.n));
    L.z.alloc(size_t(L.n));
    L.t.alloc(size_t(L.n));
    if (!H.agg.empty()) {
      L.nc = H.n_agg;
      L.agg.alloc(H.agg.size());
      L.agg.upload(H.agg.data(), H.agg.size(), s);
      std::vector<int64_t> aptr(size_t(H.n_agg) + 1, 0);
      for (int a : H.agg) aptr[size_t(a) + 1]++;
      for (int I = 0; I < H.n_agg; ++I) aptr[size_t(I) + 1] += aptr[size_t(I)];
      std::vector<int> amem(H.agg.size());
      std::vector<int64_t> fillp(aptr.begin(), aptr.end() - 1);
      for (int64_t i = 0; i < L.n; ++i) amem[size_t(fillp[size_t(H.agg[size_t(i)])]++)] = int(i);
      L.aptr.alloc(aptr.size());
      L.aptr.upload(aptr.data(), aptr.size(), s);
      L.amem.alloc(amem.size());
      L.amem.upload(amem.data(), amem.size(), s);
    }
  }
  const HostCsr& Ac = hl.back().A;
  coarse_n = Ac.n;
  if (coarse_n > 20000)  // the reference factors it densely (amg.cpp:124-126): infeasible beyond this
    numeric("AmgHierarchy: coarsest level has " + std::to_string(coarse_n) +
            " rows (aggregation stalled); too large for the dense coarse solve");
  std::vector<double> M(size_t(coarse_n) * coarse_n, 0.0);
  for (int64_t i = 0; i < coarse_n; ++i)
    for (int64_t k = Ac.ptr[size_t(i)]; k < Ac.ptr[size_t(i) + 1]; ++k)
      M[size_t(i) + size_t(coarse_n) * Ac.idx[size_t(k)]] = Ac.val[size_t(k)];
  if (device_spd_inverse(sp->ctx, coarse_n, M, coarse_inv) != 0) numeric("AmgHierarchy: coarse factorization failed");
  (void)s;
}

// AmgHierarchy::cycle (amg.cpp:140-160) with pre = post = 1 damped-Jacobi sweeps.
void CoarseSolver::amg_cycle(int l, const double* r, double* z) {
  semlab_ctx c = sp->ctx;
  cudaStream_t s = c->stream;
  Lev& L = lev[size_t(l)];
  if (l == int(lev.size()) - 1) {
    c->count(launch_symv(coarse_inv.p, coarse_n, r, z, s));
    return;
  }
  const CsrDev A{L.n, L.ptr.p, L.idx.p, L.val.p};
  c->count(launch_amg_jacobi0(L.inv_diag.p, omega, r, z, L.n, s));
  Lev& N = lev[size_t(l) + 1];
  c->count(launch_amg_restrict_split(A, L.aptr.p, L.amem.p, L.nc, r, z, L.t.p, N.r.p, s));
  amg_cycle(l + 1, N.r.p, N.z.p);
  c->count(launch_amg_prolong(L.agg.p, N.z.p, z, L.n, s));
  c->count(launch_amg_relax(A, L.inv_diag.p, omega, r, z, L.t.p, s));
  c->count(launch_copy(z, L.t.p, L.n, s));
}

void CoarseSolver::solve(const double* r_full, double* z_full) {
  semlab_ctx c = sp->ctx;
  cudaStream_t s = c->stream;
  c->count(launch_gather_free(sp->sl, r_full, rf.p, s));
  if (mode == SEMLAB_COARSE_DIRECT)
    c->count(launch_symv(Minv.p, nfree, rf.p, zf.p, s));
  else
    amg_cycle(0, rf.p, zf.p);
  c->count(launch_scatter_free(sp->sl, zf.p, z_full, s));
}

// Distributed coarse level: every rank contributes its owned p=1 planes (ncclAllGather of
// equal-size padded blocks), solves the whole coarse problem redundantly, and keeps its slab.
void CoarseSolver::solve_dist(semlab_space dsp, const double* r_loc, double* z_loc) {
  semlab_ctx c = dsp->ctx;
  cudaStream_t s = c->stream;
  const Slab& ls = dsp->sl;
  const int64_t P = ls.Nx * ls.Ny;
  const int R = c->nranks;
  int64_t maxpl = 0;
  std::vector<int64_t> z0(static_cast<size_t>(R)), z1(static_cast<size_t>(R));
  for (int k = 0; k < R; ++k) {
    const Slab sk = make_slab(ls.q, ls.Ex, ls.Ey, ls.Ez, k, R, ls.dirichlet != 0);
    z0[size_t(k)] = sk.own_z0();
    z1[size_t(k)] = sk.own_z1();
    maxpl = std::max(maxpl, z1[size_t(k)] - z0[size_t(k)]);
  }
  if (gsend.n < size_t(maxpl * P)) {
    gsend.alloc(size_t(maxpl * P));
    grecv.alloc(size_t(maxpl * P * R));
    rfull.alloc(size_t(sp->n));
    zfull.alloc(size_t(sp->n));
  }
  const int me = c->rank;
  SB_CUDA(cudaMemcpyAsync(gsend.p, r_loc + ls.lidx(0, 0, z0[size_t(me)]),
                          size_t((z1[size_t(me)] - z0[size_t(me)]) * P) * sizeof(double), cudaMemcpyDeviceToDevice, s));
  ncclResult_t rr = ncclAllGather(gsend.p, grecv.p, size_t(maxpl * P), ncclDouble, static_cast<ncclComm_t>(c->nccl), s);
  if (rr != ncclSuccess) fail(kNccl, std::string("ncclAllGather: ") + ncclGetErrorString(rr));
  for (int k = 0; k < R; ++k)
    SB_CUDA(cudaMemcpyAsync(rfull.p + z0[size_t(k)] * P, grecv.p + size_t(k) * maxpl * P,
                            size_t((z1[size_t(k)] - z0[size_t(k)]) * P) * sizeof(double), cudaMemcpyDeviceToDevice, s));
  solve(rfull.p, zfull.p);
  SB_CUDA(cudaMemcpyAsync(z_loc, zfull.p + ls.zlo * P, size_t(ls.nzl * P) * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

}  // namespace sb

// ------------------------------------------------------------------------ hierarchy
static Grid3 grid_of(const Slab& sl) {
  Grid3 g;
  g.N[0] = sl.Nx;
  g.N[1] = sl.Ny;
  g.N[2] = sl.Nz;
  g.nxl = sl.Nx;
  g.nyl = sl.Ny;
  g.zoff = sl.zlo;
  g.dirichlet = sl.dirichlet;
  return g;
}

semlab_pmg_s::~semlab_pmg_s() {
  if (ctx) cudaStreamSynchronize(ctx->stream);
  if (graph_exec) cudaGraphExecDestroy(graph_exec);
  for (auto& L : lv) {
    delete L.cheb;
    delete L.A;
    delete L.S;
    delete L.sch;
    delete L.sp;
  }
  delete coarse_full;
}

#ifndef SEMLAB_SMOOTHER_GEOM32
#define SEMLAB_SMOOTHER_GEOM32 1  // build-time A/B: 0 = FP64 factors in the FP32 smoother's operator
#endif
static constexpr bool smoother_geom32() { return SEMLAB_SMOOTHER_GEOM32 != 0; }

void semlab_pmg_s::build() {
  const size_t nl = orders.size();
  if (nl < 2) invalid("pmg: schedule needs at least two levels");
  for (size_t l = 0; l + 1 < nl; ++l)
    if (!(orders[l] > orders[l + 1])) invalid("pmg: schedule must be strictly decreasing");
  if (orders.back() != 1) invalid("pmg: schedule must end at order 1");
  lv.resize(nl);
  for (size_t l = 0; l < nl; ++l) {
    Level& L = lv[l];
    auto sp = std::make_unique<semlab_space_s>();
    sp->ctx = ctx;
    sp->mesh = mesh;
    sp->order = orders[l];
    sp->bc = bc;
    sp->build();
    L.sp = sp.release();
    const int64_t n = L.sp->n;
    L.b.alloc(size_t(n));
    L.x.alloc(size_t(n));
    if (plain()) {
      L.t.alloc(size_t(n));
      L.t.zero(ctx->stream);
    }
    L.r.alloc(size_t(n));
    L.b.zero(ctx->stream);
    L.x.zero(ctx->stream);
    L.r.zero(ctx->stream);
    if (l + 1 == nl) break;
    L.A = new semlab_op_s;
    L.A->kind = semlab_op_s::kA;
    L.A->ctx = ctx;
    L.A->n = n;
    L.A->space = L.sp;
    // FP32 smoother (the paper's setting): its operator applications use FP32-rounded
    // geometric factors too (FP64 arithmetic); the Krylov operator keeps the FP64 factors.
    if (precision == 32 && smoother_geom32()) L.A->geom32 = L.sp->enable_geom32();
    L.S = new semlab_op_s;
    L.S->ctx = ctx;
    L.S->n = n;
    L.S->space = L.sp;
    if (smoother == SEMLAB_SMOOTHER_JACOBI) {
      L.S->kind = semlab_op_s::kJacobi;
      L.sp->jacobi_inv();
    } else {
      auto sch = std::make_unique<semlab_schwarz_s>();
      sch->space = L.sp;
      sch->mode = (smoother == SEMLAB_SMOOTHER_RAS || smoother == SEMLAB_SMOOTHER_RAS_PLAIN) ? SEMLAB_SCHWARZ_RAS
                                                                                             : SEMLAB_SCHWARZ_ASM;
      sch->precision = precision;
      sch->build();
      L.sch = sch.release();
      L.S->kind = semlab_op_s::kSchwarz;
      L.S->sch = L.sch;
    }
    if (plain()) continue;  // un-accelerated smoothers: no Chebyshev, no lambda estimate
    L.lam = estimate_lambda_max(L.S, L.A, n, 10, 0).value;
    if (!(L.lam > 0.0)) numeric("pmg: lambda estimate failed on level " + std::to_string(l));
    semlab_cheby_params p{cheb_order, lmin, lmax, L.lam};
    L.cheb = new semlab_cheby_s;
    L.cheb->init(L.S, L.A, p);
  }
  J.resize(nl - 1);
  size_t scratch = 0;
  for (size_t l = 0; l + 1 < nl; ++l) {
    const int qf = orders[l], qc = orders[l + 1];
    const auto Jv = lagrange_interpolation_matrix(gll(qc).nodes, gll(qf).nodes);
    J[l] = Jmat{};
    for (size_t t = 0; t < Jv.size(); ++t) J[l].v[t] = Jv[t];
    const Slab& f = lv[l].sp->sl;
    const Slab& c = lv[l + 1].sp->sl;
    scratch = std::max<size_t>(scratch, size_t(c.Nx * f.Ny * f.nzl));
  }
  tA.alloc(scratch);
  tB.alloc(scratch);
  if (lv.back().sp->distributed()) {
    auto full = std::make_unique<semlab_space_s>();
    full->ctx = ctx;
    full->mesh = mesh;
    full->order = orders.back();
    full->bc = bc;
    full->full = true;
    full->build();
    coarse_full = full.release();
    coarse.build(coarse_full, coarse_mode);
  } else {
    coarse.build(lv.back().sp, coarse_mode);
  }
  ctx->sync();
}

// P: coarse level l+1 -> fine level l (three 1-D passes: z, y, x)
void semlab_pmg_s::prolong(int l, const double* cv, double* fv, bool add) {
  const Slab& f = lv[size_t(l)].sp->sl;
  const Slab& c = lv[size_t(l) + 1].sp->sl;
  const int qf = f.q, qc = c.q;
  cudaStream_t s = ctx->stream;
  Grid3 gc = grid_of(c), gf = grid_of(f);
  Grid3 g1 = gc;  // (Ncx, Ncy, fine z)
  g1.N[2] = f.Nz;
  g1.zoff = f.zlo;
  Grid3 g2 = g1;  // (Ncx, Nfy, fine z)
  g2.N[1] = f.Ny;
  g2.nyl = f.Ny;
  const int64_t zb = int64_t(f.ez0) * qf, nz = int64_t(f.ez1 - f.ez0) * qf + 1;
  ctx->count(launch_transfer_pass(true, cv, gc, tA.p, g1, 2, J[size_t(l)], qf, qc, f.Ez, true, gc, false, gf, zb, nz, s));
  ctx->count(launch_transfer_pass(true, tA.p, g1, tB.p, g2, 1, J[size_t(l)], qf, qc, f.Ey, false, gc, false, gf, zb, nz, s));
  ctx->count(launch_transfer_pass(true, tB.p, g2, fv, gf, 0, J[size_t(l)], qf, qc, f.Ex, false, gc, true, gf, zb, nz, s, add));
}

// P^T: fine level l -> coarse level l+1 (passes x, y, z)
void semlab_pmg_s::restrict_(int l, const double* fv, double* cv, const double* sub_from) {
  const Slab& f = lv[size_t(l)].sp->sl;
  const Slab& c = lv[size_t(l) + 1].sp->sl;
  const int qf = f.q, qc = c.q;
  cudaStream_t s = ctx->stream;
  Grid3 gc = grid_of(c), gf = grid_of(f);
  Grid3 g1 = gf;  // (Ncx, Nfy, fine z)
  g1.N[0] = c.Nx;
  g1.nxl = c.Nx;
  Grid3 g2 = g1;  // (Ncx, Ncy, fine z)
  g2.N[1] = c.Ny;
  g2.nyl = c.Ny;
  const int64_t zbf = int64_t(f.ez0) * qf, nzf = int64_t(f.ez1 - f.ez0) * qf + 1;
  const int64_t zbc = int64_t(c.ez0) * qc, nzc = int64_t(c.ez1 - c.ez0) * qc + 1;
  ctx->count(launch_transfer_pass(false, fv, gf, tA.p, g1, 0, J[size_t(l)], qf, qc, f.Ex, true, gf, false, gc, zbf, nzf, s,
                                  false, sub_from));
  ctx->count(launch_transfer_pass(false, tA.p, g1, tB.p, g2, 1, J[size_t(l)], qf, qc, f.Ey, false, gf, false, gc, zbf, nzf, s));
  Jmat Jz = J[size_t(l)];
  Jz.e_lo = f.ez0;  // z: only this slab's element layers contribute; the other rank's part
  Jz.e_hi = f.ez1;  // arrives through the interface-plane sum below
  ctx->count(launch_transfer_pass(false, tB.p, g2, cv, gc, 2, Jz, qf, qc, f.Ez, false, gf, true, gc, zbc, nzc, s));
  lv[size_t(l) + 1].sp->interface_sum(cv);
}

// Alg. 1 with x0 = 0: pre-smooth, residual, restrict, recurse, correct, post-smooth.
void semlab_pmg_s::cycle(int l) {
  Level& L = lv[size_t(l)];
  if (l == int(lv.size()) - 1) {
    if (coarse_full)
      coarse.solve_dist(L.sp, L.b.p, L.x.p);
    else
      coarse.solve(L.b.p, L.x.p);
    return;
  }
  smooth(l, true);
  // r = b - A x is not stored: the first restriction pass reads b and A x (bitwise the same
  // b - Ax), so the Ax keeps the plain-write epilogue
  L.sp->apply_A(L.x.p, L.r.p, L.A->geom32);  // (+ the interface-plane sum on a slab)
  restrict_(l, L.r.p, lv[size_t(l) + 1].b.p, L.b.p);
  cycle(l + 1);
  prolong(l, lv[size_t(l) + 1].x.p, L.x.p, true);  // x += P e_C (fused into the last pass)
  smooth(l, false);
}

// One smoothing step on level l: Chebyshev(eta) of the level's S (chebyshev.cpp:76-96), or the
// un-accelerated smoother: x = S b from x = 0, else x += S (b - A x).
void semlab_pmg_s::smooth(int l, bool x_is_zero) {
  Level& L = lv[size_t(l)];
  cudaStream_t s = ctx->stream;
  const int64_t n = L.sp->n;
  if (x_is_zero) SB_CUDA(cudaMemsetAsync(L.x.p, 0, size_t(n) * sizeof(double), s));
  if (!plain()) {
    L.cheb->smooth(L.b.p, L.x.p, x_is_zero);
    return;
  }
  if (x_is_zero) {
    L.S->apply(L.b.p, L.x.p);
    return;
  }
  L.sp->apply_A(L.x.p, L.r.p, L.A->geom32);
  ctx->count(launch_sub(L.r.p, L.b.p, L.r.p, n, s));  // r = b - A x
  L.S->apply(L.r.p, L.t.p);
  ctx->count(launch_axpby(L.x.p, 1.0, L.t.p, 1.0, n, s));
}

// Additive V-cycle (§2.2.2 "an additive V-cycle with no post-smoothing is
// used to avoid residual re-evaluation"): every level smooths its restricted right-hand side
// b_{l+1} = P^T b_l from x = 0, the coarsest level is solved, and the corrections are summed
// upwards, x_l += P x_{l+1}. No residual is re-evaluated and there is no post-smoothing.
void semlab_pmg_s::cycle_additive(int l) {
  Level& L = lv[size_t(l)];
  if (l == int(lv.size()) - 1) {
    if (coarse_full)
      coarse.solve_dist(L.sp, L.b.p, L.x.p);
    else
      coarse.solve(L.b.p, L.x.p);
    return;
  }
  restrict_(l, L.b.p, lv[size_t(l) + 1].b.p);
  smooth(l, true);
  cycle_additive(l + 1);
  prolong(l, lv[size_t(l) + 1].x.p, L.x.p, true);
}

#ifndef SEMLAB_PMG_GRAPH
#define SEMLAB_PMG_GRAPH 1  // build-time A/B: 0 = the V-cycle launched kernel by kernel
#endif
static constexpr bool pmg_graph_enabled() { return SEMLAB_PMG_GRAPH != 0; }

// The V-cycle body works on the hierarchy's own buffers only (the input and output are copied
// in and out), so after one eager warm-up call (lazy allocations, per-kernel launch setup) it is
// captured once as a CUDA graph, NCCL exchanges included, and replayed: one launch per cycle
// instead of ~100, no host launch gaps between the small coarse-level kernels.
void semlab_pmg_s::run_cycle() {
  cudaStream_t s = ctx->stream;
  if (!pmg_graph_enabled() || graph_state < 0) {
    run_body();
    return;
  }
  if (graph_state == 0) {  // eager warm-up
    run_body();
    graph_state = 1;
    return;
  }
  if (graph_state == 1) {
    const int64_t before = ctx->launches;
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      try {
        run_body();
      } catch (...) {
        ok = false;
      }
      ok = (cudaStreamEndCapture(s, &g) == cudaSuccess) && ok && g != nullptr;
    }
    if (ok) ok = cudaGraphInstantiate(&graph_exec, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    graph_launches = ctx->launches - before;
    ctx->launches = before;  // the capture executed nothing
    if (!ok) {
      (void)cudaGetLastError();
      graph_state = -1;  // not capturable here: stay eager
      run_body();
      return;
    }
    graph_state = 2;
  }
  SB_CUDA(cudaGraphLaunch(graph_exec, s));
  ctx->count(graph_launches);
}

void semlab_pmg_s::run_body() {
  if (cycle_mode == SEMLAB_CYCLE_ADDITIVE)
    cycle_additive(0);
  else
    cycle(0);
}

void semlab_pmg_s::vcycle(const double* b, double* z) {
  const int64_t n = lv[0].sp->n;
  ctx->count(launch_copy(lv[0].b.p, b, n, ctx->stream));
  run_cycle();
  ctx->count(launch_copy(z, lv[0].x.p, n, ctx->stream));
}

extern "C" {

int semlab_pmg_create_ex(semlab_mesh mesh, int nlevels, const int* orders, const semlab_pmg_options* o,
                         semlab_pmg* out) {
  return guard([&] {
    need(mesh, "pmg: mesh");
    need(orders, "pmg: orders");
    need(o, "pmg: options");
    need(out, "pmg: out");
    if (o->smoother < 0 || o->smoother > SEMLAB_SMOOTHER_ASM_PLAIN) invalid("pmg: unknown smoother");
    if (o->coarse != SEMLAB_COARSE_DIRECT && o->coarse != SEMLAB_COARSE_AMG) invalid("pmg: unknown coarse solver");
    if (o->precision != 32 && o->precision != 64) invalid("pmg: precision must be 32 or 64");
    if (o->bc != SEMLAB_BC_DIRICHLET && o->bc != SEMLAB_BC_NEUMANN) invalid("pmg: unknown boundary condition");
    if (o->cycle != SEMLAB_CYCLE_STANDARD && o->cycle != SEMLAB_CYCLE_ADDITIVE) invalid("pmg: unknown cycle");
    auto p = std::make_unique<semlab_pmg_s>();
    p->ctx = mesh->ctx;
    p->mesh = mesh;
    p->orders.assign(orders, orders + nlevels);
    p->smoother = o->smoother;
    p->cheb_order = o->cheb_order;
    p->lmin = o->lambda_min_mult;
    p->lmax = o->lambda_max_mult;
    p->precision = o->precision;
    p->coarse_mode = o->coarse;
    p->bc = o->bc;
    p->cycle_mode = o->cycle;
    // the Neumann mean removal synchronises the host (reductions): those cycles run eagerly
    if (p->bc == SEMLAB_BC_NEUMANN) p->graph_state = -1;
    p->build();
    *out = p.release();
  });
}

int semlab_pmg_create(semlab_mesh mesh, int nlevels, const int* orders, int smoother, int cheb_order, double lmin,
                      double lmax, int precision, int coarse, semlab_pmg* out) {
  if (smoother < 0 || smoother > SEMLAB_SMOOTHER_ASM) {
    sb_set_error("pmg: unknown smoother");
    return SEMLAB_EINVAL;
  }
  const semlab_pmg_options o{smoother, cheb_order, lmin, lmax, precision, coarse, SEMLAB_BC_DIRICHLET,
                             SEMLAB_CYCLE_STANDARD};
  return semlab_pmg_create_ex(mesh, nlevels, orders, &o, out);
}

int semlab_pmg_destroy(semlab_pmg p) {
  return guard([&] { delete p; });
}

int semlab_pmg_vcycle(semlab_pmg p, const double* b, double* z) {
  return guard([&] {
    need(p, "pmg: hierarchy");
    p->vcycle(b, z);
  });
}

int semlab_pmg_space(semlab_pmg p, int level, semlab_space* out) {
  return guard([&] {
    need(p, "pmg: hierarchy");
    if (level < 0 || level >= int(p->lv.size())) invalid("pmg: level out of range");
    *out = p->lv[size_t(level)].sp;
  });
}

int semlab_pmg_coarse_info(semlab_pmg p, int* nlevels, int64_t* sizes, int cap) {
  return guard([&] {
    need(p, "pmg: hierarchy");
    need(nlevels, "pmg_coarse_info: nlevels");
    const auto& lev = p->coarse.lev;
    *nlevels = int(lev.size());
    for (int l = 0; l < int(lev.size()) && l < cap; ++l) sizes[l] = lev[size_t(l)].n;
  });
}

int semlab_pmg_lambda(semlab_pmg p, int level, double* out) {
  return guard([&] {
    need(p, "pmg: hierarchy");
    if (level < 0 || level + 1 >= int(p->lv.size())) invalid("pmg: level has no smoother");
    *out = p->lv[size_t(level)].lam;
  });
}

int semlab_pmg_prolong(semlab_pmg p, int level, const double* c, double* f) {
  return guard([&] {
    need(p, "pmg: hierarchy");
    if (level < 0 || level + 1 >= int(p->lv.size())) invalid("pmg: level out of range");
    p->prolong(level, c, f);
  });
}

int semlab_pmg_restrict(semlab_pmg p, int level, const double* f, double* c) {
  return guard([&] {
    need(p, "pmg: hierarchy");
    if (level < 0 || level + 1 >= int(p->lv.size())) invalid("pmg: level out of range");
    p->restrict_(level, f, c);
  });
}

int semlab_op_pmg(semlab_pmg p, semlab_op* out) {
  return guard([&] {
    need(p, "semlab_op_pmg: hierarchy");
    auto o = std::make_unique<semlab_op_s>();
    o->kind = semlab_op_s::kPmg;
    o->ctx = p->ctx;
    o->n = p->lv[0].sp->n;
    o->space = p->lv[0].sp;
    o->pmg = p;
    *out = o.release();
  });
}

}  // extern "C"
