// Chebyshev smoother (chebyshev.cpp:58-96), lambda estimate (chebyshev.cpp:9-56), restarted
// GMRES (krylov.cpp:20-129) and a restated PCG, all over device-resident vectors. The host only
// keeps the small scalars (Hessenberg, Givens, Chebyshev coefficients) and synchronises once per
// Krylov iteration.
#include "solvers.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "host_math.hpp"
#include "capi_util.hpp"
#include "schwarz.hpp"

#include <memory>

using namespace sb;

namespace {

cudaStream_t st(semlab_ctx c) { return c->stream; }

// Fused Chebyshev-Jacobi needs S = diag(A)^-1 of the same space and a single rank (interface
// planes need the cross-rank sum before the owner epilogue).
#ifndef SEMLAB_DIST_FUSED
#define SEMLAB_DIST_FUSED 1  // build-time A/B: 0 = the generic Chebyshev path on z-slabs
#endif
constexpr bool dist_ras_enabled() { return SEMLAB_DIST_FUSED != 0; }

// The fused paths apply A through the Ax epilogues, which do not remove the mean: Neumann
// spaces (sem_space.cpp:207) take the generic path (A->apply, then S->apply).
bool fused_jacobi(semlab_op S, semlab_op A) {
  return S->kind == semlab_op_s::kJacobi && A->kind == semlab_op_s::kA && S->space == A->space &&
         !A->space->distributed() && A->space->bc == SEMLAB_BC_DIRICHLET;
}

bool fused_ras(semlab_op S, semlab_op A) {
  return S->kind == semlab_op_s::kSchwarz && S->sch->mode == SEMLAB_SCHWARZ_RAS && A->kind == semlab_op_s::kA &&
         S->space == A->space && !A->space->distributed() && A->space->bc == SEMLAB_BC_DIRICHLET;
}

bool dist_ras(semlab_op S, semlab_op A) {
  return S->kind == semlab_op_s::kSchwarz && S->sch->mode == SEMLAB_SCHWARZ_RAS && A->kind == semlab_op_s::kA &&
         S->space == A->space && A->space->distributed() && A->space->bc == SEMLAB_BC_DIRICHLET &&
         dist_ras_enabled();
}

}  // namespace

// ------------------------------------------------------------------------------ Chebyshev
void semlab_cheby_s::init(semlab_op S_, semlab_op A_, const semlab_cheby_params& p) {
  if (!S_ || !A_) invalid("ChebyshevSmoother: missing operator");
  if (p.order < 1) invalid("ChebyshevSmoother: order must be >= 1");
  if (!(p.lambda_min_mult > 0.0) || !(p.lambda_max_mult > p.lambda_min_mult))
    invalid("ChebyshevSmoother: need 0 < lambda_min_mult < lambda_max_mult");
  if (!(p.lambda_max_est > 0.0)) invalid("ChebyshevSmoother: lambda_max_est not set");
  if (S_->n != A_->n) invalid("ChebyshevSmoother: operator sizes differ");
  S = S_;
  A = A_;
  ctx = A_->ctx;
  params = p;
  const double lmin = p.lambda_min_mult * p.lambda_max_est;
  const double lmax = p.lambda_max_mult * p.lambda_max_est;
  theta = 0.5 * (lmax + lmin);
  delta = 0.5 * (lmax - lmin);
  sigma = theta / delta;
  n = A_->n;
  r.alloc(size_t(n));
  t.alloc(size_t(n));
  sad.alloc(size_t(n));
  d.alloc(size_t(n));
  // the fused RAS path writes only owned (free) nodes: masked entries must stay exactly 0
  r.zero(ctx->stream);
  t.zero(ctx->stream);
  sad.zero(ctx->stream);
  d.zero(ctx->stream);
}

void semlab_cheby_s::smooth(const double* b, double* x, bool x_is_zero) {
  cudaStream_t s = st(ctx);
  if (fused_jacobi(S, A)) {
    semlab_space sp = A->space;
    const double* inv = sp->jacobi_inv();
    if (x_is_zero) {
      ctx->count(launch_cheb_jac_zero_init(b, inv, r.p, d.p, theta, n, s));
    } else {
      EpiArgs a;
      a.r = r.p;
      a.d = d.p;
      a.b = b;
      a.inv = inv;
      a.c1 = theta;
      sp->ax(x, Epi::ChebJacInit, a, A->geom32);
    }
    double rho = 1.0 / sigma;
    for (int k = 1; k <= params.order; ++k) {
      const double rho_next = 1.0 / (2.0 * sigma - rho);
      EpiArgs a;
      a.x = x;
      a.r = r.p;
      a.d = d.p;
      a.inv = inv;
      a.c1 = rho_next * rho;
      a.c2 = 2.0 * rho_next / delta;
      sp->ax(d.p, Epi::ChebJacStep, a, A->geom32);
      rho = rho_next;
    }
    ctx->count(launch_axpby(x, 1.0, d.p, 1.0, n, s));
    return;
  }
  if (fused_ras(S, A)) {
    // S = RAS: t = A d in the fused Ax kernel, then the RAS owner write carries the whole
    // Chebyshev update (x += d; r -= S t; d = c1 d + c2 r).
    semlab_space sp = A->space;
    semlab_schwarz_s* sch = S->sch;
    RasEpi e;
    e.r = r.p;
    e.d = d.p;
    e.c1 = theta;
    e.c2 = 1.0 / theta;  // the init writes d = r * (1 / theta)
    if (x_is_zero) {
      sch->ras(b, 1, e);  // r = S (b - A 0) = S b
    } else {
      EpiArgs a;
      a.w = t.p;
      a.b = b;
      sp->ax(x, Epi::Residual, a, A->geom32);
      sch->ras(t.p, 1, e);
    }
    double rho = 1.0 / sigma;
    for (int k = 1; k <= params.order; ++k) {
      const double rho_next = 1.0 / (2.0 * sigma - rho);
      EpiArgs a;
      a.w = t.p;
      sp->ax(d.p, Epi::Write, a, A->geom32);
      RasEpi es;
      es.x = x;
      es.r = r.p;
      es.d = d.p;
      es.c1 = rho_next * rho;
      es.c2 = 2.0 * rho_next / delta;
      sch->ras(t.p, k == params.order ? 3 : 2, es);  // 3: the final x += d fused
      rho = rho_next;
    }
    if (params.order == 0) ctx->count(launch_axpby(x, 1.0, d.p, 1.0, n, s));
    return;
  }
  if (dist_ras(S, A)) {
    // RAS on z-slabs: the init stays generic; each Chebyshev step is t = A d (no interface sum
    // yet), ONE grouped exchange (interface partials + Schwarz ghost planes), the RAS owner write
    // carrying the Chebyshev update (mode 2, or 3 with the final x += d), and ONE grouped copy-up
    // of the lower rank's interface plane. Owned nodes get exactly the generic path's values.
    semlab_space sp = A->space;
    semlab_schwarz_s* sch = S->sch;
    if (x_is_zero) {
      ctx->count(launch_copy(t.p, b, n, s));
    } else {
      A->apply(x, t.p);
      ctx->count(launch_sub(t.p, b, t.p, n, s));
    }
    S->apply(t.p, r.p);
    ctx->count(launch_cheb_init(r.p, d.p, theta, n, s));
    double rho = 1.0 / sigma;
    for (int k = 1; k <= params.order; ++k) {
      const double rho_next = 1.0 / (2.0 * sigma - rho);
      EpiArgs a;
      a.w = t.p;
      sp->ax(d.p, Epi::Write, a, A->geom32);
      sp->interface_sum_halo(t.p);
      RasEpi es;
      es.x = x;
      es.r = r.p;
      es.d = d.p;
      es.c1 = rho_next * rho;
      es.c2 = 2.0 * rho_next / delta;
      const bool last = k == params.order;
      sch->ras(t.p, last ? 3 : 2, es);
      double* vs[3] = {x, r.p, d.p};
      sp->owner_copy_up_n(vs, last ? 1 : 3);
      rho = rho_next;
    }
    if (params.order == 0) ctx->count(launch_axpby(x, 1.0, d.p, 1.0, n, s));
    return;
  }
  // generic surrogate S
  if (x_is_zero) {
    ctx->count(launch_copy(t.p, b, n, s));
  } else {
    A->apply(x, t.p);
    ctx->count(launch_sub(t.p, b, t.p, n, s));
  }
  S->apply(t.p, r.p);
  ctx->count(launch_cheb_init(r.p, d.p, theta, n, s));
  double rho = 1.0 / sigma;
  for (int k = 1; k <= params.order; ++k) {
    A->apply(d.p, t.p);
    S->apply(t.p, sad.p);
    const double rho_next = 1.0 / (2.0 * sigma - rho);
    ctx->count(launch_cheb_step(x, r.p, d.p, sad.p, rho_next * rho, 2.0 * rho_next / delta, n, s));
    rho = rho_next;
  }
  ctx->count(launch_axpby(x, 1.0, d.p, 1.0, n, s));
}

namespace sb {

OwnRange own_range_of(semlab_op A) {
  if (A->space) return {A->space->n, A->space->own_off(), A->space->own_len()};
  return {A->n, 0, A->n};
}

namespace {

// Host copies of device reductions (after an allreduce over ranks).
void fetch(semlab_ctx c, const double* d, double* h, int K) {
  c->allreduce_device(const_cast<double*>(d), K);
  SB_CUDA(cudaMemcpyAsync(c->host_pinned, d, sizeof(double) * K, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  for (int k = 0; k < K; ++k) h[k] = c->host_pinned[k];
}

// One CGS2 Arnoldi step on w against V[:, :ncol] (krylov.cpp:67-76): h (incl. h2), ||w||.
// Scratch stride of cgs2's device results: h at [0, nb), h2 at [nb, 2nb), |w|^2 at 2nb.
int cgs2_stride(int ncol_max) { return std::max(kKrylovChunk, ncol_max); }

// One CGS2 step (krylov.cpp:67-72; chebyshev.cpp:36-41): h = V^T w; w -= V h; h2 = V^T w;
// w -= V h2; h += h2; hnext = |w|. Up to 32 columns the update and the next projection share one
// pass over V (fused kernels); wider bases (restart > 31) run the same steps in 32-column chunks.
void cgs2(semlab_ctx c, const OwnRange& o, const double* V, int64_t ldv, int ncol, double* w, double* d_h, int nb,
          std::vector<double>& h, double& hnext) {
  cudaStream_t s = c->stream;
  double* d_h2 = d_h + nb;
  double* d_nrm = d_h + 2 * nb;
  c->count(launch_gemv_t(V, ldv, ncol, w, o.off, o.len, d_h, c->dots(), s));
  c->allreduce_device(d_h, ncol);
  if (ncol <= kKrylovChunk) {
    c->count(launch_cgs_update_dot(V, ldv, ncol, w, d_h, o.n, o.off, o.len, d_h2, c->dots(), s));
    c->allreduce_device(d_h2, ncol);
    c->count(launch_cgs_update_norm(V, ldv, ncol, w, d_h2, o.n, o.off, o.len, d_nrm, c->dots(), s));
  } else {
    for (int c0 = 0; c0 < ncol; c0 += kKrylovChunk)  // w -= V h (the chunk dots are not used)
      c->count(launch_cgs_update_dot(V + c0 * ldv, ldv, std::min(kKrylovChunk, ncol - c0), w, d_h + c0, o.n, o.off,
                                     o.len, d_h2, c->dots(), s));
    c->count(launch_gemv_t(V, ldv, ncol, w, o.off, o.len, d_h2, c->dots(), s));
    c->allreduce_device(d_h2, ncol);
    for (int c0 = 0; c0 < ncol; c0 += kKrylovChunk)  // w -= V h2; the last chunk's norm is |w|^2
      c->count(launch_cgs_update_norm(V + c0 * ldv, ldv, std::min(kKrylovChunk, ncol - c0), w, d_h2 + c0, o.n,
                                      o.off, o.len, d_nrm, c->dots(), s));
  }
  c->allreduce_device(d_nrm, 1);
  const size_t cnt = size_t(2 * nb + 1);
  std::vector<double> big;
  double* hp = c->host_pinned;
  if (cnt > 128) {
    big.resize(cnt);
    hp = big.data();
  }
  SB_CUDA(cudaMemcpyAsync(hp, d_h, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s));
  c->sync();
  h.assign(size_t(ncol), 0.0);
  for (int k = 0; k < ncol; ++k) h[size_t(k)] = hp[k] + hp[nb + k];
  hnext = std::sqrt(hp[2 * nb]);
}

}  // namespace

semlab_lambda_estimate estimate_lambda_max(semlab_op S, semlab_op A, int64_t n, int rounds, uint64_t seed) {
  if (rounds < 1) invalid("estimate_lambda_max: rounds >= 1");
  if (!S || !A || S->n != n || A->n != n) invalid("estimate_lambda_max: operator sizes differ from n");
  semlab_ctx c = A->ctx;
  cudaStream_t s = c->stream;
  const OwnRange o = own_range_of(A);
  semlab_lambda_estimate est{0.0, 0, 0};
  // seeded U(-1,1) start vector, one draw per global lattice dof in index order
  std::vector<double> hv(static_cast<size_t>(n));
  int64_t offset = 0;
  if (A->space) offset = A->space->sl.zlo * A->space->sl.Nx * A->space->sl.Ny;
  uniform_pm1_range(seed, offset, n, hv.data());
  DevBuf<double> v(static_cast<size_t>(n)), t(static_cast<size_t>(n)), w(static_cast<size_t>(n)), V(size_t(n) * (rounds + 1)), dh(size_t(3 * cgs2_stride(rounds + 1)));
  v.upload(hv.data(), size_t(n), s);
  std::vector<double> H(size_t(rounds + 1) * rounds, 0.0);  // column-major (rounds+1) x rounds
  A->apply(v.p, t.p);
  S->apply(t.p, w.p);
  const double* wv[1] = {w.p};
  double nrm2 = 0.0;
  c->dots(1, wv, wv, o.off, o.len, &nrm2);
  const double nrm = std::sqrt(nrm2);
  if (!(nrm > 0.0)) {
    est.breakdown = 1;
    return est;
  }
  c->count(launch_div(V.p, w.p, nrm, n, s));
  int m = 0;
  std::vector<double> h;
  for (int j = 0; j < rounds; ++j) {
    A->apply(V.p + size_t(j) * n, t.p);
    S->apply(t.p, w.p);
    double hnext = 0.0;
    cgs2(c, o, V.p, n, j + 1, w.p, dh.p, cgs2_stride(rounds + 1), h, hnext);
    for (int i = 0; i <= j; ++i) H[size_t(i) + size_t(rounds + 1) * j] = h[size_t(i)];
    H[size_t(j + 1) + size_t(rounds + 1) * j] = hnext;
    m = j + 1;
    double hmax = 0.0;
    for (double e : h) hmax = std::max(hmax, std::abs(e));
    if (hnext <= 1e-12 * hmax) {
      est.breakdown = 1;
      break;
    }
    c->count(launch_div(V.p + size_t(j + 1) * n, w.p, hnext, n, s));
  }
  est.rounds_used = m;
  std::vector<double> Hm(size_t(m) * m);
  for (int jj = 0; jj < m; ++jj)
    for (int i = 0; i < m; ++i) Hm[size_t(i) + size_t(m) * jj] = H[size_t(i) + size_t(rounds + 1) * jj];
  est.value = max_abs_eig(m, Hm.data());
  c->sync();
  return est;
}

namespace {

// Columns of the Krylov workspace start on 256-byte boundaries.
int64_t padded(int64_t n) { return (n + 31) / 32 * 32; }

// The context's persistent workspace for the duration of one solve.
struct WsLease {
  semlab_ctx c;
  DevBuf<double> own;
  double* p = nullptr;
  bool leased = false;
  WsLease(semlab_ctx c_, size_t count) : c(c_) {
    if (!c->krylov_ws_busy) {
      if (c->krylov_ws.n < count) c->krylov_ws.alloc(count);
      c->krylov_ws_busy = leased = true;
      p = c->krylov_ws.p;
    } else {
      own.alloc(count);
      p = own.p;
    }
  }
  ~WsLease() {
    if (leased) c->krylov_ws_busy = false;
  }
  WsLease(const WsLease&) = delete;
  WsLease& operator=(const WsLease&) = delete;
};

}  // namespace

KrylovResult gmres_solve(semlab_op A, semlab_op M, const double* b, double* x, const semlab_gmres_config& cfg) {
  if (cfg.restart < 1) invalid("gmres: restart must be >= 1");
  if (!(cfg.tol > 0.0)) invalid("gmres: tol must be positive");
  if (!A) invalid("gmres: missing operator");
  semlab_ctx c = A->ctx;
  cudaStream_t s = c->stream;
  const int64_t n = A->n;
  const int m = cfg.restart;
  const OwnRange o = own_range_of(A);
  KrylovResult res;
  const int64_t ld = padded(n);
  // Preconditioned directions z_j = M v_j are kept (Z, m columns) and the update is x += Z y. For
  // a linear M this is the reference's x += M (V y) (krylov.cpp:108-114) up to rounding, one M
  // application cheaper per restart cycle; for the FP32 smoother's V-cycle (linear only to
  // ~1e-7) it keeps the least-squares residual estimate consistent with the true residual, so
  // the FP32-smoothed solve needs the FP64 solve's iteration count instead of an extra restart.
  const int nb = cgs2_stride(m + 1);
  // Flexible form (Z kept) when the device has room for the m extra columns; otherwise (e.g. one
  // B200 at E = 96^3, where Z alone is 49 GB) the reference's x += M (V y), one extra M per cycle.
  bool flexible = M != nullptr && gmres_flexible_allowed();
  if (flexible) {
    const size_t need = (size_t(ld) * (2 * m + 3) + size_t(3 * nb)) * sizeof(double);
    const size_t have = c->krylov_ws_busy ? 0 : c->krylov_ws.n * sizeof(double);
    if (need > have) {
      size_t free_b = 0, total_b = 0;
      SB_CUDA(cudaMemGetInfo(&free_b, &total_b));
      flexible = need - have + (size_t(2) << 30) <= free_b;
    }
  }
  const int zc = flexible ? m : 0;
  WsLease ws(c, size_t(ld) * (m + 3 + zc) + size_t(3 * nb));
  struct {
    double* p;
  } r{ws.p}, w{ws.p + ld}, V{ws.p + 2 * ld}, Z{ws.p + size_t(ld) * (m + 3)},
      dh{ws.p + size_t(ld) * (m + 3 + zc)};
  // z_j: stored column of Z (flexible), else a single scratch column (the reference form), or v_j
  // itself without a preconditioner
  auto dir = [&](int j) {
    return flexible ? Z.p + size_t(j) * ld : (M ? w.p : V.p + size_t(j) * ld);
  };
  auto norm = [&](const double* v) {
    const double* av[1] = {v};
    double r2 = 0.0;
    c->dots(1, av, av, o.off, o.len, &r2);
    return std::sqrt(r2);
  };
  A->apply(x, r.p);
  c->count(launch_sub(r.p, b, r.p, n, s));
  res.initial_residual = norm(r.p);
  const double target = cfg.use_abs_tol ? cfg.abs_tol : cfg.tol * res.initial_residual;
  auto finish = [&](double rr) {
    res.abs_residual = rr;
    res.rel_residual = res.initial_residual > 0.0 ? rr / res.initial_residual : 0.0;
  };
  double beta = res.initial_residual;
  if (beta <= target) {
    res.converged = true;
    finish(beta);
    return res;
  }
  std::vector<double> H(size_t(m + 1) * m, 0.0), g(static_cast<size_t>(m + 1)), cs(static_cast<size_t>(m)), sn(static_cast<size_t>(m)), h;
  auto Hc = [&](int i, int j) -> double& { return H[size_t(i) + size_t(m + 1) * j]; };
  while (res.iterations < cfg.max_iters) {
    c->count(launch_div(V.p, r.p, beta, n, s));
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int j = 0;
    bool lucky = false;
    for (; j < m && res.iterations < cfg.max_iters; ++j) {
      if (flexible) {
        M->apply(V.p + size_t(j) * ld, dir(j));
        A->apply(dir(j), w.p);
      } else if (M) {  // z_j is not kept: M v_j in r's column (r is free until the cycle ends)
        M->apply(V.p + size_t(j) * ld, r.p);
        A->apply(r.p, w.p);
      } else {
        A->apply(dir(j), w.p);
      }
      double hnext = 0.0;
      cgs2(c, o, V.p, ld, j + 1, w.p, dh.p, nb, h, hnext);
      for (int i = 0; i <= j; ++i) Hc(i, j) = h[size_t(i)];
      Hc(j + 1, j) = hnext;
      for (int i = 0; i < j; ++i) {  // Givens (krylov.cpp:77-89)
        const double tt = cs[i] * Hc(i, j) + sn[i] * Hc(i + 1, j);
        Hc(i + 1, j) = -sn[i] * Hc(i, j) + cs[i] * Hc(i + 1, j);
        Hc(i, j) = tt;
      }
      const double denom = std::hypot(Hc(j, j), Hc(j + 1, j));
      cs[j] = denom > 0.0 ? Hc(j, j) / denom : 1.0;
      sn[j] = denom > 0.0 ? Hc(j + 1, j) / denom : 0.0;
      Hc(j, j) = denom;
      Hc(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] *= cs[j];
      ++res.iterations;
      const double res_est = std::abs(g[j + 1]);
      res.history.push_back(res_est);
      if (hnext <= 1e-14 * beta) {
        res.breakdown = true;
        lucky = true;
        ++j;
        break;
      }
      c->count(launch_div(V.p + size_t(j + 1) * ld, w.p, hnext, n, s));
      if (res_est <= target) {
        ++j;
        break;
      }
    }
    if (j > 0) {  // x += Z y  (= M (V y) for a linear M, krylov.cpp:108-114)
      std::vector<double> y(static_cast<size_t>(j));
      for (int i = j - 1; i >= 0; --i) {
        double acc = g[size_t(i)];
        for (int k = i + 1; k < j; ++k) acc -= Hc(i, k) * y[size_t(k)];
        y[size_t(i)] = acc / Hc(i, i);
      }
      if (flexible || !M) {
        c->count(launch_gemv_n(dir(0), ld, j, y.data(), x, n, s, true));
      } else {  // x += M (V y), krylov.cpp:108-114
        c->count(launch_gemv_n(V.p, ld, j, y.data(), w.p, n, s));
        M->apply(w.p, r.p);
        c->count(launch_axpby(x, 1.0, r.p, 1.0, n, s));
      }
    }
    A->apply(x, r.p);
    c->count(launch_sub(r.p, b, r.p, n, s));
    beta = norm(r.p);
    if (beta <= target || lucky) {
      res.converged = true;
      finish(beta);
      return res;
    }
  }
  finish(beta);
  res.converged = beta <= target;
  return res;
}

KrylovResult pcg_solve(semlab_op A, semlab_op M, const double* b, double* x, const semlab_gmres_config& cfg) {
  if (!(cfg.tol > 0.0)) invalid("pcg: tol must be positive");
  if (!A) invalid("pcg: missing operator");
  semlab_ctx c = A->ctx;
  cudaStream_t s = c->stream;
  const int64_t n = A->n;
  const OwnRange o = own_range_of(A);
  KrylovResult res;
  const int64_t ld = padded(n);
  WsLease ws(c, size_t(ld) * 4);
  struct {
    double* p;
  } r{ws.p}, w{ws.p + ld}, z{ws.p + 2 * ld}, p{ws.p + 3 * ld};
  auto dot = [&](const double* a, const double* bb) {
    const double* av[1] = {a};
    const double* bv[1] = {bb};
    double v = 0.0;
    c->dots(1, av, bv, o.off, o.len, &v);
    return v;
  };
  A->apply(x, w.p);
  c->count(launch_sub(r.p, b, w.p, n, s));
  res.initial_residual = std::sqrt(dot(r.p, r.p));
  const double target = cfg.use_abs_tol ? cfg.abs_tol : cfg.tol * res.initial_residual;
  double rn = res.initial_residual;
  if (rn <= target || rn == 0.0) {
    res.converged = true;
    res.abs_residual = rn;
    res.rel_residual = 0.0;
    return res;
  }
  if (M) M->apply(r.p, z.p); else c->count(launch_copy(z.p, r.p, n, s));
  c->count(launch_copy(p.p, z.p, n, s));
  double rz = dot(r.p, z.p);
  while (res.iterations < cfg.max_iters) {
    A->apply(p.p, w.p);
    const double alpha = rz / dot(p.p, w.p);
    c->count(launch_axpby(x, alpha, p.p, 1.0, n, s));
    c->count(launch_axpby(r.p, -alpha, w.p, 1.0, n, s));
    ++res.iterations;
    rn = std::sqrt(dot(r.p, r.p));
    res.history.push_back(rn);
    if (rn <= target) break;
    if (M) M->apply(r.p, z.p); else c->count(launch_copy(z.p, r.p, n, s));
    const double rz_new = dot(r.p, z.p);
    c->count(launch_axpby(p.p, 1.0, z.p, rz_new / rz, n, s));
    rz = rz_new;
  }
  A->apply(x, w.p);
  c->count(launch_sub(w.p, b, w.p, n, s));
  res.abs_residual = std::sqrt(dot(w.p, w.p));
  res.rel_residual = res.initial_residual > 0.0 ? res.abs_residual / res.initial_residual : 0.0;
  res.converged = rn <= target;
  return res;
}

}  // namespace sb

// ------------------------------------------------------------------------------ ProjectionBasis
// krylov.cpp:131-152. The basis is column-major with 256-byte aligned columns, oldest first,
// plus one spare column that receives a new vector before the oldest is evicted.
void semlab_proj_s::init(semlab_ctx c, int64_t n_, int cap) {
  if (!c) invalid("ProjectionBasis: missing context");
  if (n_ < 1) invalid("ProjectionBasis: n must be >= 1");
  if (cap < 1 || cap > 24) invalid("ProjectionBasis: capacity must be in [1, 24] on the device path");
  ctx = c;
  n = n_;
  own = {n_, 0, n_};
  capacity = cap;
  ld = padded(n_);
  V.alloc(size_t(ld) * (cap + 1));
  w.alloc(size_t(n_));
  aw.alloc(size_t(n_));
  dh.alloc(96);
}

void semlab_proj_s::initial_guess(const double* b, double* u) {
  cudaStream_t s = ctx->stream;
  const OwnRange& o = own;
  if (size == 0) {
    ctx->count(launch_fill(u, n, 0.0, s));
    return;
  }
  std::vector<double> h(static_cast<size_t>(size));
  ctx->count(launch_gemv_t(V.p, ld, size, b, o.off, o.len, dh.p, ctx->dots(), s));
  fetch(ctx, dh.p, h.data(), size);
  ctx->count(launch_gemv_n(V.p, ld, size, h.data(), u, n, s));
}

void semlab_proj_s::insert(const double* x, semlab_op A) {
  if (!A) invalid("ProjectionBasis: missing operator");
  if (A->n != n) invalid("ProjectionBasis: operator size differs from the basis length");
  cudaStream_t s = ctx->stream;
  const OwnRange o = own_range_of(A);
  own = o;
  SB_CUDA(cudaMemcpyAsync(w.p, x, sizeof(double) * size_t(n), cudaMemcpyDeviceToDevice, s));
  A->apply(w.p, aw.p);
  const double* a[1] = {w.p};
  const double* b[1] = {aw.p};
  double wa = 0.0;
  ctx->dots(1, a, b, o.off, o.len, &wa);
  const double norm0 = std::sqrt(std::max(0.0, wa));
  if (size > 0) {
    for (int pass = 0; pass < 2; ++pass) {  // w -= sum_i (x_i . Aw) x_i with Aw fixed per pass
      ctx->count(launch_gemv_t(V.p, ld, size, aw.p, o.off, o.len, dh.p, ctx->dots(), s));
      ctx->allreduce_device(dh.p, size);
      ctx->count(launch_cgs_update_norm(V.p, ld, size, w.p, dh.p, n, o.off, o.len, dh.p + 64, ctx->dots(), s));
      A->apply(w.p, aw.p);
    }
  }
  ctx->dots(1, a, b, o.off, o.len, &wa);
  const double norm = std::sqrt(std::max(0.0, wa));
  if (!(norm > 1e-12 * std::max(norm0, 1e-300))) return;  // numerically dependent
  ctx->count(launch_div(V.p + size_t(ld) * size, w.p, norm, n, s));
  if (++size > capacity) {  // evict the oldest: shift columns down (non-overlapping copies)
    for (int k = 0; k < capacity; ++k)
      SB_CUDA(cudaMemcpyAsync(V.p + size_t(ld) * k, V.p + size_t(ld) * (k + 1), sizeof(double) * size_t(n),
                              cudaMemcpyDeviceToDevice, s));
    size = capacity;
  }
}

int semlab_proj_create(semlab_ctx ctx, int64_t n, int capacity, semlab_proj* out) {
  return guard([&] {
    need(out, "ProjectionBasis: out");
    auto p = std::make_unique<semlab_proj_s>();
    p->init(ctx, n, capacity);
    *out = p.release();
  });
}

int semlab_proj_destroy(semlab_proj p) {
  return guard([&] {
    if (p) cudaStreamSynchronize(p->ctx->stream);
    delete p;
  });
}

int semlab_proj_initial_guess(semlab_proj p, const double* b, double* u) {
  return guard([&] {
    need(p, "ProjectionBasis: basis");
    p->initial_guess(b, u);
  });
}

int semlab_proj_insert(semlab_proj p, const double* x, semlab_op A) {
  return guard([&] {
    need(p, "ProjectionBasis: basis");
    p->insert(x, A);
  });
}

int semlab_proj_size(semlab_proj p, int* out) {
  return guard([&] {
    need(p, "ProjectionBasis: basis");
    need(out, "ProjectionBasis: out");
    *out = p->size;
  });
}

int semlab_proj_clear(semlab_proj p) {
  return guard([&] {
    need(p, "ProjectionBasis: basis");
    p->size = 0;
  });
}

int semlab_proj_vector(semlab_proj p, int i, double* out) {
  return guard([&] {
    need(p, "ProjectionBasis: basis");
    if (i < 0 || i >= p->size) invalid("ProjectionBasis: vector index out of range");
    SB_CUDA(cudaMemcpyAsync(out, p->V.p + size_t(p->ld) * i, sizeof(double) * size_t(p->n),
                            cudaMemcpyDeviceToDevice, p->ctx->stream));
  });
}
