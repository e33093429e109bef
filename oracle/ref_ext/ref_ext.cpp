// ORACLE TEST INFRASTRUCTURE — the reference semlab library (its own translation units, compiled
// against oracle/eigen_shim) extended with the pieces it lists but does not ship (pmg.cpp,
// precond.cpp, bench.cpp; core/CMakeLists.txt:12-15) and a CG it never had. These restatements
// follow SPEC.md:308-373 (pMG), :292 (Jacobi), :566-574 (RHS) — the same definitions the numpy
// oracle (oracle/semlab_np.py) and the B200 product use — and are built only into
// oracle/_ref/{libsemlab_ref.so, semlab_ref_bench}. Never linked into the product.
#include "ref_ext.hpp"

#include <chrono>
#include <cmath>
#include <cstring>
#include <random>

namespace semlab_ref {

using namespace semlab;

FieldVector jacobi_inverse_diag(const SemSpace& s) {
  FieldVector d = s.stiffness_diag();
  FieldVector inv(d.size());
  for (Index i = 0; i < d.size(); ++i) inv[i] = d[i] != 0.0 ? 1.0 / d[i] : 0.0;
  return inv;
}

FieldVector build_rhs(const SemSpace& s, std::uint64_t seed) {
  const auto& X = s.lattice_coords();
  const Index n = s.n();
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  FieldVector b(n);
  const double pi = M_PI;
  for (Index g = 0; g < n; ++g) {
    const double x = X[size_t(3 * g)], y = X[size_t(3 * g + 1)], z = X[size_t(3 * g + 2)];
    const double smooth = 3.0 * pi * pi * std::sin(pi * (x + 0.5)) * std::sin(pi * (y + 0.5)) * std::sin(pi * (z + 0.5));
    const double bubble = 64.0 * (0.25 - x * x) * (0.25 - y * y) * (0.25 - z * z);
    b[g] = s.mass_diag()[g] * (smooth + dist(rng) * bubble);
  }
  s.mask_inplace(b);
  return b;
}

// ---------------------------------------------------------------- transfers
Transfer::Transfer(const SemSpace& fine, const SemSpace& coarse) : f(&fine), c(&coarse) {
  J = lagrange_interpolation_matrix(coarse.basis().nodes, fine.basis().nodes);  // (qf+1) x (qc+1)
}

static FieldVector tensor3(const Eigen::MatrixXd& M, const FieldVector& loc, Index E, int nin, int nout) {
  // out[e](i,j,k) = sum_abc M(i,a) M(j,b) M(k,c) in[e](a,b,c); x fastest in both
  FieldVector out(E * nout * nout * nout);
  std::vector<double> t1(size_t(nout) * nin * nin), t2(size_t(nout) * nout * nin);
  for (Index e = 0; e < E; ++e) {
    const double* in = loc.data() + e * nin * nin * nin;
    double* o = out.data() + e * nout * nout * nout;
    for (int c = 0; c < nin; ++c)
      for (int b = 0; b < nin; ++b)
        for (int i = 0; i < nout; ++i) {
          double s = 0.0;
          for (int a = 0; a < nin; ++a) s += M(i, a) * in[a + nin * (b + nin * c)];
          t1[size_t(i + nout * (b + nin * c))] = s;
        }
    for (int c = 0; c < nin; ++c)
      for (int j = 0; j < nout; ++j)
        for (int i = 0; i < nout; ++i) {
          double s = 0.0;
          for (int b = 0; b < nin; ++b) s += M(j, b) * t1[size_t(i + nout * (b + nin * c))];
          t2[size_t(i + nout * (j + nout * c))] = s;
        }
    for (int k = 0; k < nout; ++k)
      for (int j = 0; j < nout; ++j)
        for (int i = 0; i < nout; ++i) {
          double s = 0.0;
          for (int cc = 0; cc < nin; ++cc) s += M(k, cc) * t2[size_t(i + nout * (j + nout * cc))];
          o[i + nout * (j + nout * k)] = s;
        }
  }
  return out;
}

FieldVector Transfer::prolong(const FieldVector& uc) const {
  FieldVector u = c->masked(uc);
  const Index E = c->mesh().n_elements();
  FieldVector loc = tensor3(J, c->scatter(u), E, c->order() + 1, f->order() + 1);
  FieldVector uf = f->gather(loc);
  for (Index g = 0; g < uf.size(); ++g) uf[g] /= double(f->multiplicity()[g]);
  f->mask_inplace(uf);
  return uf;
}

FieldVector Transfer::restrict_(const FieldVector& rf) const {
  FieldVector r = f->masked(rf);
  for (Index g = 0; g < r.size(); ++g) r[g] /= double(f->multiplicity()[g]);
  const Index E = f->mesh().n_elements();
  Eigen::MatrixXd JT(J.cols(), J.rows());
  for (Index i = 0; i < J.rows(); ++i)
    for (Index j = 0; j < J.cols(); ++j) JT(j, i) = J(i, j);
  FieldVector loc = tensor3(JT, f->scatter(r), E, f->order() + 1, c->order() + 1);
  FieldVector rc = c->gather(loc);
  c->mask_inplace(rc);
  return rc;
}

// ---------------------------------------------------------------- coarse
CoarseSolve::CoarseSolve(const SemSpace& s, const std::string& mode) : sp(&s), mode_(mode) {
  const int nl = s.nodes_per_element();
  const Index E = s.mesh().n_elements();
  std::vector<Index> fidx(size_t(s.n()), -1);
  for (Index g = 0; g < s.n(); ++g)
    if (!s.is_masked(g)) {
      fidx[size_t(g)] = Index(free_.size());
      free_.push_back(g);
    }
  std::vector<Eigen::Triplet<double>> trip;
  std::vector<double> in(size_t(nl)), out(size_t(nl));
  const int nd = s.order() + 1;
  for (Index e = 0; e < E; ++e) {
    std::vector<Index> g(size_t(nl));
    for (int k = 0, l = 0; k < nd; ++k)
      for (int j = 0; j < nd; ++j)
        for (int i = 0; i < nd; ++i, ++l) g[size_t(l)] = s.global_index(int(e), i, j, k);
    for (int col = 0; col < nl; ++col) {
      std::fill(in.begin(), in.end(), 0.0);
      in[size_t(col)] = 1.0;
      s.apply_local_stiffness(int(e), in.data(), out.data());
      if (fidx[size_t(g[size_t(col)])] < 0) continue;
      for (int row = 0; row < nl; ++row)
        if (fidx[size_t(g[size_t(row)])] >= 0)
          trip.emplace_back(fidx[size_t(g[size_t(row)])], fidx[size_t(g[size_t(col)])], out[size_t(row)]);
    }
  }
  const Index nf = Index(free_.size());
  A_.resize(nf, nf);
  A_.setFromTriplets(trip.begin(), trip.end());
  if (mode_ == "direct") {
    Eigen::MatrixXd Ad(A_);
    if (s.bc() == BcMode::Neumann) {  // constants span the nullspace: A + 1 1^T / n is SPD
      const double c = 1.0 / double(nf);
      for (Index j = 0; j < nf; ++j)
        for (Index i = 0; i < nf; ++i) Ad(i, j) += c;
    }
    ldlt_.compute(Ad);
    if (ldlt_.info() != Eigen::Success) throw std::runtime_error("coarse: factorization failed");
  } else {
    amg_ = std::make_unique<AmgHierarchy>(AmgHierarchy::build(A_));
  }
}

FieldVector CoarseSolve::solve(const FieldVector& r) const {
  const Index nf = Index(free_.size());
  FieldVector rf(nf), zf;
  for (Index t = 0; t < nf; ++t) rf[t] = r[free_[size_t(t)]];
  const bool neu = sp->bc() == BcMode::Neumann;
  if (neu) rf.array() -= rf.mean();  // project onto the zero-mean range, solve, project back
  if (mode_ == "direct")
    zf = ldlt_.solve(rf);
  else
    amg_->vcycle(rf, zf);
  if (neu) zf.array() -= zf.mean();
  FieldVector z = FieldVector::Zero(sp->n());
  for (Index t = 0; t < nf; ++t) z[free_[size_t(t)]] = zf[t];
  return z;
}

// ---------------------------------------------------------------- pMG (Alg. 1)
Pmg::Pmg(const HexMesh& mesh, const std::vector<int>& orders, const std::string& smoother_kind, int eta, double lmin,
         double lmax, const std::string& coarse, BcMode bc, bool additive) {
  plain_ = smoother_kind == "ras_plain" || smoother_kind == "asm_plain";
  additive_ = additive;
  const std::string smoother = plain_ ? smoother_kind.substr(0, 3) : smoother_kind;
  for (int q : orders) spaces.push_back(std::make_unique<SemSpace>(mesh, q, bc));
  for (size_t l = 0; l + 1 < orders.size(); ++l) {
    const SemSpace& s = *spaces[l];
    Level L;
    L.A = [&s](const FieldVector& in, FieldVector& out) { out = s.apply_A(in); };
    if (smoother == "jacobi") {
      auto inv = std::make_shared<FieldVector>(jacobi_inverse_diag(s));
      L.S = [inv](const FieldVector& in, FieldVector& out) { out = inv->cwiseProduct(in); };
    } else {
      L.sch = std::make_unique<SchwarzSmoother>(s, smoother == "ras" ? SchwarzMode::Ras : SchwarzMode::Asm);
      L.S = L.sch->as_linop();
    }
    if (!plain_) {
      L.lam = estimate_lambda_max(L.S, L.A, s.n(), 10, 0).value;
      L.cheb = std::make_unique<ChebyshevSmoother>(L.S, L.A, ChebyParams{eta, lmin, lmax, L.lam});
    }
    levels.push_back(std::move(L));
    transfers.push_back(std::make_unique<Transfer>(s, *spaces[l + 1]));
  }
  coarse_ = std::make_unique<CoarseSolve>(*spaces.back(), coarse);
}

// one smoothing step: Chebyshev(eta) from x (x = 0 when null), or the plain smoother:
// x = S b from zero, else x + S (b - A x)
FieldVector Pmg::smooth(size_t l, const FieldVector& b, const FieldVector* x0) const {
  const Level& L = levels[l];
  FieldVector x = x0 ? *x0 : FieldVector::Zero(b.size());
  if (!plain_) {
    L.cheb->smooth(b, x);
    return x;
  }
  FieldVector t(b.size()), z(b.size());
  if (!x0) {
    L.S(b, z);
    return z;
  }
  L.A(x, t);
  t = b - t;
  L.S(t, z);
  x += z;
  return x;
}

FieldVector Pmg::cycle(size_t l, const FieldVector& b) const {
  if (l == levels.size()) return coarse_->solve(b);
  const Level& L = levels[l];
  FieldVector x = smooth(l, b, nullptr);
  FieldVector r(b.size());
  L.A(x, r);
  r = b - r;
  FieldVector ec = cycle(l + 1, transfers[l]->restrict_(r));
  x += transfers[l]->prolong(ec);
  return smooth(l, b, &x);
}

// additive V-cycle: smooth every level's restricted right-hand side from zero,
// solve the coarsest, sum the prolongated corrections; no residual re-evaluation, no post-smoothing
FieldVector Pmg::cycle_additive(size_t l, const FieldVector& b) const {
  if (l == levels.size()) return coarse_->solve(b);
  FieldVector x = smooth(l, b, nullptr);
  x += transfers[l]->prolong(cycle_additive(l + 1, transfers[l]->restrict_(b)));
  return x;
}

LinOp Pmg::as_linop() const {
  return [this](const FieldVector& in, FieldVector& out) { out = vcycle(in); };
}

// ---------------------------------------------------------------- PCG (textbook; not in the reference)
GmresStats pcg_solve(const LinOp& A, const LinOp& M, const FieldVector& b, FieldVector& x, double tol, int max_iters) {
  GmresStats st;
  const Index n = b.size();
  FieldVector r(n), z(n), p(n), w(n);
  A(x, w);
  r = b - w;
  st.initial_residual = r.norm();
  const double target = tol * st.initial_residual;
  double rn = st.initial_residual;
  if (rn <= target || rn == 0.0) {
    st.converged = true;
    return st;
  }
  if (M) M(r, z); else z = r;
  p = z;
  double rz = r.dot(z);
  while (st.iterations < max_iters) {
    A(p, w);
    const double alpha = rz / p.dot(w);
    x += alpha * p;
    r -= alpha * w;
    ++st.iterations;
    rn = r.norm();
    st.history.push_back(rn);
    if (rn <= target) break;
    if (M) M(r, z); else z = r;
    const double rz_new = r.dot(z);
    p = z + (rz_new / rz) * p;
    rz = rz_new;
  }
  A(x, w);
  w = b - w;
  st.abs_residual = w.norm();
  st.rel_residual = st.abs_residual / st.initial_residual;
  st.converged = rn <= target;
  return st;
}

}  // namespace semlab_ref
