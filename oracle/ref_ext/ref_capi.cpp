// ORACLE TEST INFRASTRUCTURE — extern "C" entry points over the reference semlab library (own
// TUs + Eigen shim) and its restated extension, used by tests/golden/make_golden.py to produce
// golden vectors and by tests/test_oracle_pin.py to pin the numpy oracle. Output: oracle/_ref/.
#include <cstring>
#include <random>

#include "ref_ext.hpp"
#include "semlab/semfem.hpp"

using namespace semlab;
using namespace semlab_ref;

namespace {
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
HexMesh mesh_of(double eps, int E, int p) { return generate_kershaw(KershawParams{eps, E}, p); }
std::vector<int> orders_of(const int* o, int n) { return std::vector<int>(o, o + n); }
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_gll(int p, double* nodes, double* weights, double* diff) {
  return guard([&] {
    const Gll1D& g = gll(p);
    std::memcpy(nodes, g.nodes.data(), sizeof(double) * size_t(p + 1));
    std::memcpy(weights, g.weights.data(), sizeof(double) * size_t(p + 1));
    std::memcpy(diff, g.diff.data(), sizeof(double) * size_t((p + 1) * (p + 1)));
  });
}

int ref_uniform(uint64_t seed, int64_t n, double* out) {
  return guard([&] {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
  });
}

int ref_sizes(double eps, int E, int p, int64_t* n, int64_t* nlocal) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p);
    *n = s.n();
    *nlocal = s.n_local_total();
  });
}

int ref_lattice(double eps, int E, int p, double* out) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    auto c = m.lattice_coords(p);
    std::memcpy(out, c.data(), c.size() * sizeof(double));
  });
}

int ref_geom(double eps, int E, int p, double* out) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p);
    const int nl = s.nodes_per_element();
    for (int e = 0; e < m.n_elements(); ++e)
      for (int node = 0; node < nl; ++node) std::memcpy(out + (size_t(e) * nl + node) * 6, s.metric_at(e, node), 48);
  });
}

int ref_apply_A(double eps, int E, int p, const double* u, double* out) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p);
    FieldVector v = Eigen::Map<const Eigen::MatrixXd>(u, s.n(), 1);
    FieldVector w = s.apply_A(v);
    std::memcpy(out, w.data(), sizeof(double) * size_t(s.n()));
  });
}

int ref_diag_mass(double eps, int E, int p, double* diag, double* mass) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p);
    FieldVector d = s.stiffness_diag();
    std::memcpy(diag, d.data(), sizeof(double) * size_t(s.n()));
    std::memcpy(mass, s.mass_diag().data(), sizeof(double) * size_t(s.n()));
  });
}

int ref_gather(double eps, int E, int p, const double* loc, double* out) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p);
    FieldVector l = Eigen::Map<const Eigen::MatrixXd>(loc, s.n_local_total(), 1);
    FieldVector g = s.gather(l);
    std::memcpy(out, g.data(), sizeof(double) * size_t(s.n()));
  });
}

int ref_schwarz_apply(double eps, int E, int p, int mode, const double* r, double* z, double* lengths,
                      double* lambda0) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p);
    SchwarzSmoother sch(s, mode == 1 ? SchwarzMode::Ras : SchwarzMode::Asm);
    FieldVector rv = Eigen::Map<const Eigen::MatrixXd>(r, s.n(), 1);
    FieldVector zv = sch.apply(rv);
    std::memcpy(z, zv.data(), sizeof(double) * size_t(s.n()));
    for (int e = 0; e < m.n_elements(); ++e) {
      const auto L = sch.box_lengths(e);
      for (int d = 0; d < 3; ++d) lengths[e * 3 + d] = L[size_t(d)];
    }
    const auto& d0 = sch.direction(0, 0);
    for (Index i = 0; i < d0.lambda.size(); ++i) lambda0[i] = d0.lambda[i];
  });
}

// Neumann mode (sem_space.hpp:12, 28): apply_A with mean removal (sem_space.cpp:207), the
// unmasked diagonal (sem_space.cpp:211-236) and RAS/ASM with Neumann faces (schwarz.cpp:151-160).
int ref_neumann(double eps, int E, int p, const double* u, double* Au, double* diag, const double* r,
                double* ras, double* asm_) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p, BcMode::Neumann);
    const size_t n = size_t(s.n());
    FieldVector uv = Eigen::Map<const Eigen::MatrixXd>(u, s.n(), 1);
    FieldVector w = s.apply_A(uv);
    std::memcpy(Au, w.data(), sizeof(double) * n);
    FieldVector d = s.stiffness_diag();
    std::memcpy(diag, d.data(), sizeof(double) * n);
    FieldVector rv = Eigen::Map<const Eigen::MatrixXd>(r, s.n(), 1);
    SchwarzSmoother sr(s, SchwarzMode::Ras), sa(s, SchwarzMode::Asm);
    FieldVector zr = sr.apply(rv), za = sa.apply(rv);
    std::memcpy(ras, zr.data(), sizeof(double) * n);
    std::memcpy(asm_, za.data(), sizeof(double) * n);
  });
}

// ProjectionBasis (krylov.cpp:131-152): insert the K columns of X (n x K, column-major) one by
// one with A = apply_A of the space, then return the basis (oldest first) and the projected
// guess for b.
int ref_projection(double eps, int E, int p, int capacity, int K, const double* X, const double* b,
                   int* size, double* basis, double* guess) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p);
    LinOp A = [&s](const FieldVector& in, FieldVector& out) { out = s.apply_A(in); };
    ProjectionBasis pb(capacity);
    const size_t n = size_t(s.n());
    for (int k = 0; k < K; ++k) {
      FieldVector x = Eigen::Map<const Eigen::MatrixXd>(X + n * size_t(k), s.n(), 1);
      pb.insert(x, A);
    }
    *size = pb.size();
    for (int i = 0; i < pb.size(); ++i) std::memcpy(basis + n * size_t(i), pb.vectors()[size_t(i)].data(), 8 * n);
    FieldVector bv = Eigen::Map<const Eigen::MatrixXd>(b, s.n(), 1);
    FieldVector u = pb.initial_guess(bv);
    std::memcpy(guess, u.data(), 8 * n);
  });
}

int ref_lambda(double eps, int E, int p, int smoother, double* value, int* rounds) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p);
    LinOp A = [&s](const FieldVector& in, FieldVector& out) { out = s.apply_A(in); };
    LinOp S;
    std::unique_ptr<SchwarzSmoother> sch;
    FieldVector inv;
    if (smoother == 0) {
      inv = jacobi_inverse_diag(s);
      S = [&inv](const FieldVector& in, FieldVector& out) { out = inv.cwiseProduct(in); };
    } else {
      sch = std::make_unique<SchwarzSmoother>(s, smoother == 1 ? SchwarzMode::Ras : SchwarzMode::Asm);
      S = sch->as_linop();
    }
    const LambdaEstimate est = estimate_lambda_max(S, A, s.n(), 10, 0);
    *value = est.value;
    *rounds = est.rounds_used;
  });
}

int ref_build_rhs(double eps, int E, int p, uint64_t seed, double* out) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p);
    FieldVector b = build_rhs(s, seed);
    std::memcpy(out, b.data(), sizeof(double) * size_t(s.n()));
  });
}

int ref_cheby_smooth(double eps, int E, int p, int smoother, int eta, double lam, const double* b, double* x) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p);
    LinOp A = [&s](const FieldVector& in, FieldVector& out) { out = s.apply_A(in); };
    FieldVector inv = jacobi_inverse_diag(s);
    std::unique_ptr<SchwarzSmoother> sch;
    LinOp S = [&inv](const FieldVector& in, FieldVector& out) { out = inv.cwiseProduct(in); };
    if (smoother != 0) {
      sch = std::make_unique<SchwarzSmoother>(s, smoother == 1 ? SchwarzMode::Ras : SchwarzMode::Asm);
      S = sch->as_linop();
    }
    ChebyshevSmoother cheb(S, A, ChebyParams{eta, 0.1, 1.1, lam});
    FieldVector bv = Eigen::Map<const Eigen::MatrixXd>(b, s.n(), 1);
    FieldVector xv = Eigen::Map<const Eigen::MatrixXd>(x, s.n(), 1);
    cheb.smooth(bv, xv);
    std::memcpy(x, xv.data(), sizeof(double) * size_t(s.n()));
  });
}

int ref_vcycle(double eps, int E, const int* orders, int nlev, const char* smoother, const char* coarse, int eta,
               const double* b, double* z, double* lams) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, orders[0]);
    Pmg pmg(m, orders_of(orders, nlev), smoother, eta, 0.1, 1.1, coarse);
    const Index n = pmg.spaces[0]->n();
    FieldVector bv = Eigen::Map<const Eigen::MatrixXd>(b, n, 1);
    FieldVector zv = pmg.vcycle(bv);
    std::memcpy(z, zv.data(), sizeof(double) * size_t(n));
    for (size_t l = 0; l < pmg.levels.size(); ++l) lams[l] = pmg.levels[l].lam;
  });
}

// Full solve from x0 = 0 with b = build_rhs(seed 1): krylov 0 = GMRES(20), 1 = PCG; precond "none",
// "jacobi" or a pMG smoother name with the given schedule.
int ref_solve(double eps, int E, const int* orders, int nlev, const char* precond, const char* coarse, int eta,
              int krylov, double tol, double* x, int* iters, double* rel_res, double* history, int hcap) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, orders[0]);
    std::unique_ptr<Pmg> pmg;
    std::unique_ptr<SemSpace> sp;
    const SemSpace* s0;
    LinOp M;
    FieldVector inv;
    const std::string pc(precond);
    if (pc == "none" || (pc == "jacobi" && nlev == 1)) {  // plain (Jacobi-)preconditioned Krylov
      sp = std::make_unique<SemSpace>(m, orders[0]);
      s0 = sp.get();
      if (pc == "jacobi") {
        inv = jacobi_inverse_diag(*s0);
        M = [&inv](const FieldVector& in, FieldVector& out) { out = inv.cwiseProduct(in); };
      }
    } else {
      pmg = std::make_unique<Pmg>(m, orders_of(orders, nlev), pc, eta, 0.1, 1.1, coarse);
      s0 = pmg->spaces[0].get();
      M = pmg->as_linop();
    }
    LinOp A = [s0](const FieldVector& in, FieldVector& out) { out = s0->apply_A(in); };
    FieldVector b = build_rhs(*s0, 1);
    FieldVector xv = FieldVector::Zero(s0->n());
    GmresStats st;
    if (krylov == 0) {
      GmresConfig cfg;
      cfg.tol = tol;
      st = gmres_solve(A, M, b, xv, cfg);
    } else {
      st = pcg_solve(A, M, b, xv, tol, 500);
    }
    std::memcpy(x, xv.data(), sizeof(double) * size_t(s0->n()));
    *iters = st.iterations;
    *rel_res = st.rel_residual;
    for (int i = 0; i < hcap && i < int(st.history.size()); ++i) history[i] = st.history[size_t(i)];
  });
}

// ---- handle-based cases (tests/golden/make_golden_scale.py): the mesh, spaces, smoothers and pMG of
// one configuration are built once and reused for every output at BASELINE sizes (E = 8^3 .. 32^3).
struct RefCase {
  HexMesh mesh;
  std::unique_ptr<Pmg> pmg;
  std::unique_ptr<SemSpace> own;
  const SemSpace* s0 = nullptr;
  FieldVector inv;
  LinOp A, M;
  std::unique_ptr<SchwarzSmoother> ras, asm_;
  RefCase(double eps, int E, int p) : mesh(mesh_of(eps, E, p)) {}
};

void* ref_case_create(double eps, int E, const int* orders, int nlev, const char* precond, const char* coarse,
                      int eta) {
  RefCase* c = nullptr;
  const int rc = guard([&] {
    auto cs = std::make_unique<RefCase>(eps, E, orders[0]);
    const std::string pc(precond);
    if (pc == "none" || (pc == "jacobi" && nlev == 1)) {
      cs->own = std::make_unique<SemSpace>(cs->mesh, orders[0]);
      cs->s0 = cs->own.get();
      if (pc == "jacobi") {
        cs->inv = jacobi_inverse_diag(*cs->s0);
        const FieldVector* inv = &cs->inv;
        cs->M = [inv](const FieldVector& in, FieldVector& out) { out = inv->cwiseProduct(in); };
      }
    } else {
      cs->pmg = std::make_unique<Pmg>(cs->mesh, orders_of(orders, nlev), pc, eta, 0.1, 1.1, coarse);
      cs->s0 = cs->pmg->spaces[0].get();
      cs->M = cs->pmg->as_linop();
    }
    const SemSpace* s0 = cs->s0;
    cs->A = [s0](const FieldVector& in, FieldVector& out) { out = s0->apply_A(in); };
    c = cs.release();
  });
  return rc == 0 ? c : nullptr;
}

void ref_case_destroy(void* h) { delete static_cast<RefCase*>(h); }

int64_t ref_case_n(void* h) { return static_cast<RefCase*>(h)->s0->n(); }

int ref_case_apply_A(void* h, const double* u, double* out) {
  return guard([&] {
    auto* c = static_cast<RefCase*>(h);
    FieldVector v = Eigen::Map<const Eigen::MatrixXd>(u, c->s0->n(), 1);
    FieldVector w = c->s0->apply_A(v);
    std::memcpy(out, w.data(), sizeof(double) * size_t(c->s0->n()));
  });
}

int ref_case_diag(void* h, double* out) {
  return guard([&] {
    auto* c = static_cast<RefCase*>(h);
    FieldVector d = c->s0->stiffness_diag();
    std::memcpy(out, d.data(), sizeof(double) * size_t(c->s0->n()));
  });
}

// mode 1 = RAS, 0 = ASM on the finest space (schwarz.cpp:242-289)
int ref_case_schwarz(void* h, int mode, const double* r, double* z) {
  return guard([&] {
    auto* c = static_cast<RefCase*>(h);
    auto& sch = mode == 1 ? c->ras : c->asm_;
    if (!sch) sch = std::make_unique<SchwarzSmoother>(*c->s0, mode == 1 ? SchwarzMode::Ras : SchwarzMode::Asm);
    FieldVector rv = Eigen::Map<const Eigen::MatrixXd>(r, c->s0->n(), 1);
    FieldVector zv = sch->apply(rv);
    std::memcpy(z, zv.data(), sizeof(double) * size_t(c->s0->n()));
  });
}

int ref_case_rhs(void* h, uint64_t seed, double* out) {
  return guard([&] {
    auto* c = static_cast<RefCase*>(h);
    FieldVector b = build_rhs(*c->s0, seed);
    std::memcpy(out, b.data(), sizeof(double) * size_t(c->s0->n()));
  });
}

// one V-cycle z = M b (pMG cases only); lams = the per-level lambda estimates
int ref_case_vcycle(void* h, const double* b, double* z, double* lams) {
  return guard([&] {
    auto* c = static_cast<RefCase*>(h);
    if (!c->pmg) throw std::invalid_argument("ref_case_vcycle: not a pMG case");
    FieldVector bv = Eigen::Map<const Eigen::MatrixXd>(b, c->s0->n(), 1);
    FieldVector zv = c->pmg->vcycle(bv);
    std::memcpy(z, zv.data(), sizeof(double) * size_t(c->s0->n()));
    for (size_t l = 0; l < c->pmg->levels.size(); ++l) lams[l] = c->pmg->levels[l].lam;
  });
}

// full solve from x0 = 0 with b = build_rhs(seed 1): krylov 0 = GMRES(restart), 1 = PCG
int ref_case_solve(void* h, int krylov, int restart, double tol, int max_iters, double* x, int* iters, double* rel_res,
                   double* history, int hcap) {
  return guard([&] {
    auto* c = static_cast<RefCase*>(h);
    FieldVector b = build_rhs(*c->s0, 1);
    FieldVector xv = FieldVector::Zero(c->s0->n());
    GmresStats st;
    if (krylov == 0) {
      GmresConfig cfg;
      cfg.restart = restart;
      cfg.tol = tol;
      cfg.max_iters = max_iters;
      st = gmres_solve(c->A, c->M, b, xv, cfg);
    } else {
      st = pcg_solve(c->A, c->M, b, xv, tol, max_iters);
    }
    std::memcpy(x, xv.data(), sizeof(double) * size_t(c->s0->n()));
    *iters = st.iterations;
    *rel_res = st.rel_residual;
    for (int i = 0; i < hcap && i < int(st.history.size()); ++i) history[i] = st.history[size_t(i)];
  });
}

// V-cycle with the extended pMG options (plain smoothers, additive cycle, Neumann levels): z = M b.
int ref_vcycle_ex(double eps, int E, const int* orders, int nlev, const char* smoother, const char* coarse, int eta,
                  int neumann, int additive, const double* b, double* z) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, orders[0]);
    Pmg pmg(m, orders_of(orders, nlev), smoother, eta, 0.1, 1.1, coarse,
            neumann ? BcMode::Neumann : BcMode::Dirichlet, additive != 0);
    const Index n = pmg.spaces[0]->n();
    FieldVector bv = Eigen::Map<const Eigen::MatrixXd>(b, n, 1);
    FieldVector zv = pmg.vcycle(bv);
    std::memcpy(z, zv.data(), sizeof(double) * size_t(n));
  });
}

// GMRES(20) to tol with that preconditioner on b (caller's vector), x0 = 0.
int ref_solve_ex(double eps, int E, const int* orders, int nlev, const char* smoother, const char* coarse, int eta,
                 int neumann, int additive, const double* b, double tol, double* x, int* iters, double* rel_res) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, orders[0]);
    Pmg pmg(m, orders_of(orders, nlev), smoother, eta, 0.1, 1.1, coarse,
            neumann ? BcMode::Neumann : BcMode::Dirichlet, additive != 0);
    const SemSpace* s0 = pmg.spaces[0].get();
    LinOp A = [s0](const FieldVector& in, FieldVector& out) { out = s0->apply_A(in); };
    LinOp M = pmg.as_linop();
    FieldVector bv = Eigen::Map<const Eigen::MatrixXd>(b, s0->n(), 1);
    FieldVector xv = FieldVector::Zero(s0->n());
    GmresConfig cfg;
    cfg.tol = tol;
    const GmresStats st = gmres_solve(A, M, bv, xv, cfg);
    std::memcpy(x, xv.data(), sizeof(double) * size_t(s0->n()));
    *iters = st.iterations;
    *rel_res = st.rel_residual;
  });
}

// SEMFEM preconditioner (semfem.cpp:12-134), AMG inner solve: z = M r, and the AMG level sizes.
int ref_semfem_apply(double eps, int E, int p, const double* r, double* z, int* nlev, int64_t* sizes, int cap) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p);
    SemfemPreconditioner pc(s, SemfemInner::Amg);
    FieldVector rv = Eigen::Map<const Eigen::MatrixXd>(r, s.n(), 1), zv;
    pc.apply(rv, zv);
    std::memcpy(z, zv.data(), sizeof(double) * size_t(s.n()));
    const AmgHierarchy* h = pc.hierarchy();
    *nlev = h->n_levels();
    for (int l = 0; l < h->n_levels() && l < cap; ++l) sizes[l] = h->level_size(l);
  });
}

// assemble_semfem (semfem.cpp:12-98) as CSR: ptr (n+1), idx/val (cap entries); *nnz set always.
int ref_semfem_matrix(double eps, int E, int p, int64_t* nnz, int64_t* ptr, int64_t* idx, double* val, int64_t cap) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p);
    const CsrMatrix A = assemble_semfem(s);
    *nnz = A.nonZeros();
    if (!ptr || A.nonZeros() > cap) return;
    int64_t k = 0;
    ptr[0] = 0;
    for (Index i = 0; i < A.rows(); ++i) {
      for (CsrMatrix::InnerIterator it(A, i); it; ++it) {
        idx[k] = it.col();
        val[k] = it.value();
        ++k;
      }
      ptr[i + 1] = k;
    }
  });
}

// GMRES(20) with A = apply_A and M = SEMFEM-AMG on b (caller's), x0 = 0.
int ref_semfem_solve(double eps, int E, int p, const double* b, double tol, double* x, int* iters, double* rel_res) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, p);
    SemSpace s(m, p);
    SemfemPreconditioner pc(s, SemfemInner::Amg);
    LinOp A = [&s](const FieldVector& in, FieldVector& out) { out = s.apply_A(in); };
    LinOp M = pc.as_linop();
    FieldVector bv = Eigen::Map<const Eigen::MatrixXd>(b, s.n(), 1);
    FieldVector xv = FieldVector::Zero(s.n());
    GmresConfig cfg;
    cfg.tol = tol;
    const GmresStats st = gmres_solve(A, M, bv, xv, cfg);
    std::memcpy(x, xv.data(), sizeof(double) * size_t(s.n()));
    *iters = st.iterations;
    *rel_res = st.rel_residual;
  });
}

// AMG hierarchy of the p=1 coarse problem (CoarseSolve "amg"): level sizes and the level-0
// aggregate of every free dof (tests compare the product's hierarchy against it).
int ref_amg_info(double eps, int E, int* nlev, int64_t* sizes, int cap, int* agg0) {
  return guard([&] {
    HexMesh m = mesh_of(eps, E, 1);
    SemSpace s(m, 1);
    CoarseSolve cs(s, "amg");
    const AmgHierarchy* h = cs.amg();
    *nlev = h->n_levels();
    for (int l = 0; l < h->n_levels() && l < cap; ++l) sizes[l] = h->level_size(l);
    if (agg0 && h->n_levels() > 1) {
      const auto& a = h->aggregates(0);
      for (size_t i = 0; i < a.size(); ++i) agg0[i] = a[i];
    }
  });
}

}  // extern "C"
