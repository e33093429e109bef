// semlab_b200.hpp — header-only C++ wrapper over the C-ABI (semlab_b200.h) that re-exposes the
// reference library's API (proj/core/include/semlab/*.hpp) so a caller of semlab can switch by
// changing the include and the namespace. Names, argument meaning and exceptions follow the
// reference: std::invalid_argument for bad parameters, std::runtime_error for numerical failure,
// non-convergence reported in GmresStats::converged.
//
// FieldVector here is a host std::vector<double> (the reference uses Eigen::VectorXd); every
// host-vector call copies to/from the device and is meant for drop-in use and parity checks.
// The DeviceVector overloads keep a whole solve resident in HBM (the production path).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "semlab_b200.h"

namespace semlab_b200 {

using Index = int64_t;
using FieldVector = std::vector<double>;

inline void check(int rc) {
  if (rc == SEMLAB_OK) return;
  const std::string msg = semlab_last_error();
  if (rc == SEMLAB_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

class DeviceVector {  // owning device buffer
 public:
  DeviceVector() = default;
  explicit DeviceVector(Index n) : n_(n) {
    if (cudaMalloc(&p_, size_t(n) * sizeof(double)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
    cudaMemset(p_, 0, size_t(n) * sizeof(double));
  }
  DeviceVector(const FieldVector& h) : DeviceVector(Index(h.size())) { upload(h); }
  DeviceVector(const DeviceVector&) = delete;
  DeviceVector(DeviceVector&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  ~DeviceVector() { if (p_) cudaFree(p_); }
  double* data() { return p_; }
  const double* data() const { return p_; }
  Index size() const { return n_; }
  void upload(const FieldVector& h) { cudaMemcpy(p_, h.data(), size_t(n_) * sizeof(double), cudaMemcpyHostToDevice); }
  FieldVector download() const {
    FieldVector h(static_cast<size_t>(n_));
    cudaMemcpy(h.data(), p_, size_t(n_) * sizeof(double), cudaMemcpyDeviceToHost);
    return h;
  }

 private:
  double* p_ = nullptr;
  Index n_ = 0;
};

class Context {
 public:
  explicit Context(int device = 0, cudaStream_t stream = nullptr) { check(semlab_ctx_create(device, stream, &h_)); }
  ~Context() { semlab_ctx_destroy(h_); }
  Context(const Context&) = delete;
  semlab_ctx handle() const { return h_; }
  void synchronize() const { check(semlab_ctx_synchronize(h_)); }

 private:
  semlab_ctx h_ = nullptr;
};

struct KershawParams {  // mesh.hpp:17-20
  double eps = 1.0;
  int elements_per_axis = 6;
};
enum class BcMode { Dirichlet = SEMLAB_BC_DIRICHLET, Neumann = SEMLAB_BC_NEUMANN };
enum class SchwarzMode { Asm = SEMLAB_SCHWARZ_ASM, Ras = SEMLAB_SCHWARZ_RAS };

class HexMesh {  // mesh.hpp:44-100
 public:
  static std::shared_ptr<HexMesh> box(Context& ctx, std::array<int, 3> dims, std::array<double, 3> lo,
                                      std::array<double, 3> hi) {
    auto m = std::shared_ptr<HexMesh>(new HexMesh);
    check(semlab_mesh_box(ctx.handle(), dims.data(), lo.data(), hi.data(), &m->h_));
    return m;
  }
  ~HexMesh() { semlab_mesh_destroy(h_); }
  semlab_mesh handle() const { return h_; }

 private:
  HexMesh() = default;
  friend std::shared_ptr<HexMesh> generate_kershaw(Context&, const KershawParams&, int);
  semlab_mesh h_ = nullptr;
};

// generate_kershaw(params, p), mesh.cpp:138-171 (p is accepted for signature parity)
inline std::shared_ptr<HexMesh> generate_kershaw(Context& ctx, const KershawParams& params, int /*p*/) {
  auto m = std::shared_ptr<HexMesh>(new HexMesh);
  check(semlab_mesh_kershaw(ctx.handle(), params.eps, params.elements_per_axis, &m->h_));
  return m;
}

class LinOp {  // types.hpp:13 (device-resident operator)
 public:
  explicit LinOp(semlab_op h = nullptr, bool own = true) : h_(h), own_(own) {}
  LinOp(LinOp&& o) noexcept : h_(o.h_), own_(o.own_) { o.h_ = nullptr; }
  LinOp(const LinOp&) = delete;
  ~LinOp() { if (h_ && own_) semlab_op_destroy(h_); }
  explicit operator bool() const { return h_ != nullptr; }
  semlab_op handle() const { return h_; }
  void operator()(const DeviceVector& in, DeviceVector& out) const { check(semlab_op_apply(h_, in.data(), out.data())); }

 private:
  semlab_op h_;
  bool own_;
};

class SemSpace {  // sem_space.hpp:26-129
 public:
  SemSpace(std::shared_ptr<HexMesh> mesh, int order, BcMode bc = BcMode::Dirichlet) : mesh_(std::move(mesh)) {
    check(semlab_space_create(mesh_->handle(), order, int(bc), &h_));
    check(semlab_space_sizes(h_, sizes_));
  }
  ~SemSpace() { semlab_space_destroy(h_); }
  SemSpace(const SemSpace&) = delete;
  semlab_space handle() const { return h_; }
  Index n() const { return sizes_[0]; }
  Index n_free() const { return sizes_[1]; }
  Index n_local_total() const { return sizes_[2]; }
  // apply_A, sem_space.cpp:195-209
  FieldVector apply_A(const FieldVector& u) const {
    DeviceVector du(u), dw(n());
    apply_A(du, dw);
    return dw.download();
  }
  void apply_A(const DeviceVector& u, DeviceVector& w) const { check(semlab_space_apply_A(h_, u.data(), w.data())); }
  FieldVector stiffness_diag() const {
    DeviceVector d(n());
    check(semlab_space_stiffness_diag(h_, d.data()));
    return d.download();
  }
  FieldVector mass_diag() const {
    DeviceVector d(n());
    check(semlab_space_mass_diag(h_, d.data()));
    return d.download();
  }
  FieldVector gather(const FieldVector& local) const {
    DeviceVector dl(local), dg(n());
    check(semlab_space_gather(h_, dl.data(), dg.data()));
    return dg.download();
  }
  FieldVector scatter(const FieldVector& global) const {
    DeviceVector dg(global), dl(n_local_total());
    check(semlab_space_scatter(h_, dg.data(), dl.data()));
    return dl.download();
  }
  LinOp as_linop() const {
    semlab_op o;
    check(semlab_op_A(h_, &o));
    return LinOp(o);
  }
  LinOp jacobi() const {
    semlab_op o;
    check(semlab_op_jacobi(h_, &o));
    return LinOp(o);
  }

 private:
  std::shared_ptr<HexMesh> mesh_;
  semlab_space h_ = nullptr;
  int64_t sizes_[11] = {};
};

class SchwarzSmoother {  // schwarz.hpp:31-86 (precision: 32 = paper's FP32 FDM, 64 = reference arithmetic)
 public:
  SchwarzSmoother(const SemSpace& space, SchwarzMode mode, int precision = 32) : n_(space.n()) {
    check(semlab_schwarz_create(space.handle(), int(mode), precision, &h_));
  }
  ~SchwarzSmoother() { semlab_schwarz_destroy(h_); }
  FieldVector apply(const FieldVector& r) const {
    DeviceVector dr(r), dz(n_);
    check(semlab_schwarz_apply(h_, dr.data(), dz.data()));
    return dz.download();
  }
  LinOp as_linop() const {
    semlab_op o;
    check(semlab_op_schwarz(h_, &o));
    return LinOp(o);
  }

 private:
  semlab_schwarz h_ = nullptr;
  Index n_;
};

struct ChebyParams {  // chebyshev.hpp:9-14
  int order = 2;
  double lambda_min_mult = 0.1;
  double lambda_max_mult = 1.1;
  double lambda_max_est = 0.0;
};
struct LambdaEstimate {
  double value = 0.0;
  bool breakdown = false;
  int rounds_used = 0;
};

inline LambdaEstimate estimate_lambda_max(const LinOp& S, const LinOp& A, Index n, int rounds = 10,
                                          uint64_t seed = 0) {  // chebyshev.cpp:9-56
  semlab_lambda_estimate e;
  check(semlab_estimate_lambda_max(S.handle(), A.handle(), n, rounds, seed, &e));
  return {e.value, e.breakdown != 0, e.rounds_used};
}

class ChebyshevSmoother {  // chebyshev.hpp:36-46
 public:
  ChebyshevSmoother(const LinOp& S, const LinOp& A, const ChebyParams& p) {
    semlab_cheby_params cp{p.order, p.lambda_min_mult, p.lambda_max_mult, p.lambda_max_est};
    check(semlab_cheby_create(S.handle(), A.handle(), &cp, &h_));
  }
  ~ChebyshevSmoother() { semlab_cheby_destroy(h_); }
  void smooth(const DeviceVector& b, DeviceVector& x) const { check(semlab_cheby_smooth(h_, b.data(), x.data())); }

 private:
  semlab_cheby h_ = nullptr;
};

// ProjectionBasis, krylov.hpp:39-59. The device basis needs its context and vector length up
// front (the reference sizes it from the first inserted vector).
class ProjectionBasis {
 public:
  ProjectionBasis(const Context& ctx, Index n, int capacity = 10) : capacity_(capacity) {
    check(semlab_proj_create(ctx.handle(), n, capacity, &h_));
  }
  ~ProjectionBasis() { semlab_proj_destroy(h_); }
  ProjectionBasis(const ProjectionBasis&) = delete;
  void initial_guess(const DeviceVector& b, DeviceVector& u) const {
    check(semlab_proj_initial_guess(h_, b.data(), u.data()));
  }
  void insert(const DeviceVector& x, const LinOp& A) {
    if (!A) throw std::invalid_argument("ProjectionBasis: missing operator");
    check(semlab_proj_insert(h_, x.data(), A.handle()));
  }
  int size() const {
    int k = 0;
    check(semlab_proj_size(h_, &k));
    return k;
  }
  int capacity() const { return capacity_; }
  void clear() { check(semlab_proj_clear(h_)); }

 private:
  semlab_proj h_ = nullptr;
  int capacity_;
};

class Pmg {  // pMG V-cycle (pmg.cpp missing in the reference)
 public:
  Pmg(std::shared_ptr<HexMesh> mesh, std::vector<int> orders, int smoother = SEMLAB_SMOOTHER_RAS, int cheb_order = 2,
      int precision = 32, int coarse = SEMLAB_COARSE_AMG)
      : mesh_(std::move(mesh)) {
    check(semlab_pmg_create(mesh_->handle(), int(orders.size()), orders.data(), smoother, cheb_order, 0.1, 1.1,
                            precision, coarse, &h_));
  }
  ~Pmg() { semlab_pmg_destroy(h_); }
  semlab_space fine_space() const {
    semlab_space s;
    check(semlab_pmg_space(h_, 0, &s));
    return s;
  }
  LinOp as_linop() const {
    semlab_op o;
    check(semlab_op_pmg(h_, &o));
    return LinOp(o);
  }

 private:
  std::shared_ptr<HexMesh> mesh_;
  semlab_pmg h_ = nullptr;
};

struct GmresConfig {  // krylov.hpp:9-15
  int restart = 20;
  double tol = 1e-8;
  int max_iters = 500;
  bool use_abs_tol = false;
  double abs_tol = 0.0;
};
struct GmresStats {  // krylov.hpp:17-25
  int iterations = 0;
  bool converged = false;
  bool breakdown = false;
  double initial_residual = 0.0, abs_residual = 0.0, rel_residual = 0.0;
  std::vector<double> history;
};

namespace detail {
inline GmresStats run(int (*fn)(semlab_op, semlab_op, const double*, double*, const semlab_gmres_config*,
                                semlab_gmres_stats*),
                      const LinOp& A, const LinOp* M, const DeviceVector& b, DeviceVector& x, const GmresConfig& c) {
  semlab_gmres_config cfg{c.restart, c.tol, c.max_iters, c.use_abs_tol ? 1 : 0, c.abs_tol};
  GmresStats st;
  st.history.assign(size_t(c.max_iters), 0.0);
  semlab_gmres_stats s{};
  s.history = st.history.data();
  s.history_capacity = c.max_iters;
  check(fn(A.handle(), M ? M->handle() : nullptr, b.data(), x.data(), &cfg, &s));
  st.iterations = s.iterations;
  st.converged = s.converged != 0;
  st.breakdown = s.breakdown != 0;
  st.initial_residual = s.initial_residual;
  st.abs_residual = s.abs_residual;
  st.rel_residual = s.rel_residual;
  st.history.resize(size_t(s.history_len));
  return st;
}
}  // namespace detail

// gmres_solve(A, M, b, x, config), krylov.cpp:20-129 (M may be null = identity)
inline GmresStats gmres_solve(const LinOp& A, const LinOp* M, const DeviceVector& b, DeviceVector& x,
                              const GmresConfig& config) {
  return detail::run(semlab_gmres_solve, A, M, b, x, config);
}
inline GmresStats pcg_solve(const LinOp& A, const LinOp* M, const DeviceVector& b, DeviceVector& x,
                            const GmresConfig& config) {
  return detail::run(semlab_pcg_solve, A, M, b, x, config);
}

}  // namespace semlab_b200
