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

// Move-only owner of a C handle: every wrapper object below owns exactly one handle, so a copy
// (vector push_back, reallocation) can never destroy it twice. Moves transfer ownership.
template <class H, int (*Destroy)(H)>
class Owned {
 public:
  Owned() = default;
  explicit Owned(H h) : h_(h) {}
  Owned(Owned&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  Owned& operator=(Owned&& o) noexcept {
    if (this != &o) {
      reset();
      h_ = o.h_;
      o.h_ = nullptr;
    }
    return *this;
  }
  Owned(const Owned&) = delete;
  Owned& operator=(const Owned&) = delete;
  ~Owned() { reset(); }
  void reset() {
    if (h_) Destroy(h_);
    h_ = nullptr;
  }
  H get() const { return h_; }
  H* out() {
    reset();
    return &h_;
  }

 private:
  H h_ = nullptr;
};

class DeviceVector {  // owning device buffer
 public:
  DeviceVector() = default;
  explicit DeviceVector(Index n) : n_(n) {
    if (cudaMalloc(&p_, size_t(n) * sizeof(double)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
    cudaMemset(p_, 0, size_t(n) * sizeof(double));
  }
  DeviceVector(const FieldVector& h) : DeviceVector(Index(h.size())) { upload(h); }
  DeviceVector(const DeviceVector&) = delete;
  DeviceVector& operator=(const DeviceVector&) = delete;
  DeviceVector(DeviceVector&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DeviceVector& operator=(DeviceVector&& o) noexcept {
    if (this != &o) {
      if (p_) cudaFree(p_);
      p_ = o.p_;
      n_ = o.n_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
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
  explicit Context(int device = 0, cudaStream_t stream = nullptr) { check(semlab_ctx_create(device, stream, h_.out())); }
  semlab_ctx handle() const { return h_.get(); }
  void synchronize() const { check(semlab_ctx_synchronize(h_.get())); }

 private:
  Owned<semlab_ctx, semlab_ctx_destroy> h_;
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
    check(semlab_mesh_box(ctx.handle(), dims.data(), lo.data(), hi.data(), m->h_.out()));
    return m;
  }
  semlab_mesh handle() const { return h_.get(); }

 private:
  HexMesh() = default;
  friend std::shared_ptr<HexMesh> generate_kershaw(Context&, const KershawParams&, int);
  Owned<semlab_mesh, semlab_mesh_destroy> h_;
};

// generate_kershaw(params, p), mesh.cpp:138-171 (p is accepted for signature parity)
inline std::shared_ptr<HexMesh> generate_kershaw(Context& ctx, const KershawParams& params, int /*p*/) {
  auto m = std::shared_ptr<HexMesh>(new HexMesh);
  check(semlab_mesh_kershaw(ctx.handle(), params.eps, params.elements_per_axis, m->h_.out()));
  return m;
}

class LinOp {  // types.hpp:13 (device-resident operator)
  // Copyable like the reference's std::function: copies share the one native operator, which is
  // destroyed with the last copy. Objects that use a LinOp (ChebyshevSmoother) keep a copy.
 public:
  LinOp() = default;
  explicit LinOp(semlab_op h) : h_(h, [](semlab_op o) { semlab_op_destroy(o); }) {}
  explicit operator bool() const { return h_ != nullptr; }
  semlab_op handle() const { return h_.get(); }
  void operator()(const DeviceVector& in, DeviceVector& out) const {
    check(semlab_op_apply(h_.get(), in.data(), out.data()));
  }

 private:
  std::shared_ptr<semlab_op_s> h_;
};

class SemSpace {  // sem_space.hpp:26-129
 public:
  SemSpace(std::shared_ptr<HexMesh> mesh, int order, BcMode bc = BcMode::Dirichlet) : mesh_(std::move(mesh)) {
    check(semlab_space_create(mesh_->handle(), order, int(bc), h_.out()));
    check(semlab_space_sizes(h_.get(), sizes_));
  }
  semlab_space handle() const { return h_.get(); }
  Index n() const { return sizes_[0]; }
  Index n_free() const { return sizes_[1]; }
  Index n_local_total() const { return sizes_[2]; }
  // apply_A, sem_space.cpp:195-209
  FieldVector apply_A(const FieldVector& u) const {
    DeviceVector du(u), dw(n());
    apply_A(du, dw);
    return dw.download();
  }
  void apply_A(const DeviceVector& u, DeviceVector& w) const { check(semlab_space_apply_A(h_.get(), u.data(), w.data())); }
  FieldVector stiffness_diag() const {
    DeviceVector d(n());
    check(semlab_space_stiffness_diag(h_.get(), d.data()));
    return d.download();
  }
  FieldVector mass_diag() const {
    DeviceVector d(n());
    check(semlab_space_mass_diag(h_.get(), d.data()));
    return d.download();
  }
  FieldVector gather(const FieldVector& local) const {
    DeviceVector dl(local), dg(n());
    check(semlab_space_gather(h_.get(), dl.data(), dg.data()));
    return dg.download();
  }
  FieldVector scatter(const FieldVector& global) const {
    DeviceVector dg(global), dl(n_local_total());
    check(semlab_space_scatter(h_.get(), dg.data(), dl.data()));
    return dl.download();
  }
  LinOp as_linop() const {
    semlab_op o;
    check(semlab_op_A(h_.get(), &o));
    return LinOp(o);
  }
  LinOp jacobi() const {
    semlab_op o;
    check(semlab_op_jacobi(h_.get(), &o));
    return LinOp(o);
  }

 private:
  std::shared_ptr<HexMesh> mesh_;
  Owned<semlab_space, semlab_space_destroy> h_;
  int64_t sizes_[11] = {};
};

class SchwarzSmoother {  // schwarz.hpp:31-86 (precision: 32 = paper's FP32 FDM, 64 = reference arithmetic)
 public:
  SchwarzSmoother(const SemSpace& space, SchwarzMode mode, int precision = 32) : n_(space.n()) {
    check(semlab_schwarz_create(space.handle(), int(mode), precision, h_.out()));
  }
  FieldVector apply(const FieldVector& r) const {
    DeviceVector dr(r), dz(n_);
    check(semlab_schwarz_apply(h_.get(), dr.data(), dz.data()));
    return dz.download();
  }
  LinOp as_linop() const {
    semlab_op o;
    check(semlab_op_schwarz(h_.get(), &o));
    return LinOp(o);
  }

 private:
  Owned<semlab_schwarz, semlab_schwarz_destroy> h_;
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
  // Takes its operators by value like the reference (chebyshev.hpp:36) and keeps them: the C
  // object only borrows the native operators, so temporaries such as
  // ChebyshevSmoother c(sch.as_linop(), sp.as_linop(), p) stay alive as long as the smoother.
 public:
  ChebyshevSmoother(LinOp S, LinOp A, const ChebyParams& p) : S_(std::move(S)), A_(std::move(A)) {
    semlab_cheby_params cp{p.order, p.lambda_min_mult, p.lambda_max_mult, p.lambda_max_est};
    check(semlab_cheby_create(S_.handle(), A_.handle(), &cp, h_.out()));
  }
  void smooth(const DeviceVector& b, DeviceVector& x) const {
    check(semlab_cheby_smooth(h_.get(), b.data(), x.data()));
  }

 private:
  LinOp S_, A_;  // declared before h_: destroyed after the smoother that borrows them
  Owned<semlab_cheby, semlab_cheby_destroy> h_;
};

// ProjectionBasis, krylov.hpp:39-59. The device basis needs its context and vector length up
// front (the reference sizes it from the first inserted vector).
class ProjectionBasis {
 public:
  ProjectionBasis(const Context& ctx, Index n, int capacity = 10) : capacity_(capacity) {
    check(semlab_proj_create(ctx.handle(), n, capacity, h_.out()));
  }
  void initial_guess(const DeviceVector& b, DeviceVector& u) const {
    check(semlab_proj_initial_guess(h_.get(), b.data(), u.data()));
  }
  void insert(const DeviceVector& x, const LinOp& A) {
    if (!A) throw std::invalid_argument("ProjectionBasis: missing operator");
    check(semlab_proj_insert(h_.get(), x.data(), A.handle()));
  }
  int size() const {
    int k = 0;
    check(semlab_proj_size(h_.get(), &k));
    return k;
  }
  int capacity() const { return capacity_; }
  void clear() { check(semlab_proj_clear(h_.get())); }

 private:
  Owned<semlab_proj, semlab_proj_destroy> h_;
  int capacity_;
};

class Pmg {  // pMG V-cycle (pmg.cpp missing in the reference)
 public:
  Pmg(std::shared_ptr<HexMesh> mesh, std::vector<int> orders, int smoother = SEMLAB_SMOOTHER_RAS, int cheb_order = 2,
      int precision = 32, int coarse = SEMLAB_COARSE_AMG)
      : mesh_(std::move(mesh)) {
    check(semlab_pmg_create(mesh_->handle(), int(orders.size()), orders.data(), smoother, cheb_order, 0.1, 1.1,
                            precision, coarse, h_.out()));
  }
  semlab_space fine_space() const {
    semlab_space s;
    check(semlab_pmg_space(h_.get(), 0, &s));
    return s;
  }
  LinOp as_linop() const {
    semlab_op o;
    check(semlab_op_pmg(h_.get(), &o));
    return LinOp(o);
  }

 private:
  std::shared_ptr<HexMesh> mesh_;
  Owned<semlab_pmg, semlab_pmg_destroy> h_;
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
