// The reference-side binding, exercised: the UNMODIFIED reference gmres_solve (krylov.cpp:20-129,
// compiled from /root/reference into oracle/_ref by oracle/Makefile) runs with A = the B200
// apply_A and M = the B200 pMG V-cycle, through include/semlab_b200_linop.hpp. The same solve
// then runs device-resident through semlab_gmres_solve. Prints one line:
//   OK <ref iterations> <ref rel residual> <b200 iterations> <b200 rel residual> <max |x_ref - x_b200| / max |x|>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "semlab/krylov.hpp"
#include "semlab_b200_linop.hpp"

#define CK(call)                                                          \
  do {                                                                    \
    if ((call) != SEMLAB_OK) {                                            \
      std::printf("FAIL %s: %s\n", #call, semlab_last_error());           \
      return 1;                                                           \
    }                                                                     \
  } while (0)

int main(int argc, char** argv) {
  const int E = argc > 1 ? std::atoi(argv[1]) : 4;
  semlab_ctx ctx;
  CK(semlab_ctx_create(0, nullptr, &ctx));
  semlab_mesh mesh;
  CK(semlab_mesh_kershaw(ctx, 0.3, E, &mesh));
  const int orders[3] = {7, 3, 1};
  semlab_pmg pmg;
  CK(semlab_pmg_create(mesh, 3, orders, SEMLAB_SMOOTHER_RAS, 2, 0.1, 1.1, 64, SEMLAB_COARSE_DIRECT, &pmg));
  semlab_space sp;
  CK(semlab_pmg_space(pmg, 0, &sp));
  int64_t sizes[11];
  CK(semlab_space_sizes(sp, sizes));
  const int64_t n = sizes[0];
  semlab_op A, M;
  CK(semlab_op_A(sp, &A));
  CK(semlab_op_pmg(pmg, &M));
  double *db, *dx;
  cudaMalloc(&db, n * sizeof(double));
  cudaMalloc(&dx, n * sizeof(double));
  CK(semlab_space_build_rhs(sp, 1, db));
  Eigen::VectorXd b(n), x_ref = Eigen::VectorXd::Zero(n);
  cudaMemcpy(b.data(), db, n * sizeof(double), cudaMemcpyDeviceToHost);
  // the reference's own GMRES(20) over B200 operators
  semlab::LinOp Aop = b200_linop(A, n), Mop = b200_linop(M, n);
  semlab::GmresConfig cfg;
  const semlab::GmresStats st = semlab::gmres_solve(Aop, Mop, b, x_ref, cfg);
  // the device-resident product solve
  cudaMemset(dx, 0, n * sizeof(double));
  semlab_gmres_config c{cfg.restart, cfg.tol, cfg.max_iters, 0, 0.0};
  std::vector<double> hist(size_t(cfg.max_iters));
  semlab_gmres_stats s{};
  s.history = hist.data();
  s.history_capacity = cfg.max_iters;
  CK(semlab_gmres_solve(A, M, db, dx, &c, &s));
  std::vector<double> x(size_t(n));
  cudaMemcpy(x.data(), dx, n * sizeof(double), cudaMemcpyDeviceToHost);
  double dmax = 0.0, xmax = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    dmax = std::max(dmax, std::abs(x[size_t(i)] - x_ref[i]));
    xmax = std::max(xmax, std::abs(x_ref[i]));
  }
  std::printf("OK %d %.6e %d %.6e %.3e\n", st.iterations, st.rel_residual, s.iterations, s.rel_residual, dmax / xmax);
  semlab_op_destroy(A);
  semlab_op_destroy(M);
  semlab_pmg_destroy(pmg);
  semlab_mesh_destroy(mesh);
  semlab_ctx_destroy(ctx);
  return 0;
}
