// ORACLE / CPU BASELINE — times the reference semlab solve on the host for bench.py's
// --impl reference arm and its cpu_baseline leg: the reference's own translation units (compiled
// unmodified against the Eigen-API shim; single-threaded like the reference) + the restated
// pMG/PCG/RHS of ref_ext. Prints one JSON line.
//
//   semlab_ref_bench --eps 0.3 --elems 32 --order 7 --smoother ras --coarse amg --cheb-order 2
//                    --krylov gmres --iters 20 --warmup-iters 1
//
// Workload: the bench configuration itself (same mesh, order, schedule, smoother, coarse solve,
// Krylov method, b = build_rhs(seed 1), x0 = 0). After setup, --warmup-iters Krylov iterations
// run untimed (a separate solve call), then ONE solve call limited to --iters iterations is
// timed: the first --iters Arnoldi steps of the bench's solve (A, the V-cycle, CGS2), less one
// separately timed M + A application for the cycle close the solve call adds.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "ref_ext.hpp"

using namespace semlab;
using namespace semlab_ref;

int main(int argc, char** argv) {
  double eps = 0.3;
  int E = 32, p = 7, eta = 2, iters = 20, warm = 1, use_pmg = 1;
  std::string smoother = "ras", coarse = "amg", krylov = "gmres";
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--eps") eps = std::stod(v);
    else if (k == "--elems") E = std::stoi(v);
    else if (k == "--order") p = std::stoi(v);
    else if (k == "--smoother") smoother = v;
    else if (k == "--coarse") coarse = v;
    else if (k == "--cheb-order") eta = std::stoi(v);
    else if (k == "--krylov") krylov = v;
    else if (k == "--iters") iters = std::stoi(v);
    else if (k == "--warmup-iters") warm = std::stoi(v);
    else if (k == "--pmg") use_pmg = std::stoi(v);
  }
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  HexMesh m = generate_kershaw(KershawParams{eps, E}, p);
  std::vector<int> orders = p > 3 ? std::vector<int>{p, 3, 1} : std::vector<int>{p, 1};
  std::unique_ptr<Pmg> pmg;
  std::unique_ptr<SemSpace> own;
  FieldVector inv;
  LinOp M;
  if (use_pmg) {
    pmg = std::make_unique<Pmg>(m, orders, smoother, eta, 0.1, 1.1, coarse);
    M = pmg->as_linop();
  } else {  // config c1: Jacobi-preconditioned CG, no multigrid
    own = std::make_unique<SemSpace>(m, p);
    inv = jacobi_inverse_diag(*own);
    M = [&inv](const FieldVector& in, FieldVector& out) { out = inv.cwiseProduct(in); };
  }
  const SemSpace& s = use_pmg ? *pmg->spaces[0] : *own;
  LinOp A = [&s](const FieldVector& in, FieldVector& out) { out = s.apply_A(in); };
  FieldVector b = build_rhs(s, 1);
  const double t_setup = std::chrono::duration<double>(clk::now() - t0).count();
  auto solve = [&](int k) {
    FieldVector x = FieldVector::Zero(s.n());
    if (krylov == "gmres") {
      GmresConfig cfg;
      cfg.max_iters = k;
      return gmres_solve(A, M, b, x, cfg);
    }
    return pcg_solve(A, M, b, x, 1e-8, k);
  };
  double t_warm = 0.0;
  if (warm > 0) {
    const auto tw = clk::now();
    solve(warm);
    t_warm = std::chrono::duration<double>(clk::now() - tw).count();
  }
  const auto ts = clk::now();
  const GmresStats st = solve(iters);
  const double t = std::chrono::duration<double>(clk::now() - ts).count();
  // A solve call also runs the restart-cycle close: x += M (V y) and the true residual b - A x
  // (krylov.cpp:108-118), one M and one A application. Timed separately here and taken out, so
  // the rate is per Arnoldi iteration (A, M, CGS2) of the timed solve.
  double t_close = 0.0;
  if (krylov == "gmres") {
    FieldVector z(s.n()), w(s.n());
    const auto tc = clk::now();
    M(b, z);
    A(z, w);
    t_close = std::chrono::duration<double>(clk::now() - tc).count();
  }
  const double t_iter = std::max(t - t_close, 1e-9);
  std::printf("{\"n\": %ld, \"iters\": %d, \"t_solve_s\": %.6f, \"t_close_s\": %.6f, \"t_setup_s\": %.3f, "
              "\"t_warmup_s\": %.3f, \"rel_residual\": %.6e, \"gdof_iter_per_s\": %.9g}\n",
              long(s.n()), st.iterations, t, t_close, t_setup, t_warm, st.rel_residual,
              double(s.n()) * double(st.iterations) / t_iter / 1e9);
  return 0;
}
