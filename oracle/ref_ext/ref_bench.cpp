// ORACLE / CPU BASELINE — times the reference semlab solve on the host (single-threaded, like the
// reference) for bench.py's cpu_baseline / --impl reference: the reference's own translation
// units (Eigen shim) + restated pMG/PCG/RHS. Prints one JSON line.
//   semlab_ref_bench --eps 0.3 --elems 8 --order 7 --smoother ras --coarse amg --cheb-order 2
//                    --krylov gmres --seconds 15
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>

#include "ref_ext.hpp"

using namespace semlab;
using namespace semlab_ref;

int main(int argc, char** argv) {
  double eps = 0.3, seconds = 15.0;
  int E = 8, p = 7, eta = 2, chunk = 5;
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
    else if (k == "--seconds") seconds = std::stod(v);
    else if (k == "--chunk") chunk = std::stoi(v);
  }
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  HexMesh m = generate_kershaw(KershawParams{eps, E}, p);
  std::vector<int> orders = p > 3 ? std::vector<int>{p, 3, 1} : std::vector<int>{p, 1};
  Pmg pmg(m, orders, smoother, eta, 0.1, 1.1, coarse);
  const SemSpace& s = *pmg.spaces[0];
  LinOp A = [&s](const FieldVector& in, FieldVector& out) { out = s.apply_A(in); };
  LinOp M = pmg.as_linop();
  FieldVector b = build_rhs(s, 1);
  const double t_setup = std::chrono::duration<double>(clk::now() - t0).count();
  long iters = 0;
  double t = 0.0;
  while (t < seconds && iters < 2000) {  // bounded sample: repeated chunks of Krylov iterations from x0 = 0
    FieldVector x = FieldVector::Zero(s.n());
    const auto ts = clk::now();
    GmresStats st;
    if (krylov == "gmres") {
      GmresConfig cfg;
      cfg.max_iters = chunk;
      st = gmres_solve(A, M, b, x, cfg);
    } else {
      st = pcg_solve(A, M, b, x, 1e-8, chunk);
    }
    t += std::chrono::duration<double>(clk::now() - ts).count();
    iters += st.iterations;
  }
  std::printf("{\"n\": %ld, \"iters\": %ld, \"t_solve_s\": %.6f, \"t_setup_s\": %.3f, \"gdof_iter_per_s\": %.9g}\n",
              long(s.n()), iters, t, t_setup, double(s.n()) * double(iters) / t / 1e9);
  return 0;
}
