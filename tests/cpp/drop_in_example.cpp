// Drop-in example: the reference call sequence (mesh -> space -> smoother -> Chebyshev ->
// GMRES), written against include/semlab_b200.hpp instead of proj/core/include/semlab/*.hpp.
// Built and run by tests/test_cpp_dropin_gpu.py; prints "OK <iterations> <rel_residual>".
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <type_traits>
#include <vector>

#include "semlab_b200.hpp"

// handle-owning wrappers are move-only (a copy would destroy the native handle twice)
static_assert(!std::is_copy_constructible<semlab_b200::SchwarzSmoother>::value, "copyable smoother");
static_assert(std::is_move_constructible<semlab_b200::SchwarzSmoother>::value, "immovable smoother");
static_assert(!std::is_copy_constructible<semlab_b200::Pmg>::value, "copyable pmg");
static_assert(std::is_copy_constructible<semlab_b200::LinOp>::value, "LinOp is copyable like std::function");

int main() {
  using namespace semlab_b200;
  Context ctx(0);
  auto mesh = generate_kershaw(ctx, KershawParams{0.3, 4}, 7);
  SemSpace space(mesh, 7);
  // operator check: A * 1 on the free dofs is 0 only in the Neumann sense; use a random vector
  FieldVector u(size_t(space.n()), 1.0);
  FieldVector w = space.apply_A(u);
  double s = 0.0;
  for (double v : w) s += std::abs(v);
  if (!(s > 0.0)) { std::printf("FAIL apply_A\n"); return 1; }
  // Chebyshev-RAS as in the reference chebyshev.hpp/schwarz.hpp
  SchwarzSmoother ras(space, SchwarzMode::Ras, 32);
  LinOp A = space.as_linop(), S = ras.as_linop();
  const LambdaEstimate lam = estimate_lambda_max(S, A, space.n(), 10, 0);
  ChebyshevSmoother cheb(S, A, ChebyParams{2, 0.1, 1.1, lam.value});
  // the reference's temporary-operator form: the smoother keeps its LinOps alive
  ChebyshevSmoother cheb_tmp(ras.as_linop(), space.as_linop(), ChebyParams{2, 0.1, 1.1, lam.value});
  {
    DeviceVector bb(space.n()), x1(space.n()), x2(space.n());
    check(semlab_space_build_rhs(space.handle(), 1, bb.data()));
    cheb.smooth(bb, x1);
    cheb_tmp.smooth(bb, x2);
    const FieldVector h1 = x1.download(), h2 = x2.download();
    if (h1 != h2) { std::printf("FAIL temporary-LinOp smoother\n"); return 1; }
  }
  // wrappers move through containers without double destruction
  std::vector<SchwarzSmoother> smoothers;
  smoothers.emplace_back(space, SchwarzMode::Ras, 32);
  smoothers.emplace_back(space, SchwarzMode::Asm, 64);
  smoothers.emplace_back(space, SchwarzMode::Ras, 64);
  // pMG-preconditioned GMRES(20) to 1e-8 (krylov.hpp)
  Pmg pmg(mesh, {7, 3, 1}, SEMLAB_SMOOTHER_RAS, 2, 32, SEMLAB_COARSE_DIRECT);
  LinOp M = pmg.as_linop();
  DeviceVector b(space.n()), x(space.n());
  check(semlab_space_build_rhs(space.handle(), 1, b.data()));
  GmresConfig cfg;
  GmresStats st = gmres_solve(A, &M, b, x, cfg);
  // projection onto prior solutions (krylov.hpp:39-59): the guess for a solved b is its solution
  ProjectionBasis proj(ctx, space.n(), 10);
  proj.insert(x, A);
  DeviceVector ug(space.n());
  proj.initial_guess(b, ug);
  const FieldVector xh = x.download(), uh = ug.download();
  double du = 0.0, xn = 0.0;
  for (size_t i = 0; i < xh.size(); ++i) {
    du = std::max(du, std::abs(uh[i] - xh[i]));
    xn = std::max(xn, std::abs(xh[i]));
  }
  if (proj.size() != 1 || !(du <= 1e-7 * xn)) { std::printf("FAIL projection %.3e\n", du / xn); return 1; }
  // exceptions mirror the reference: invalid parameters -> std::invalid_argument
  bool threw = false;
  try {
    ChebyshevSmoother bad(S, A, ChebyParams{0, 0.1, 1.1, 1.0});
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  if (!st.converged || !threw || !(lam.value > 0.0)) { std::printf("FAIL\n"); return 1; }
  std::printf("OK %d %.3e\n", st.iterations, st.rel_residual);
  return 0;
}
