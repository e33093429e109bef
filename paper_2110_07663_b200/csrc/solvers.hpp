// Chebyshev smoother, lambda estimate and Krylov solvers over device-resident vectors.
#pragma once

#include "objects.hpp"

struct semlab_cheby_s {
  semlab_ctx ctx = nullptr;
  semlab_op S = nullptr, A = nullptr;
  semlab_cheby_params params{};
  double theta = 0, delta = 0, sigma = 0;
  int64_t n = 0;
  sb::DevBuf<double> r, t, sad, d;
  void init(semlab_op S_, semlab_op A_, const semlab_cheby_params& p);
  // chebyshev.cpp:76-96; x_is_zero lets the first A x be skipped exactly (A 0 = 0).
  void smooth(const double* b, double* x, bool x_is_zero = false);
};

namespace sb {

semlab_lambda_estimate estimate_lambda_max(semlab_op S, semlab_op A, int64_t n, int rounds, uint64_t seed);

struct KrylovResult {
  int iterations = 0;
  bool converged = false, breakdown = false;
  double initial_residual = 0, abs_residual = 0, rel_residual = 0;
  std::vector<double> history;
};

// Owned-range descriptor for reductions of vectors of length n (single GPU: [0,n)).
struct OwnRange {
  int64_t n, off, len;
};
OwnRange own_range_of(semlab_op A);

KrylovResult gmres_solve(semlab_op A, semlab_op M, const double* b, double* x, const semlab_gmres_config& cfg);
KrylovResult pcg_solve(semlab_op A, semlab_op M, const double* b, double* x, const semlab_gmres_config& cfg);

}  // namespace sb

// ProjectionBasis (krylov.hpp:39-59) over device vectors.
struct semlab_proj_s {
  semlab_ctx ctx = nullptr;
  int64_t n = 0, ld = 0;
  int capacity = 0, size = 0;
  sb::OwnRange own{0, 0, 0};  // reduction range of the operator last inserted with
  sb::DevBuf<double> V, w, aw, dh;
  void init(semlab_ctx c, int64_t n_, int cap);
  void initial_guess(const double* b, double* u);
  void insert(const double* x, semlab_op A);
};
