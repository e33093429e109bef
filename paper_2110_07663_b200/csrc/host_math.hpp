// Host-side setup mathematics (no Eigen: it is not available on this image).
#pragma once

#include <array>
#include <cstdint>
#include <vector>

namespace sb {

// GLL nodes/weights/differentiation matrix (column-major, D(i,m) = diff[i + nd*m], like
// Eigen's default storage read at sem_space.cpp:132) — gll.cpp:12-134.
struct Gll {
  int order = 0;
  std::vector<double> nodes, weights, diff;
};
const Gll& gll(int order);
std::vector<double> lagrange_interpolation_matrix(const std::vector<double>& from,
                                                  const std::vector<double>& to);  // row-major m x n

// Kershaw map, mesh.cpp:17-55.
std::array<double, 3> kershaw_map(double eps, double x, double y, double z);

// std::uniform_real_distribution<double>(-1,1) over std::mt19937_64(seed) (chebyshev.cpp:12-15).
void uniform_pm1(uint64_t seed, int64_t n, double* out);
// The same stream starting at draw `offset` (for slab-local pieces of a global vector).
void uniform_pm1_range(uint64_t seed, int64_t offset, int64_t n, double* out);

// A s = lambda B s, A symmetric, B SPD, n <= 16: lambda ascending, S (column-major) with
// S^T B S = I — the contract of GeneralizedSelfAdjointEigenSolver used at schwarz.cpp:207-212.
// Returns false if B is not positive definite.
bool gen_sym_eig(int n, const double* A, const double* B, double* lambda, double* S);

// max |eig(H)| for a small real (Hessenberg) matrix, column-major — EigenSolver at
// chebyshev.cpp:53-54. Francis double-shift QR.
double max_abs_eig(int n, const double* H_colmajor);

}  // namespace sb
