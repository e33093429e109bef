// Launchers of the Schwarz/FDM kernels (k_fdm.cu).
#pragma once

#include <cuda_runtime.h>

#include "common.hpp"

namespace sb {

// Owner-write epilogue of the RAS kernel. mode 0: out = z. mode 1 (Chebyshev init):
// r = z, d = z * c2 (c2 = 1 / theta). mode 2 (Chebyshev step): x += d; r -= z; d = c1 d + c2 r.
// mode 3 (last step): mode 2 followed by the final x += d, bit for bit; r and d not written.
struct RasEpi {
  double* out = nullptr;
  double* x = nullptr;
  double* r = nullptr;
  double* d = nullptr;
  double c1 = 0.0, c2 = 0.0;
};

// S: E x 3 x P x P (row-major S(a, a')), L: E x 3 x P eigenvalues (padding: S = 0, L = 1);
// P = order + 3; precision 32 -> float arrays, 64 -> double arrays.
int64_t launch_ras(const Slab& sl, int precision, const void* S, const void* L, const double* r, int mode,
                   const RasEpi& e, cudaStream_t s);
// ASM: boxes = E x P^3 scratch of the precision's type; out written on the slab's planes. On a
// slab (internal boundaries) the exchange planes get raw sums in out and counts in cnt
// (6 planes of Nx*Ny: zb-1, zb, zb+1, zt-1, zt, zt+1); see semlab_schwarz_s::apply.
int64_t launch_asm(const Slab& sl, int precision, const void* S, const void* L, const double* r, void* boxes,
                   double* out, double* cnt, cudaStream_t s);
// v = (lo_sum + hi_sum) / (lo_cnt + hi_cnt) over one plane (0 where the count is 0)
int64_t launch_asm_combine(double* v, const double* lo_sum, const double* lo_cnt, const double* hi_sum,
                           const double* hi_cnt, int64_t P, cudaStream_t s);
// fdm_solve on E padded boxes (FP64 in/out).
int64_t launch_fdm_boxes(const Slab& sl, int precision, const void* S, const void* L, const double* in,
                         double* out, cudaStream_t s);

}  // namespace sb
