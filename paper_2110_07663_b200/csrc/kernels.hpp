// Launchers of the sm_100a kernels (host-callable, plain pointers, no torch types).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.hpp"

namespace sb {

// ---- Ax epilogues: what the owner of a lattice node does with (A u)[g] ----------------------
enum class Epi : int {
  Write = 0,        // w[g] = Au
  Residual = 1,     // w[g] = b[g] - Au
  ChebJacStep = 2,  // x += d; r -= inv*Au; d = c1 d + c2 r        (chebyshev.cpp:86-92, S = Jacobi)
  ChebJacInit = 3,  // r = inv*(b - Au); d = r / c1                  (chebyshev.cpp:80-84, S = Jacobi)
};
struct EpiArgs {
  double* w = nullptr;
  const double* b = nullptr;
  double* x = nullptr;
  double* r = nullptr;
  double* d = nullptr;
  const double* inv = nullptr;
  double c1 = 0.0, c2 = 0.0;
};

// Sync state of the owner-ordered Ax kernel (one per space).
struct AxSync {
  double* dep = nullptr;      // E * nloc deposits (non-owned contributions)
  unsigned* flags = nullptr;  // E per-element completion counters
  unsigned* ticket = nullptr; // 1 dynamic CTA ticket counter
};

int64_t launch_geom(const Slab& sl, const double* d_X, double* d_geom, double* d_massw,
                    unsigned long long* d_bad, cudaStream_t s);
int64_t launch_ax(const Slab& sl, const double* d_u, const double* d_geom, const AxSync& sync, Epi epi,
                  const EpiArgs& a, cudaStream_t s);
// Same operator with FP32-rounded geometric factors (order 7 only): the smoother's A.
// orders with an FP32-factor Ax: 7 (k_axe) and the split-path orders (k_ax + k_gather_epi)
bool ax_g32_supported(int q);
int64_t launch_ax_g32(const Slab& sl, const double* d_u, const float* d_geom32, const AxSync& sync, Epi epi,
                      const EpiArgs& a, cudaStream_t s);
int64_t launch_to_f32(const double* in, float* out, int64_t n, cudaStream_t s);
int64_t launch_ax_local(const Slab& sl, const double* d_uloc, const double* d_geom, double* d_out,
                        cudaStream_t s);
int64_t launch_local_diag(const Slab& sl, const double* d_geom, double* d_out_local, cudaStream_t s);
int64_t launch_gather(const Slab& sl, const double* d_local, double* d_glob, cudaStream_t s);
int64_t launch_scatter(const Slab& sl, const double* d_glob, double* d_local, cudaStream_t s);
int64_t launch_qqt(const Slab& sl, const double* d_in, double* d_out, cudaStream_t s);
int64_t launch_mask(const Slab& sl, double* d_v, cudaStream_t s);
int64_t launch_invert_masked(const Slab& sl, const double* d_in, double* d_out, cudaStream_t s);

// ---- vector kernels ------------------------------------------------------------------------
int64_t launch_fill(double* d, int64_t n, double v, cudaStream_t s);
int64_t launch_copy(double* dst, const double* src, int64_t n, cudaStream_t s);
int64_t launch_axpby(double* y, double a, const double* x, double b, int64_t n, cudaStream_t s);  // y = a x + b y
int64_t launch_mul(double* y, const double* a, const double* x, int64_t n, cudaStream_t s);       // y = a .* x
int64_t launch_sub(double* y, const double* a, const double* b, int64_t n, cudaStream_t s);       // y = a - b
int64_t launch_div(double* y, const double* x, double a, int64_t n, cudaStream_t s);             // y = x / a
int64_t launch_add_planes(double* y, const double* a, const double* b, int64_t n, cudaStream_t s);  // y = a + b
// Chebyshev vector steps for a generic surrogate S (chebyshev.cpp:80-95)
int64_t launch_cheb_init(double* r, double* d, double theta, int64_t n, cudaStream_t s);  // d = r / theta
int64_t launch_cheb_step(double* x, double* r, double* d, const double* sad, double c1, double c2,
                         int64_t n, cudaStream_t s);  // x += d; r -= sad; d = c1 d + c2 r
int64_t launch_cheb_jac_zero_init(const double* b, const double* inv, double* r, double* d, double theta,
                                  int64_t n, cudaStream_t s);  // x = 0: r = inv*b; d = r/theta

// Deterministic multi-dot over [0, n): out[k] = sum_i a_k[i] * b_k[i] (device result).
struct DotScratch {
  double* partial = nullptr;  // >= kMaxDotBlocks * 32
  unsigned* counter = nullptr;
};
constexpr int kMaxDotBlocks = 148 * 8;  // enough CTAs in flight to stream at HBM rate
int64_t launch_dots(int K, const double* const* a, const double* const* b, int64_t n, double* d_out,
                    const DotScratch& ws, cudaStream_t s);

// ---- Krylov (CGS2 fused passes over the column-major basis V (ld = ldv)) -------------------
// h[0..j] = V^T w (any ncol, chunked by 32)
int64_t launch_gemv_t(const double* V, int64_t ldv, int ncol, const double* w, int64_t off, int64_t len,
                      double* d_h, const DotScratch& ws, cudaStream_t s);
// w -= V h ; h2 = V^T w  (update and re-projection in one pass)
int64_t launch_cgs_update_dot(const double* V, int64_t ldv, int ncol, double* w, const double* d_h,
                              int64_t n, int64_t off, int64_t len, double* d_h2, const DotScratch& ws,
                              cudaStream_t s);
// w -= V h2 ; nrm2 = w.w
int64_t launch_cgs_update_norm(const double* V, int64_t ldv, int ncol, double* w, const double* d_h2,
                               int64_t n, int64_t off, int64_t len, double* d_nrm2, const DotScratch& ws,
                               cudaStream_t s);
// y = V c, or y += V c with accumulate (host coefficients; any ncol, chunked by 32)
int64_t launch_gemv_n(const double* V, int64_t ldv, int ncol, const double* c_host, double* y, int64_t n,
                      cudaStream_t s, bool accumulate = false);
// Widest basis the fused CGS passes take in one launch; wider bases go in 32-column chunks.
constexpr int kKrylovChunk = 32;

}  // namespace sb
