// Krylov kernels for sm_100a: fused classical Gram-Schmidt passes over the column-major basis
// V (krylov.cpp:67-72, chebyshev.cpp:36-41), and the basis combination V*y (krylov.cpp:111).
// Every reduction is deterministic: per-block partials in a fixed shape, then the last block to
// finish sums the partials in block order. Kernels are instantiated per column-count bucket
// (NC >= ncol) so accumulators stay in registers.
#include <algorithm>

#include "device.cuh"
#include "kernels.hpp"

namespace sb {

namespace {

#ifndef SEMLAB_CGS_MINB
#define SEMLAB_CGS_MINB 2  // resident blocks per SM the dot kernels are register-capped for (1: 12% slower at 24 columns)
#endif

constexpr int kMaxCol = 32;
constexpr int kNT = 256;

struct Coef {
  double c[kMaxCol];
};

// Sum per-block partial vectors (ncol each) in block order; the last block writes out.
template <int NC>
__device__ __forceinline__ void finish_partials(double (&acc)[NC], int ncol, double* partial, unsigned* counter,
                                                double* out) {
  __shared__ double sred[NC * (kNT / 32)];
  __shared__ bool last;
  block_sum<NC, kNT>(acc, sred);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c)  // static indices keep acc in registers
      if (c < ncol) partial[blockIdx.x * kMaxCol + c] = acc[c];
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  // the whole last block reduces the partials: fixed strided shape, then a block sum
  __threadfence();
  double s[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) s[c] = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += kNT)
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c < ncol) s[c] += __ldcg(&partial[b * kMaxCol + c]);
  block_sum<NC, kNT>(s, sred);
  if (threadIdx.x < NC && threadIdx.x < ncol) {
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c == int(threadIdx.x)) out[c] = s[c];
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// h = V^T w over the owned range
template <int NC>
__global__ void __launch_bounds__(kNT, SEMLAB_CGS_MINB) k_gemv_t(const double* __restrict__ V, int64_t ldv, int ncol,
                                                const double* __restrict__ w, int64_t off, int64_t len,
                                                double* __restrict__ h, double* partial, unsigned* counter) {
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  for (int64_t t = int64_t(blockIdx.x) * kNT + threadIdx.x; t < len; t += int64_t(gridDim.x) * kNT) {
    const int64_t i = off + t;
    const double wi = w[i];
    double v[NC];  // every column load issued before the first use (no per-column branch)
#pragma unroll
    for (int c = 0; c < NC; ++c) v[c] = c < ncol ? __ldcs(V + c * ldv + i) : 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = fma(v[c], wi, acc[c]);
  }
  finish_partials<NC>(acc, ncol, partial, counter, h);
}

// w -= V h over [0,n); h2 = V^T w over the owned range (one read of V for both)
template <int NC>
__global__ void __launch_bounds__(kNT, SEMLAB_CGS_MINB) k_cgs_update_dot(const double* __restrict__ V, int64_t ldv, int ncol,
                                                        double* __restrict__ w, const double* __restrict__ h,
                                                        int64_t n, int64_t off, int64_t len,
                                                        double* __restrict__ h2, double* partial,
                                                        unsigned* counter) {
  __shared__ double sh[NC];
  if (threadIdx.x < NC) sh[threadIdx.x] = threadIdx.x < ncol ? h[threadIdx.x] : 0.0;
  __syncthreads();
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kNT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kNT) {
    double v[NC];
    double wi = w[i];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      v[c] = c < ncol ? __ldcs(V + c * ldv + i) : 0.0;
      wi -= v[c] * sh[c];
    }
    w[i] = wi;
    const double wo = (i >= off && i < off + len) ? wi : 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = fma(v[c], wo, acc[c]);
  }
  finish_partials<NC>(acc, ncol, partial, counter, h2);
}

// w -= V h2 over [0,n); nrm2 = w.w over the owned range
template <int NC>
__global__ void __launch_bounds__(kNT) k_cgs_update_norm(const double* __restrict__ V, int64_t ldv, int ncol,
                                                         double* __restrict__ w, const double* __restrict__ h2,
                                                         int64_t n, int64_t off, int64_t len,
                                                         double* __restrict__ nrm2, double* partial,
                                                         unsigned* counter) {
  __shared__ double sh[NC];
  if (threadIdx.x < NC) sh[threadIdx.x] = threadIdx.x < ncol ? h2[threadIdx.x] : 0.0;
  __syncthreads();
  double acc[1] = {0.0};
  for (int64_t i = int64_t(blockIdx.x) * kNT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kNT) {
    double wi = w[i];
    // all column loads in flight together: the values are kept live to the end through a
    // running sum the kernel tests but never uses (w is finite), so ptxas hoists every load
    // (with a branch per column it kept two in flight and the pass ran at half the rate)
    double v[NC], keep = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) v[c] = c < ncol ? __ldcs(V + c * ldv + i) : 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) wi -= v[c] * sh[c];
#pragma unroll
    for (int c = 0; c < NC; ++c) keep += v[c];
    if (keep != keep && wi == 0.0) wi = keep;  // NaN input only, where wi is NaN anyway
    w[i] = wi;
    if (i >= off && i < off + len) acc[0] = fma(wi, wi, acc[0]);
  }
  finish_partials<1>(acc, 1, partial, counter, nrm2);
}

// y = V c, or y += V c (accumulate; the sum V c is formed first, then added: x + (V y) rounding)
template <int NC>
__global__ void __launch_bounds__(kNT) k_gemv_n(const double* __restrict__ V, int64_t ldv, int ncol, const Coef cf,
                                                double* __restrict__ y, int64_t n, bool accumulate) {
  for (int64_t i = int64_t(blockIdx.x) * kNT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kNT) {
    double v[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) v[c] = c < ncol ? V[c * ldv + i] : 0.0;
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c < ncol) s += v[c] * cf.c[c];
    y[i] = accumulate ? y[i] + s : s;
  }
}

int blocks_for(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>(kMaxDotBlocks, (n + kNT - 1) / kNT))); }

void check_ncol(int ncol) {
  if (ncol < 1 || ncol > kMaxCol) invalid("krylov: basis width must be in [1,32], got " + std::to_string(ncol));
}

// smallest instantiated bucket >= ncol
#define SB_NC_DISPATCH(ncol, CALL) \
  do {                             \
    if ((ncol) <= 4) {             \
      CALL(4);                     \
    } else if ((ncol) <= 8) {      \
      CALL(8);                     \
    } else if ((ncol) <= 12) {     \
      CALL(12);                    \
    } else if ((ncol) <= 16) {     \
      CALL(16);                    \
    } else if ((ncol) <= 24) {     \
      CALL(24);                    \
    } else {                       \
      CALL(32);                    \
    }                              \
  } while (0)

}  // namespace

int64_t launch_gemv_t(const double* V, int64_t ldv, int ncol, const double* w, int64_t off, int64_t len,
                      double* d_h, const DotScratch& ws, cudaStream_t s) {
  if (ncol > kMaxCol) {  // wide bases (restart > 31): 32-column chunks, one launch each
    int64_t k = 0;
    for (int c0 = 0; c0 < ncol; c0 += kMaxCol)
      k += launch_gemv_t(V + c0 * ldv, ldv, std::min(kMaxCol, ncol - c0), w, off, len, d_h + c0, ws, s);
    return k;
  }
  check_ncol(ncol);
#define L_(NC) k_gemv_t<NC><<<blocks_for(len), kNT, 0, s>>>(V, ldv, ncol, w, off, len, d_h, ws.partial, ws.counter)
  SB_NC_DISPATCH(ncol, L_);
#undef L_
  SB_LAUNCH_CHECK();
  return 1;
}

int64_t launch_cgs_update_dot(const double* V, int64_t ldv, int ncol, double* w, const double* d_h, int64_t n,
                              int64_t off, int64_t len, double* d_h2, const DotScratch& ws, cudaStream_t s) {
  check_ncol(ncol);
#define L_(NC) \
  k_cgs_update_dot<NC><<<blocks_for(n), kNT, 0, s>>>(V, ldv, ncol, w, d_h, n, off, len, d_h2, ws.partial, ws.counter)
  SB_NC_DISPATCH(ncol, L_);
#undef L_
  SB_LAUNCH_CHECK();
  return 1;
}

int64_t launch_cgs_update_norm(const double* V, int64_t ldv, int ncol, double* w, const double* d_h2, int64_t n,
                               int64_t off, int64_t len, double* d_nrm2, const DotScratch& ws, cudaStream_t s) {
  check_ncol(ncol);
#define L_(NC)                                                                                                    \
  k_cgs_update_norm<NC><<<blocks_for(n), kNT, 0, s>>>(V, ldv, ncol, w, d_h2, n, off, len, d_nrm2, ws.partial, \
                                                      ws.counter)
  SB_NC_DISPATCH(ncol, L_);
#undef L_
  SB_LAUNCH_CHECK();
  return 1;
}

int64_t launch_gemv_n(const double* V, int64_t ldv, int ncol, const double* c_host, double* y, int64_t n,
                      cudaStream_t s, bool accumulate) {
  if (ncol > kMaxCol) {  // wide bases: 32-column chunks, the later ones accumulate
    int64_t k = 0;
    for (int c0 = 0; c0 < ncol; c0 += kMaxCol)
      k += launch_gemv_n(V + c0 * ldv, ldv, std::min(kMaxCol, ncol - c0), c_host + c0, y, n, s,
                         accumulate || c0 > 0);
    return k;
  }
  check_ncol(ncol);
  Coef cf;
  for (int c = 0; c < kMaxCol; ++c) cf.c[c] = c < ncol ? c_host[c] : 0.0;
#define L_(NC) k_gemv_n<NC><<<blocks_for(n), kNT, 0, s>>>(V, ldv, ncol, cf, y, n, accumulate)
  SB_NC_DISPATCH(ncol, L_);
#undef L_
  SB_LAUNCH_CHECK();
  return 1;
}

}  // namespace sb
