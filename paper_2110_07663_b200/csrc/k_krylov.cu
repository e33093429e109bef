// Krylov kernels for sm_100a: fused classical Gram-Schmidt passes over the column-major basis
// V (krylov.cpp:67-72, chebyshev.cpp:36-41), and the basis combination V*y (krylov.cpp:111).
// Every reduction is deterministic: per-block partials in a fixed shape, then the last block
// to finish sums the partials in block order.
#include <algorithm>

#include "device.cuh"
#include "kernels.hpp"

namespace sb {

namespace {

constexpr int kMaxCol = 32;
constexpr int kNT = 256;

struct Coef {
  double c[kMaxCol];
};

// Sum the per-block partial vectors (ncol each) in block order; last block writes out.
__device__ __forceinline__ void finish_partials(double (&acc)[kMaxCol], int ncol, double* partial, unsigned* counter,
                                                double* out) {
  __shared__ double sred[kMaxCol * (kNT / 32)];
  __shared__ bool last;
  block_sum<kMaxCol, kNT>(acc, sred);
  if (threadIdx.x == 0) {
    for (int c = 0; c < ncol; ++c) partial[blockIdx.x * kMaxCol + c] = acc[c];
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x < ncol) {
    __threadfence();
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) s += __ldcg(&partial[b * kMaxCol + threadIdx.x]);
    out[threadIdx.x] = s;
  }
  if (last && threadIdx.x == 0) *counter = 0u;
}

// h = V^T w over the owned range
__global__ void __launch_bounds__(kNT) k_gemv_t(const double* __restrict__ V, int64_t ldv, int ncol,
                                                const double* __restrict__ w, int64_t off, int64_t len,
                                                double* __restrict__ h, double* partial, unsigned* counter) {
  double acc[kMaxCol];
#pragma unroll
  for (int c = 0; c < kMaxCol; ++c) acc[c] = 0.0;
  for (int64_t t = int64_t(blockIdx.x) * kNT + threadIdx.x; t < len; t += int64_t(gridDim.x) * kNT) {
    const int64_t i = off + t;
    const double wi = w[i];
#pragma unroll
    for (int c = 0; c < kMaxCol; ++c)
      if (c < ncol) acc[c] = fma(V[c * ldv + i], wi, acc[c]);
  }
  finish_partials(acc, ncol, partial, counter, h);
}

// w -= V h over [0,n); h2 = V^T w over the owned range (one read of V for both)
__global__ void __launch_bounds__(kNT) k_cgs_update_dot(const double* __restrict__ V, int64_t ldv, int ncol,
                                                        double* __restrict__ w, const double* __restrict__ h,
                                                        int64_t n, int64_t off, int64_t len,
                                                        double* __restrict__ h2, double* partial,
                                                        unsigned* counter) {
  __shared__ double sh[kMaxCol];
  if (threadIdx.x < kMaxCol) sh[threadIdx.x] = threadIdx.x < ncol ? h[threadIdx.x] : 0.0;
  __syncthreads();
  double acc[kMaxCol];
#pragma unroll
  for (int c = 0; c < kMaxCol; ++c) acc[c] = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kNT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kNT) {
    double v[kMaxCol];
    double wi = w[i];
#pragma unroll
    for (int c = 0; c < kMaxCol; ++c)
      if (c < ncol) {
        v[c] = V[c * ldv + i];
        wi -= v[c] * sh[c];
      }
    w[i] = wi;
    if (i >= off && i < off + len) {
#pragma unroll
      for (int c = 0; c < kMaxCol; ++c)
        if (c < ncol) acc[c] = fma(v[c], wi, acc[c]);
    }
  }
  finish_partials(acc, ncol, partial, counter, h2);
}

// w -= V h2 over [0,n); nrm2 = w.w over the owned range
__global__ void __launch_bounds__(kNT) k_cgs_update_norm(const double* __restrict__ V, int64_t ldv, int ncol,
                                                         double* __restrict__ w, const double* __restrict__ h2,
                                                         int64_t n, int64_t off, int64_t len,
                                                         double* __restrict__ nrm2, double* partial,
                                                         unsigned* counter) {
  __shared__ double sh[kMaxCol];
  if (threadIdx.x < kMaxCol) sh[threadIdx.x] = threadIdx.x < ncol ? h2[threadIdx.x] : 0.0;
  __syncthreads();
  double acc[kMaxCol];
#pragma unroll
  for (int c = 0; c < kMaxCol; ++c) acc[c] = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kNT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kNT) {
    double wi = w[i];
#pragma unroll
    for (int c = 0; c < kMaxCol; ++c)
      if (c < ncol) wi -= V[c * ldv + i] * sh[c];
    w[i] = wi;
    if (i >= off && i < off + len) acc[0] = fma(wi, wi, acc[0]);
  }
  finish_partials(acc, 1, partial, counter, nrm2);
}

__global__ void __launch_bounds__(kNT) k_gemv_n(const double* __restrict__ V, int64_t ldv, int ncol, const Coef cf,
                                                double* __restrict__ y, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * kNT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kNT) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kMaxCol; ++c)
      if (c < ncol) s += V[c * ldv + i] * cf.c[c];
    y[i] = s;
  }
}

int blocks_for(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>(kMaxDotBlocks, (n + kNT - 1) / kNT))); }

void check_ncol(int ncol) {
  if (ncol < 1 || ncol > kMaxCol) invalid("krylov: basis width must be in [1,32], got " + std::to_string(ncol));
}

}  // namespace

int64_t launch_gemv_t(const double* V, int64_t ldv, int ncol, const double* w, int64_t off, int64_t len,
                      double* d_h, const DotScratch& ws, cudaStream_t s) {
  check_ncol(ncol);
  k_gemv_t<<<blocks_for(len), kNT, 0, s>>>(V, ldv, ncol, w, off, len, d_h, ws.partial, ws.counter);
  SB_LAUNCH_CHECK();
  return 1;
}

int64_t launch_cgs_update_dot(const double* V, int64_t ldv, int ncol, double* w, const double* d_h, int64_t n,
                              int64_t off, int64_t len, double* d_h2, const DotScratch& ws, cudaStream_t s) {
  check_ncol(ncol);
  k_cgs_update_dot<<<blocks_for(n), kNT, 0, s>>>(V, ldv, ncol, w, d_h, n, off, len, d_h2, ws.partial, ws.counter);
  SB_LAUNCH_CHECK();
  return 1;
}

int64_t launch_cgs_update_norm(const double* V, int64_t ldv, int ncol, double* w, const double* d_h2, int64_t n,
                               int64_t off, int64_t len, double* d_nrm2, const DotScratch& ws, cudaStream_t s) {
  check_ncol(ncol);
  k_cgs_update_norm<<<blocks_for(n), kNT, 0, s>>>(V, ldv, ncol, w, d_h2, n, off, len, d_nrm2, ws.partial,
                                                  ws.counter);
  SB_LAUNCH_CHECK();
  return 1;
}

int64_t launch_gemv_n(const double* V, int64_t ldv, int ncol, const double* c_host, double* y, int64_t n,
                      cudaStream_t s) {
  check_ncol(ncol);
  Coef cf;
  for (int c = 0; c < kMaxCol; ++c) cf.c[c] = c < ncol ? c_host[c] : 0.0;
  k_gemv_n<<<blocks_for(n), kNT, 0, s>>>(V, ldv, ncol, cf, y, n);
  SB_LAUNCH_CHECK();
  return 1;
}

}  // namespace sb
