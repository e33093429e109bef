// Launchers of the p-multigrid kernels (k_mg.cu).
#pragma once

#include <cuda_runtime.h>

#include "common.hpp"

namespace sb {

// A 3-D lattice array (x fastest) holding global planes [zoff, zoff + N[2]_local).
struct Grid3 {
  int64_t N[3];    // global lattice extent per axis (for the boundary mask)
  int64_t nxl, nyl;  // local storage extents in x, y (== N[0], N[1])
  int64_t zoff;    // global z of local plane 0
  int dirichlet;
  __host__ __device__ int64_t idx(int64_t x, int64_t y, int64_t z) const { return x + nxl * (y + nyl * (z - zoff)); }
};

struct Jmat {  // (qf+1) x (qc+1) row-major, qf <= 15
  double v[16 * 16] = {};
  int e_lo = 0, e_hi = 1 << 30;  // elements along the pass axis present on this rank (restrict)
};

struct CsrDev {
  int64_t n = 0;
  const int64_t* ptr = nullptr;
  const int* idx = nullptr;
  const double* val = nullptr;
};

#ifdef __CUDACC__
template <class F>
__global__ void k_foreach_mg(int64_t n, F f) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) f(t);
}
#endif

int64_t launch_transfer_pass(bool prolong, const double* in, const Grid3& gin, double* out, const Grid3& gout,
                             int axis, const Jmat& J, int qf, int qc, int E_axis, bool mask_in, const Grid3& gmi,
                             bool mask_out, const Grid3& gmo, int64_t zb, int64_t nz, cudaStream_t s,
                             bool add_out = false,  // add_out: out += pass result
                             const double* sub_from = nullptr);  // input is (sub_from - in)
int64_t launch_gather_free(const Slab& sl, const double* full, double* freev, cudaStream_t s);
int64_t launch_scatter_free(const Slab& sl, const double* freev, double* full, cudaStream_t s);
int64_t launch_symv(const double* M, int64_t n, const double* x, double* y, cudaStream_t s);
int64_t launch_amg_jacobi0(const double* inv_diag, double omega, const double* r, double* z, int64_t n, cudaStream_t s);
int64_t launch_amg_relax(const CsrDev& A, const double* inv_diag, double omega, const double* r, const double* z,
                         double* zout, cudaStream_t s);
int64_t launch_amg_restrict(const CsrDev& A, const int64_t* aptr, const int* amem, int64_t nc, const double* r,
                            const double* z, double* rc, cudaStream_t s);
int64_t launch_amg_restrict_split(const CsrDev& A, const int64_t* aptr, const int* amem, int64_t nc, const double* r,
                                  const double* z, double* res, double* rc, cudaStream_t s);
int64_t launch_amg_prolong(const int* agg, const double* zc, double* z, int64_t n, cudaStream_t s);

}  // namespace sb
