// p-multigrid kernels for sm_100a: separable GLL transfers (P and its exact transpose),
// the coarse-grid solves (dense inverse GEMV, aggregation-AMG V-cycle pieces), free-dof maps.
//
// Transfers (pmg.cpp is missing in the reference): on the structured lattice the
// assembled element-wise interpolation is the separable operator P = P_z (x) P_y (x) P_x whose
// 1-D factor maps the coarse GLL lattice of one axis to the fine one with the element matrix
// J = lagrange_interpolation_matrix (gll.cpp:93-118). It is applied as three 1-D passes; the
// restriction runs the exact transpose passes (each coarse node sums its 1-D support once, so
// shared fine nodes are not double counted). Masks are applied on the input of the first pass
// and the output of the last.
#include <algorithm>

#include "device.cuh"
#include "kernels_mg.hpp"

namespace sb {

namespace {

int grid_for(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148LL * 32))); }

__device__ __forceinline__ bool on_boundary(int64_t x, int64_t y, int64_t z, const Grid3& g) {
  return x == 0 || x == g.N[0] - 1 || y == 0 || y == g.N[1] - 1 || z == 0 || z == g.N[2] - 1;
}

// One 1-D pass along AXIS. in/out are (x,y,z) arrays, x fastest, with local z offsets.
// PROLONG: out[X] = sum_a J(i(X), a) in[e(X) qc + a]
// RESTRICT: out[I] = sum over the 1-D support of coarse node I of J(i, a) in[X] (each X once)
// The pass axis is a template parameter and the output coordinates come from 32-bit divisions
// (the launcher checks the extents), so the index arithmetic stays off the critical path.
// QF/QC > 0: the orders are compile-time constants (the (7,3,1) schedule), so the 1-D support
// loops unroll and the element divisions become multiplications; 0: runtime orders.
template <bool PROLONG, int AXIS, int QF, int QC>
__global__ void __launch_bounds__(256) k_pass(const double* __restrict__ in, const Grid3 gin, double* __restrict__ out,
                                              const Grid3 gout, const Jmat J, const int qf_rt, const int qc_rt,
                                              const int E_axis, const int mask_in, const Grid3 gmask_in,
                                              const int mask_out, const Grid3 gmask_out, const int zb, const int nz,
                                              const int add_out, const double* __restrict__ sub_from) {
  const int qf = QF > 0 ? QF : qf_rt, qc = QC > 0 ? QC : qc_rt;
  const unsigned nx = unsigned(gout.N[0]), ny = unsigned(gout.N[1]);
  const unsigned total = nx * ny * unsigned(nz);
  const int jn = qc + 1;  // J is (qf+1) x (qc+1), row-major
  const int64_t sin = AXIS == 0 ? 1 : (AXIS == 1 ? gin.nxl : gin.nxl * gin.nyl);
  const int64_t nax_in = gmask_in.N[AXIS];
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const unsigned row = t / nx;
    const int c[3] = {int(t - row * nx), int(row % ny), zb + int(row / ny)};
    if (mask_out && gmask_out.dirichlet && on_boundary(c[0], c[1], c[2], gmask_out)) {
      if (!add_out) out[gout.idx(c[0], c[1], c[2])] = 0.0;  // (add: out += 0)
      continue;
    }
    // input row through this point along AXIS; the other two coordinates fix the mask test
    int c0[3] = {c[0], c[1], c[2]};
    c0[AXIS] = 0;
    const int64_t row_off = gin.idx(c0[0], c0[1], c0[2]);
    const double* row_in = in + row_off;
    const double* row_sub = sub_from ? sub_from + row_off : nullptr;
    bool other_bnd = false;
    if (mask_in && gmask_in.dirichlet) {
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (d != AXIS) other_bnd = other_bnd || c[d] == 0 || c[d] == gmask_in.N[d] - 1;
    }
    const bool min_ = mask_in && gmask_in.dirichlet;
    // branch-free: both loads always issue (coord is inside the lattice) and the mask selects, so
    // the compiler can put the whole 1-D support's loads in flight together
    const double* row_s = row_sub ? row_sub : row_in;
    const bool has_sub = row_sub != nullptr;
    auto fetch = [&](int coord) -> double {
      const double a = __ldg(row_in + coord * sin), b = __ldg(row_s + coord * sin);
      // sub_from: the input is (sub_from - in), e.g. the residual b - A x fused into Pᵀ
      const double v = has_sub ? b - a : a;
      return (min_ && (other_bnd || coord == 0 || coord == nax_in - 1)) ? 0.0 : v;
    };
    // every weight is applied, zero or not (w = 0 adds exactly +0): a branch on w would keep the
    // compiler from issuing the support loads together, and the pass would be load-latency bound
    const int X = c[AXIS];
    double acc = 0.0;
    if (PROLONG) {
      int e = X / qf;
      int i = X - e * qf;
      if (e == E_axis) {
        e -= 1;
        i = qf;
      }
#pragma unroll
      for (int a = 0; a < (QC > 0 ? QC + 1 : 16); ++a) {
        if (QC == 0 && a >= jn) break;
        const double w = J.v[i * jn + a];
        acc += w * fetch(e * qc + a);
      }
    } else {
      const int I = X;
      int e = I / qc;
      const int a = I - e * qc;
      if (a == 0 && e > 0) {  // shared coarse node: left element (a' = qc), then right element
        // (on a slab, an element of the other rank contributes through the interface sum; the
        // shared fine node X = e qf is counted with the left element only)
        if (e - 1 >= J.e_lo)
#pragma unroll
          for (int i = 0; i < (QF > 0 ? QF + 1 : 16); ++i) {
            if (QF == 0 && i > qf) break;
            const double w = J.v[i * jn + qc];
            acc += w * fetch((e - 1) * qf + i);
          }
        if (e < E_axis && e < J.e_hi)
#pragma unroll
          for (int i = 1; i < (QF > 0 ? QF + 1 : 16); ++i) {
            if (QF == 0 && i > qf) break;
            const double w = J.v[i * jn + 0];
            acc += w * fetch(e * qf + i);
          }
      } else {
        if (e == E_axis) e -= 1;  // last coarse node belongs to the last element
        const int aa = I - e * qc;
#pragma unroll
        for (int i = 0; i < (QF > 0 ? QF + 1 : 16); ++i) {
          if (QF == 0 && i > qf) break;
          const double w = J.v[i * jn + aa];
          acc += w * fetch(e * qf + i);
        }
      }
    }
    double* o = out + gout.idx(c[0], c[1], c[2]);
    *o = add_out ? *o + acc : acc;  // add: the coarse correction x += P e fused into the last pass
  }
}

}  // namespace

int64_t launch_transfer_pass(bool prolong, const double* in, const Grid3& gin, double* out, const Grid3& gout,
                             int axis, const Jmat& J, int qf, int qc, int E_axis, bool mask_in, const Grid3& gmi,
                             bool mask_out, const Grid3& gmo, int64_t zb, int64_t nz, cudaStream_t s, bool add_out,
                             const double* sub_from) {
  const int64_t total = gout.N[0] * gout.N[1] * nz;
  if (total <= 0) return 0;
  if (total >= (int64_t(1) << 32) || gmi.N[2] >= (int64_t(1) << 31) || zb >= (int64_t(1) << 31))
    invalid("transfer pass: lattice too large for 32-bit pass indexing");
  if (axis < 0 || axis > 2) invalid("transfer pass: axis must be 0, 1 or 2");
#define L3_(PR, AX, QF, QC)                                                                                       \
  k_pass<PR, AX, QF, QC><<<grid_for(total), 256, 0, s>>>(in, gin, out, gout, J, qf, qc, E_axis, mask_in, gmi, mask_out, \
                                                          gmo, int(zb), int(nz), int(add_out), sub_from)
#define L_(PR, AX)                                     \
  do {                                                 \
    if (qf == 7 && qc == 3) L3_(PR, AX, 7, 3);         \
    else if (qf == 3 && qc == 1) L3_(PR, AX, 3, 1);    \
    else L3_(PR, AX, 0, 0);                            \
  } while (0)
  if (prolong) {
    if (axis == 0) L_(true, 0); else if (axis == 1) L_(true, 1); else L_(true, 2);
  } else {
    if (axis == 0) L_(false, 0); else if (axis == 1) L_(false, 1); else L_(false, 2);
  }
#undef L_
#undef L3_
  SB_LAUNCH_CHECK();
  return 1;
}

// ---------------------------------------------------------------- free-dof maps (Dirichlet p=1)
// free index f = (x-1) + (Nx-2)((y-1) + (Ny-2)(z-1)); lattice vector uses the space layout.
// Free dofs: the lattice interior (Dirichlet: the boundary is masked) or the whole lattice (Neumann).
int64_t launch_gather_free(const Slab& sl, const double* full, double* freev, cudaStream_t s) {
  const int64_t mb = sl.dirichlet ? 1 : 0;
  const int64_t fx = sl.Nx - 2 * mb, fy = sl.Ny - 2 * mb, fz = sl.Nz - 2 * mb;
  const Slab g = sl;
  auto body = [=] __device__(int64_t f) {
    const int64_t x = mb + f % fx, y = mb + (f / fx) % fy, z = mb + f / (fx * fy);
    freev[f] = full[g.lidx(x, y, z)];
  };
  const int64_t n = fx * fy * fz;
  if (n <= 0) return 0;
  k_foreach_mg<<<grid_for(n), 256, 0, s>>>(n, body);
  SB_LAUNCH_CHECK();
  return 1;
}

int64_t launch_scatter_free(const Slab& sl, const double* freev, double* full, cudaStream_t s) {
  const int64_t mb = sl.dirichlet ? 1 : 0;
  const int64_t fx = sl.Nx - 2 * mb, fy = sl.Ny - 2 * mb;
  const Slab g = sl;
  const int64_t n = g.n_local();
  auto body = [=] __device__(int64_t t) {
    const int64_t x = t % g.Nx, y = (t / g.Nx) % g.Ny, z = g.zlo + t / (g.Nx * g.Ny);
    full[t] = g.masked(x, y, z) ? 0.0 : freev[(x - mb) + fx * ((y - mb) + fy * (z - mb))];
  };
  k_foreach_mg<<<grid_for(n), 256, 0, s>>>(n, body);
  SB_LAUNCH_CHECK();
  return 1;
}

// ---------------------------------------------------------------- dense GEMV (coarse inverse)
// y = M x, M n x n column-major symmetric: row i = column i -> coalesced by reading columns.
__global__ void __launch_bounds__(256) k_symv(const double* __restrict__ M, int64_t n, const double* __restrict__ x,
                                             double* __restrict__ y) {
  // one warp per output row i: y_i = sum_j M(j, i) x_j (column i is contiguous)
  const int lane = threadIdx.x & 31;
  for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; i < n;
       i += int64_t(gridDim.x) * blockDim.x / 32) {
    const double* col = M + i * n;
    double acc = 0.0;
    for (int64_t j = lane; j < n; j += 32) acc = fma(col[j], x[j], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[i] = acc;
  }
}

int64_t launch_symv(const double* M, int64_t n, const double* x, double* y, cudaStream_t s) {
  if (n <= 0) return 0;
  const int blocks = int(std::min<int64_t>((n * 32 + 255) / 256, 148LL * 16));
  k_symv<<<blocks, 256, 0, s>>>(M, n, x, y);
  SB_LAUNCH_CHECK();
  return 1;
}

// ---------------------------------------------------------------- AMG pieces (amg.cpp:131-165)
// z = omega D^-1 r (first relaxation from a zero guess)
int64_t launch_amg_jacobi0(const double* inv_diag, double omega, const double* r, double* z, int64_t n,
                           cudaStream_t s) {
  auto body = [=] __device__(int64_t i) { z[i] = 0.0 + omega * inv_diag[i] * (r[i] - 0.0); };
  if (n <= 0) return 0;
  k_foreach_mg<<<grid_for(n), 256, 0, s>>>(n, body);
  SB_LAUNCH_CHECK();
  return 1;
}

// zout = z + omega D^-1 (r - A z)   (one damped-Jacobi sweep, amg.cpp:131-138)
__global__ void k_amg_relax(const int64_t* __restrict__ ptr, const int* __restrict__ idx, const double* __restrict__ val,
                            const double* __restrict__ inv_diag, double omega, const double* __restrict__ r,
                            const double* __restrict__ z, double* __restrict__ zout, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double az = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) az += val[k] * z[idx[k]];
    zout[i] = z[i] + omega * inv_diag[i] * (r[i] - az);
  }
}

int64_t launch_amg_relax(const CsrDev& A, const double* inv_diag, double omega, const double* r, const double* z,
                         double* zout, cudaStream_t s) {
  if (A.n <= 0) return 0;
  k_amg_relax<<<grid_for(A.n), 256, 0, s>>>(A.ptr, A.idx, A.val, inv_diag, omega, r, z, zout, A.n);
  SB_LAUNCH_CHECK();
  return 1;
}

// rc[I] = sum_{i in aggregate I, ascending} (r - A z)_i   (res then P^T res, amg.cpp:153-154)
__global__ void k_amg_restrict(const int64_t* __restrict__ ptr, const int* __restrict__ idx,
                               const double* __restrict__ val, const int64_t* __restrict__ aptr,
                               const int* __restrict__ amem, const double* __restrict__ r,
                               const double* __restrict__ z, double* __restrict__ rc, int64_t nc) {
  for (int64_t I = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; I < nc; I += int64_t(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int64_t m = aptr[I]; m < aptr[I + 1]; ++m) {
      const int i = amem[m];
      double az = 0.0;
      for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) az += val[k] * z[idx[k]];
      acc += r[i] - az;
    }
    rc[I] = acc;
  }
}

int64_t launch_amg_restrict(const CsrDev& A, const int64_t* aptr, const int* amem, int64_t nc, const double* r,
                            const double* z, double* rc, cudaStream_t s) {
  if (nc <= 0) return 0;
  k_amg_restrict<<<grid_for(nc), 256, 0, s>>>(A.ptr, A.idx, A.val, aptr, amem, r, z, rc, nc);
  SB_LAUNCH_CHECK();
  return 1;
}

// res = r - A z (row parallel), then rc[I] = sum of res over aggregate I's members, ascending
__global__ void k_amg_residual(const int64_t* __restrict__ ptr, const int* __restrict__ idx,
                               const double* __restrict__ val, const double* __restrict__ r,
                               const double* __restrict__ z, double* __restrict__ res, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double az = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) az += val[k] * z[idx[k]];
    res[i] = r[i] - az;
  }
}
__global__ void k_amg_aggsum(const int64_t* __restrict__ aptr, const int* __restrict__ amem,
                             const double* __restrict__ res, double* __restrict__ rc, int64_t nc) {
  for (int64_t I = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; I < nc; I += int64_t(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int64_t m = aptr[I]; m < aptr[I + 1]; ++m) acc += res[amem[m]];
    rc[I] = acc;
  }
}

int64_t launch_amg_restrict_split(const CsrDev& A, const int64_t* aptr, const int* amem, int64_t nc, const double* r,
                                  const double* z, double* res, double* rc, cudaStream_t s) {
  if (A.n <= 0) return 0;
  k_amg_residual<<<grid_for(A.n), 256, 0, s>>>(A.ptr, A.idx, A.val, r, z, res, A.n);
  k_amg_aggsum<<<grid_for(nc), 128, 0, s>>>(aptr, amem, res, rc, nc);
  SB_LAUNCH_CHECK();
  return 2;
}

// z += P zc   (amg.cpp:156)
int64_t launch_amg_prolong(const int* agg, const double* zc, double* z, int64_t n, cudaStream_t s) {
  auto body = [=] __device__(int64_t i) { z[i] += zc[agg[i]]; };
  if (n <= 0) return 0;
  k_foreach_mg<<<grid_for(n), 256, 0, s>>>(n, body);
  SB_LAUNCH_CHECK();
  return 1;
}

}  // namespace sb
