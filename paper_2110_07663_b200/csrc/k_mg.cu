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

#ifndef SEMLAB_PASS_YCOL
#define SEMLAB_PASS_YCOL 1  // y passes of the (7,3) level by element columns (k_pass_ycol)
#endif

// The 1-D passes. PROLONG: out[X] = sum_a J(i(X), a) in[e(X) qc + a]; RESTRICT: out[I] = sum over
// the 1-D support of coarse node I of J(i, a) in[X] (each X once: a coarse node shared by two
// elements sums the left element, then the right one). Input masks zero the boundary sites of the
// input lattice, output masks the boundary sites of the output; sub_from makes the input
// (sub_from - in) (the residual b - A x fused into the first restriction pass); add_out adds the
// result to out (x += P e fused into the last prolongation pass). Every weight is applied, zero or
// not (w = 0 adds exactly +0), so the support's loads issue together. QF/QC > 0 are the
// compile-time orders of the (7,3,1) schedule; 0: runtime orders.

// y / z passes: one thread per output site, x along the threads, (y, z) from the block indices —
// no divisions, and the row of J a block uses is uniform (a broadcast from the parameter bank).
template <bool PROLONG, int AXIS, int QF, int QC, bool SUB>
__global__ void __launch_bounds__(256) k_pass(const double* __restrict__ in, const Grid3 gin, double* __restrict__ out,
                                              const Grid3 gout, const Jmat J, const int qf_rt, const int qc_rt,
                                              const int E_axis, const int mask_in, const Grid3 gmask_in,
                                              const int mask_out, const Grid3 gmask_out, const int zb,
                                              const int add_out, const double* __restrict__ sub_from) {
  static_assert(AXIS == 1 || AXIS == 2, "k_pass: y or z");
  const int qf = QF > 0 ? QF : qf_rt, qc = QC > 0 ? QC : qc_rt;
  const int jn = qc + 1;
  const int x = int(blockIdx.x * blockDim.x + threadIdx.x);
  if (x >= gout.N[0]) return;
  const int y = int(blockIdx.y), z = zb + int(blockIdx.z);
  double* o = out + gout.idx(x, y, z);
  if (mask_out && gmask_out.dirichlet &&
      (x == 0 || x == gmask_out.N[0] - 1 || y == 0 || y == gmask_out.N[1] - 1 || z == 0 || z == gmask_out.N[2] - 1)) {
    if (!add_out) *o = 0.0;
    return;
  }
  const bool min_ = mask_in && gmask_in.dirichlet;
  const int oth = AXIS == 1 ? z : y;  // the coordinate that is neither x nor the pass axis
  const bool other_bnd = min_ && (x == 0 || x == gmask_in.N[0] - 1 || oth == 0 || oth == gmask_in.N[AXIS == 1 ? 2 : 1] - 1);
  const int nax_in = int(gmask_in.N[AXIS]);
  const int64_t sin = AXIS == 1 ? gin.nxl : gin.nxl * gin.nyl;
  const int64_t row_off = AXIS == 1 ? gin.idx(x, 0, z) : gin.idx(x, y, 0);  // + coord sin: global coord
  const double* row_in = in + row_off;
  const double* row_sub = SUB ? sub_from + row_off : nullptr;
  auto fetch = [&](int coord) -> double {
    const double a = __ldg(row_in + coord * sin);
    double v = a;
    if constexpr (SUB) v = __ldg(row_sub + coord * sin) - a;
    return (min_ && (other_bnd || coord == 0 || coord == nax_in - 1)) ? 0.0 : v;
  };
  const int X = AXIS == 1 ? y : z;
  double acc = 0.0;
  if (PROLONG) {
    int e = X / qf;
    int i = X - e * qf;
    if (e == E_axis) {
      e -= 1;
      i = qf;
    }
    if (i == 0 || i == qf) {
      // a vertex site: its row of J is exactly the unit vector (lagrange_interpolation_matrix
      // sets it on coinciding nodes), so the one nonzero term is the whole sum, bitwise — and
      // a slab's top interface plane (e = ez1, i = 0) must not read past the slab's coarse planes
      const int a = i == 0 ? 0 : qc;
      acc += J.v[i * jn + a] * fetch(e * qc + a);
    } else {
#pragma unroll
      for (int a = 0; a < (QC > 0 ? QC + 1 : 16); ++a) {
        if (QC == 0 && a >= jn) break;
        acc += J.v[i * jn + a] * fetch(e * qc + a);
      }
    }
  } else {
    int e = X / qc;
    const int a = X - e * qc;
    if (a == 0 && e > 0) {  // shared coarse node: left element (a' = qc), then right element
      // (on a slab, an element of the other rank contributes through the interface sum; the
      // shared fine node X = e qf is counted with the left element only)
      if (e - 1 >= J.e_lo)
#pragma unroll
        for (int i = 0; i < (QF > 0 ? QF + 1 : 16); ++i) {
          if (QF == 0 && i > qf) break;
          acc += J.v[i * jn + qc] * fetch((e - 1) * qf + i);
        }
      if (e < E_axis && e < J.e_hi)
#pragma unroll
        for (int i = 1; i < (QF > 0 ? QF + 1 : 16); ++i) {
          if (QF == 0 && i > qf) break;
          acc += J.v[i * jn + 0] * fetch(e * qf + i);
        }
    } else {
      if (e == E_axis) e -= 1;  // last coarse node belongs to the last element
      const int aa = X - e * qc;
#pragma unroll
      for (int i = 0; i < (QF > 0 ? QF + 1 : 16); ++i) {
        if (QF == 0 && i > qf) break;
        acc += J.v[i * jn + aa] * fetch(e * qf + i);
      }
    }
  }
  *o = add_out ? *o + acc : acc;  // add: the coarse correction x += P e fused into the last pass
}

// The y pass for the compile-time orders: one thread per (x, element along y, z) forms all the
// sites of its element column from one set of loads — prolongation: the qf sites of the element
// from its qc+1 coarse values; restriction: the qc coarse nodes of the element from its qf+1 fine
// values and those of the left element (the shared node). Same arithmetic and order as k_pass.
template <bool PROLONG, int QF, int QC, bool SUB>
__global__ void __launch_bounds__(256) k_pass_ycol(const double* __restrict__ in, const Grid3 gin,
                                                   double* __restrict__ out, const Grid3 gout, const Jmat J,
                                                   const int E_axis, const int mask_in, const Grid3 gmask_in,
                                                   const int mask_out, const Grid3 gmask_out, const int zb,
                                                   const int add_out, const double* __restrict__ sub_from) {
  static_assert(QF > 0 && QC > 0, "k_pass_ycol: compile-time orders");
  constexpr int jn = QC + 1;
  const int x = int(blockIdx.x * blockDim.x + threadIdx.x);
  if (x >= gout.N[0]) return;
  const int e = int(blockIdx.y), z = zb + int(blockIdx.z);
  const bool min_ = mask_in && gmask_in.dirichlet;
  const bool other_bnd = min_ && (x == 0 || x == gmask_in.N[0] - 1 || z == 0 || z == gmask_in.N[2] - 1);
  const int nax_in = int(gmask_in.N[1]);
  const int64_t sin = gin.nxl;
  const int64_t row_off = gin.idx(x, 0, z);
  auto fetch = [&](int coord) -> double {
    const double a = __ldg(in + row_off + coord * sin);
    double v = a;
    if constexpr (SUB) v = __ldg(sub_from + row_off + coord * sin) - a;
    return (min_ && (other_bnd || coord == 0 || coord == nax_in - 1)) ? 0.0 : v;
  };
  const bool mout = mask_out && gmask_out.dirichlet;
  const bool out_bnd = mout && (x == 0 || x == gmask_out.N[0] - 1 || z == 0 || z == gmask_out.N[2] - 1);
  auto put = [&](int Y, double acc) {
    double* o = out + gout.idx(x, Y, z);
    if (mout && (out_bnd || Y == 0 || Y == gmask_out.N[1] - 1)) {
      if (!add_out) *o = 0.0;
      return;
    }
    *o = add_out ? *o + acc : acc;
  };
  if (PROLONG) {
    double f[QC + 1];
#pragma unroll
    for (int a = 0; a <= QC; ++a) f[a] = fetch(e * QC + a);
    const int ni = e == E_axis - 1 ? QF + 1 : QF;  // the last element also writes its far site
#pragma unroll
    for (int i = 0; i <= QF; ++i) {
      if (i >= ni) break;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a <= QC; ++a) acc += J.v[i * jn + a] * f[a];
      put(e * QF + i, acc);
    }
  } else {
    double f[QF + 1], fl[QF + 1];
#pragma unroll
    for (int i = 0; i <= QF; ++i) f[i] = fetch(e * QF + i);
    if (e > 0) {
#pragma unroll
      for (int i = 0; i <= QF; ++i) fl[i] = fetch((e - 1) * QF + i);
    }
    {  // node e qc
      double acc = 0.0;
      if (e > 0) {
        if (e - 1 >= J.e_lo)
#pragma unroll
          for (int i = 0; i <= QF; ++i) acc += J.v[i * jn + QC] * fl[i];
        if (e < J.e_hi)
#pragma unroll
          for (int i = 1; i <= QF; ++i) acc += J.v[i * jn + 0] * f[i];
      } else {
#pragma unroll
        for (int i = 0; i <= QF; ++i) acc += J.v[i * jn + 0] * f[i];
      }
      put(e * QC, acc);
    }
#pragma unroll
    for (int a = 1; a < QC; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i <= QF; ++i) acc += J.v[i * jn + a] * f[i];
      put(e * QC + a, acc);
    }
    if (e == E_axis - 1) {  // the last coarse node E qc: the last element's local qc
      double acc = 0.0;
      if (e >= J.e_lo)
#pragma unroll
        for (int i = 0; i <= QF; ++i) acc += J.v[i * jn + QC] * f[i];
      put(E_axis * QC, acc);
    }
  }
}

// The x pass: one block per (y, z) row, staged in shared memory. The input row is loaded
// coalesced (masked, sub_from subtracted); the outputs are formed with the threads ordered
// (local index, element) so a warp reads one row of J (a broadcast) and strided shared-memory
// sites; they go to a shared output row and then to HBM coalesced (mask, add). Along x the
// supports of neighbouring outputs overlap and the row of J differs per site, which made the
// one-thread-per-site form latency- and replay-bound.
template <bool PROLONG, int QF, int QC, bool SUB>
__global__ void __launch_bounds__(1024) k_pass_x(const double* __restrict__ in, const Grid3 gin,
                                                 double* __restrict__ out, const Grid3 gout, const Jmat J,
                                                 const int qf_rt, const int qc_rt, const int E_axis,
                                                 const int mask_in, const Grid3 gmask_in, const int mask_out,
                                                 const Grid3 gmask_out, const int zb, const int nz, const int add_out,
                                                 const double* __restrict__ sub_from) {
  constexpr int RB = 4;  // rows per block step: each thread has RB independent loads per array in flight
  extern __shared__ double sm[];
  const int qf = QF > 0 ? QF : qf_rt, qc = QC > 0 ? QC : qc_rt;
  const int jn = qc + 1;
  const int nin = int(gin.N[0]), nout = int(gout.N[0]), ny = int(gout.N[1]);
  double* srow = sm;             // RB input rows
  double* sout = sm + RB * nin;  // RB output rows
  const bool min_ = mask_in && gmask_in.dirichlet;
  const bool mout = mask_out && gmask_out.dirichlet;
  const int q_out = PROLONG ? qf : qc;  // sites per element on the output side
  // one input site and one output site per thread (blockDim >= nin, nout): the site maps are
  // computed once. Output t -> (l, e), l = t / E (uniform over most of a warp so the row of J is
  // a broadcast), site X = e q_out + l; the last site E q_out last.
  const int x = threadIdx.x;
  const bool has_in = x < nin, has_out = x < nout;
  const bool x_edge_in = x == 0 || x == gmask_in.N[0] - 1;
  int l = x / E_axis, e = x - l * E_axis;
  if (l == q_out) e = E_axis - 1;
  const int X = e * q_out + l;
  const bool x_edge_out = X == 0 || X == gmask_out.N[0] - 1;
  {
    // block (blockIdx.x, blockIdx.y) = rows y0 .. y0+RB-1 of plane z: no divisions, and the row
    // bases are a stride apart
    const int y0 = blockIdx.x * RB, z = zb + int(blockIdx.y);
    const int64_t gi0 = gin.idx(0, y0, z), go0 = gout.idx(0, y0, z);
    const bool zedge_in = z == 0 || z == gmask_in.N[2] - 1, zedge_out = z == 0 || z == gmask_out.N[2] - 1;
    double vin[RB], vsub[RB], vout[RB];
    int64_t gi[RB], go[RB];
    bool edge_in[RB], edge_out[RB];
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      const int y = min(y0 + rr, ny - 1);  // (a short last block repeats its last row; only nr are stored)
      gi[rr] = gi0 + int64_t(y - y0) * gin.nxl;
      go[rr] = go0 + int64_t(y - y0) * gout.nxl;
      edge_in[rr] = zedge_in || y == 0 || y == gmask_in.N[1] - 1;
      edge_out[rr] = zedge_out || y == 0 || y == gmask_out.N[1] - 1;
      if (has_in) {
        vin[rr] = __ldg(in + gi[rr] + x);
        if constexpr (SUB) vsub[rr] = __ldg(sub_from + gi[rr] + x);
      }
      if (add_out && has_out) vout[rr] = out[go[rr] + X];
    }
    if (has_in) {
#pragma unroll
      for (int rr = 0; rr < RB; ++rr) {
        double v = vin[rr];
        if constexpr (SUB) v = vsub[rr] - v;
        srow[rr * nin + x] = (min_ && (edge_in[rr] || x_edge_in)) ? 0.0 : v;
      }
    }
    __syncthreads();
    if (has_out) {
#pragma unroll
      for (int rr = 0; rr < RB; ++rr) {
        const double* si = srow + rr * nin;
        double acc = 0.0;
        if (PROLONG) {
#pragma unroll
          for (int a = 0; a < (QC > 0 ? QC + 1 : 16); ++a) {
            if (QC == 0 && a >= jn) break;
            acc += J.v[l * jn + a] * si[e * qc + a];
          }
        } else if (l == 0 && e > 0) {  // shared coarse node e qc: left element, then right element
          if (e - 1 >= J.e_lo)
#pragma unroll
            for (int i = 0; i < (QF > 0 ? QF + 1 : 16); ++i) {
              if (QF == 0 && i > qf) break;
              acc += J.v[i * jn + qc] * si[(e - 1) * qf + i];
            }
          if (e < J.e_hi)
#pragma unroll
            for (int i = 1; i < (QF > 0 ? QF + 1 : 16); ++i) {
              if (QF == 0 && i > qf) break;
              acc += J.v[i * jn + 0] * si[e * qf + i];
            }
        } else if (l == q_out) {  // the last coarse node E qc: the last element's local qc
          if (e >= J.e_lo)
#pragma unroll
            for (int i = 0; i < (QF > 0 ? QF + 1 : 16); ++i) {
              if (QF == 0 && i > qf) break;
              acc += J.v[i * jn + qc] * si[e * qf + i];
            }
        } else {
#pragma unroll
          for (int i = 0; i < (QF > 0 ? QF + 1 : 16); ++i) {
            if (QF == 0 && i > qf) break;
            acc += J.v[i * jn + l] * si[e * qf + i];
          }
        }
        const bool masked = mout && (edge_out[rr] || x_edge_out);
        double v = add_out ? vout[rr] + acc : acc;
        if (masked) v = add_out ? vout[rr] : 0.0;  // (add: out += 0)
        sout[rr * nout + X] = v;
      }
    }
    __syncthreads();
    if (x < nout) {
      const int nr = min(RB, ny - y0);
#pragma unroll
      for (int rr = 0; rr < RB; ++rr)
        if (rr < nr) out[go[rr] + x] = sout[rr * nout + x];
    }
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
  if (gout.N[1] > 65535 || nz > 65535) invalid("transfer pass: more than 65535 rows along y or z");
  if (axis == 0) {
    const int64_t wid = std::max(gin.N[0], gout.N[0]);
    const size_t smem = size_t(4) * size_t(gin.N[0] + gout.N[0]) * sizeof(double);
    if (wid > 1024 || smem > 48 * 1024) invalid("transfer pass: x rows longer than 1024 sites");
    if (gout.N[0] != (prolong ? int64_t(E_axis) * qf : int64_t(E_axis) * qc) + 1)
      invalid("transfer pass: x extent does not match the element count");
    const int block = int((wid + 31) / 32 * 32);
    const dim3 grid(unsigned((gout.N[1] + 3) / 4), unsigned(nz));  // RB = 4 rows per block
#define LX_(PR, QF, QC, SUB)                                                                                 \
  k_pass_x<PR, QF, QC, SUB><<<grid, block, smem, s>>>(in, gin, out, gout, J, qf, qc, E_axis, mask_in, gmi,   \
                                                      mask_out, gmo, int(zb), int(nz), int(add_out), sub_from)
#define LXS_(PR, QF, QC) \
  do {                   \
    if (sub_from) LX_(PR, QF, QC, true); else LX_(PR, QF, QC, false); \
  } while (0)
#define LXQ_(PR)                                      \
  do {                                                \
    if (qf == 7 && qc == 3) LXS_(PR, 7, 3);           \
    else if (qf == 3 && qc == 1) LXS_(PR, 3, 1);      \
    else LXS_(PR, 0, 0);                              \
  } while (0)
    if (prolong) LXQ_(true); else LXQ_(false);
#undef LXQ_
#undef LXS_
#undef LX_
  } else {
    const unsigned bx = unsigned(std::min<int64_t>(256, (gout.N[0] + 31) / 32 * 32));
    const dim3 grid(unsigned((gout.N[0] + bx - 1) / bx), unsigned(gout.N[1]), unsigned(nz));
#define LP_(PR, AX, QF, QC, SUB)                                                                            \
  k_pass<PR, AX, QF, QC, SUB><<<grid, bx, 0, s>>>(in, gin, out, gout, J, qf, qc, E_axis, mask_in, gmi,     \
                                                 mask_out, gmo, int(zb), int(add_out), sub_from)
#define LPS_(PR, AX, QF, QC) \
  do {                       \
    if (sub_from) LP_(PR, AX, QF, QC, true); else LP_(PR, AX, QF, QC, false); \
  } while (0)
#define LPQ_(PR, AX)                                  \
  do {                                                \
    if (qf == 7 && qc == 3) LPS_(PR, AX, 7, 3);       \
    else if (qf == 3 && qc == 1) LPS_(PR, AX, 3, 1);  \
    else LPS_(PR, AX, 0, 0);                          \
  } while (0)
    if (axis == 1 && qf == 7 && qc == 3 && SEMLAB_PASS_YCOL) {
      if (gout.N[1] != (prolong ? int64_t(E_axis) * qf : int64_t(E_axis) * qc) + 1)
        invalid("transfer pass: y extent does not match the element count");
      const dim3 gcol(grid.x, unsigned(E_axis), unsigned(nz));
#define LC_(PR, SUB)                                                                                        \
  k_pass_ycol<PR, 7, 3, SUB><<<gcol, bx, 0, s>>>(in, gin, out, gout, J, E_axis, mask_in, gmi, mask_out, gmo, \
                                                 int(zb), int(add_out), sub_from)
      if (prolong) LC_(true, false);
      else if (sub_from) LC_(false, true);
      else LC_(false, false);
#undef LC_
    } else if (prolong) {
      if (axis == 1) LPQ_(true, 1); else LPQ_(true, 2);
    } else {
      if (axis == 1) LPQ_(false, 1); else LPQ_(false, 2);
    }
#undef LPQ_
#undef LPS_
#undef LP_
  }
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
// (A z)_i summed over the row in ascending k (amg.cpp's order), with the row's column indices,
// values and z gathers issued 8 at a time instead of one dependent pair per step
__device__ __forceinline__ double csr_row_dot(const int64_t* __restrict__ ptr, const int* __restrict__ idx,
                                              const double* __restrict__ val, const double* __restrict__ z,
                                              int64_t i) {
  constexpr int C = 8;
  const int64_t k0 = ptr[i], k1 = ptr[i + 1];
  double az = 0.0;
  for (int64_t kb = k0; kb < k1; kb += C) {
    int col[C];
    double a[C], zv[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const bool ok = kb + c < k1;
      col[c] = ok ? __ldg(idx + kb + c) : 0;
      a[c] = ok ? __ldg(val + kb + c) : 0.0;
    }
#pragma unroll
    for (int c = 0; c < C; ++c) zv[c] = kb + c < k1 ? z[col[c]] : 0.0;
#pragma unroll
    for (int c = 0; c < C; ++c)
      if (kb + c < k1) az += a[c] * zv[c];
  }
  return az;
}

__global__ void k_amg_relax(const int64_t* __restrict__ ptr, const int* __restrict__ idx, const double* __restrict__ val,
                            const double* __restrict__ inv_diag, double omega, const double* __restrict__ r,
                            const double* __restrict__ z, double* __restrict__ zout, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double az = csr_row_dot(ptr, idx, val, z, i);
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
      acc += r[i] - csr_row_dot(ptr, idx, val, z, i);
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
    res[i] = r[i] - csr_row_dot(ptr, idx, val, z, i);
  }
}
__global__ void k_amg_aggsum(const int64_t* __restrict__ aptr, const int* __restrict__ amem,
                             const double* __restrict__ res, double* __restrict__ rc, int64_t nc) {
  for (int64_t I = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; I < nc; I += int64_t(gridDim.x) * blockDim.x) {
    // members in ascending order, their indices and values gathered 8 at a time
    constexpr int C = 8;
    const int64_t m0 = aptr[I], m1 = aptr[I + 1];
    double acc = 0.0;
    for (int64_t mb = m0; mb < m1; mb += C) {
      int mi[C];
      double v[C];
#pragma unroll
      for (int c = 0; c < C; ++c) mi[c] = mb + c < m1 ? __ldg(amem + mb + c) : 0;
#pragma unroll
      for (int c = 0; c < C; ++c) v[c] = mb + c < m1 ? res[mi[c]] : 0.0;
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (mb + c < m1) acc += v[c];
    }
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
