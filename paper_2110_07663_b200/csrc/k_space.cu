// SemSpace kernels for sm_100a: geometric factors, the fused owner-ordered Ax, Q/Q^T/QQ^T,
// the assembled diagonal, and deterministic reductions.
//
// Ax design (replaces SemSpace::apply_A, sem_space.cpp:195-209, and the innermost
// local_stiffness_kernel, sem_space.cpp:127-175):
//   * global -> global in ONE kernel: the element reads u straight from the lattice vector
//     (Q is arithmetic, sem_space.hpp:44-49: no index arrays), the 6 geometric factors of the
//     element stream into shared memory with one cp.async.bulk (TMA engine) while u is loaded
//     and the three D-derivatives are formed, then G*(ur,us,ut) and the transposed contractions.
//   * Q^T without atomics and in the reference's summation order: every lattice node is owned
//     by the highest-id element containing it. A CTA takes a dynamic ticket (element group in
//     ascending id), deposits the values of the nodes it does not own, publishes a per-element
//     counter with st.release, waits (ld.acquire) for its <= 7 lower neighbours, and sums each
//     owned node over its contributors in ASCENDING element id — exactly the order of the
//     reference gather (sem_space.cpp:40-52, 110-119). Tickets are taken in order by running
//     CTAs and a CTA only waits on lower tickets, so the scheme cannot deadlock.
//   * the owner applies an epilogue (plain write, residual, or a whole Chebyshev-Jacobi
//     vector update) so the smoother needs no extra pass over the vectors.
#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include "device.cuh"
#include "host_math.hpp"
#include "kernels.hpp"

#ifndef SEMLAB_AX_BATCH_EPI
#define SEMLAB_AX_BATCH_EPI 1  // owner epilogue: issue all vector loads before the stores
#endif
#ifndef SEMLAB_AX_SPLIT_ND
#define SEMLAB_AX_SPLIT_ND 6  // orders p <= 5: element-local Ax + ordered gather (no counter waits)
#endif
#ifndef SEMLAB_AXP_MINB
#define SEMLAB_AXP_MINB 6  // resident CTAs per SM the persistent Ax is register-capped for
#endif

namespace sb {

namespace {

template <int ND>
DMat<ND> dmat(int q) {
  DMat<ND> m;
  const auto& g = gll(q);
  for (int t = 0; t < ND * ND; ++t) m.d[t] = g.diff[t];
  return m;
}

template <int ND>
struct W1 {
  double w[ND];
};

template <int ND>
constexpr int epb() {
  return ND * ND >= 64 ? 1 : (64 + ND * ND - 1) / (ND * ND);
}

int grid1d(int64_t n, int nt) { return int(std::min<int64_t>((n + nt - 1) / nt, 148LL * 64)); }

// ------------------------------------------------------------------------ epilogues
// Each epilogue splits into load (vector inputs at node g) and store (combine with (A u)[g]) so
// a thread can issue the loads of all its nodes before the first store.
struct EWrite {
  double* w;
  struct In {};
  __device__ In load(int64_t) const { return {}; }
  __device__ void store(int64_t g, const In&, double v) const { w[g] = v; }
  __device__ void operator()(int64_t g, double v) const { store(g, load(g), v); }
};
struct EResidual {
  double* w;
  const double* b;
  struct In {
    double b;
  };
  __device__ In load(int64_t g) const { return {b[g]}; }
  __device__ void store(int64_t g, const In& in, double v) const { w[g] = in.b - v; }
  __device__ void operator()(int64_t g, double v) const { store(g, load(g), v); }
};
struct EChebJacStep {  // chebyshev.cpp:86-92 with S = diag(A)^-1 fused at the owner
  double* x;
  double* r;
  double* d;
  const double* inv;
  double c1, c2;
  struct In {
    double d, x, r, inv;
  };
  __device__ In load(int64_t g) const { return {d[g], x[g], r[g], inv[g]}; }
  __device__ void store(int64_t g, const In& in, double v) const {
    x[g] = in.x + in.d;
    const double rg = in.r - in.inv * v;
    r[g] = rg;
    d[g] = c1 * in.d + c2 * rg;
  }
  __device__ void operator()(int64_t g, double v) const { store(g, load(g), v); }
};
struct EChebJacInit {  // chebyshev.cpp:80-84: r = S(b - A x); d = r / theta
  double* r;
  double* d;
  const double* b;
  const double* inv;
  double theta;
  struct In {
    double b, inv;
  };
  __device__ In load(int64_t g) const { return {b[g], inv[g]}; }
  __device__ void store(int64_t g, const In& in, double v) const {
    const double rg = in.inv * (in.b - v);
    r[g] = rg;
    d[g] = rg / theta;
  }
  __device__ void operator()(int64_t g, double v) const { store(g, load(g), v); }
};

// ------------------------------------------------------------------------ geometry
// G = w det(J) J^-1 J^-T packed (rr,rs,rt,ss,st,tt), mass weight w det(J): sem_space.cpp:58-97.
// Layout: SoA per element, geom[(e*6 + c)*nloc + node].
template <int ND>
__global__ void k_geom(const Slab sl, const DMat<ND> Dm, const W1<ND> w1, const double* __restrict__ X,
                       double* __restrict__ geom, double* __restrict__ massw,
                       unsigned long long* __restrict__ bad) {
  constexpr int NLOC = ND * ND * ND;
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= sl.elems() * NLOC) return;
  const int64_t el = idx / NLOC;
  const int node = int(idx % NLOC);
  const int i = node % ND, j = (node / ND) % ND, k = node / (ND * ND);
  const int q = ND - 1;
  const int ex = int(el % sl.Ex), ey = int((el / sl.Ex) % sl.Ey), ez = sl.ez0 + int(el / (int64_t(sl.Ex) * sl.Ey));
  const int64_t x0 = int64_t(ex) * q, y0 = int64_t(ey) * q, z0 = int64_t(ez) * q;
  double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
  for (int m = 0; m < ND; ++m) {
    const double* pr = X + 3 * sl.lidx(x0 + m, y0 + j, z0 + k);
    const double* ps = X + 3 * sl.lidx(x0 + i, y0 + m, z0 + k);
    const double* pt = X + 3 * sl.lidx(x0 + i, y0 + j, z0 + m);
    const double dr = Dm.d[i + ND * m], ds = Dm.d[j + ND * m], dt = Dm.d[k + ND * m];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      J[c][0] += dr * pr[c];
      J[c][1] += ds * ps[c];
      J[c][2] += dt * pt[c];
    }
  }
  const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  const double c10 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  const double c20 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  const double det = J[0][0] * c00 + J[0][1] * c10 + J[0][2] * c20;
  if (!(det > 0.0)) {
    atomicMin(bad, (unsigned long long)(el + int64_t(sl.ez0) * sl.Ex * sl.Ey));
    return;
  }
  const double id = 1.0 / det;
  double Ji[3][3];
  Ji[0][0] = c00 * id;
  Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
  Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
  Ji[1][0] = c10 * id;
  Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
  Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
  Ji[2][0] = c20 * id;
  Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
  Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
  const double wd = w1.w[i] * w1.w[j] * w1.w[k] * det;
  auto G = [&](int a, int b) { return wd * (Ji[a][0] * Ji[b][0] + Ji[a][1] * Ji[b][1] + Ji[a][2] * Ji[b][2]); };
  double* ge = geom + el * 6 * NLOC + node;
  ge[0 * NLOC] = G(0, 0);
  ge[1 * NLOC] = G(0, 1);
  ge[2 * NLOC] = G(0, 2);
  ge[3 * NLOC] = G(1, 1);
  ge[4 * NLOC] = G(1, 2);
  ge[5 * NLOC] = G(2, 2);
  massw[el * NLOC + node] = wd;
}

// ------------------------------------------------------------------------ Ax
#ifndef SEMLAB_AX_PERSISTENT
#define SEMLAB_AX_PERSISTENT 1  // build-time A/B: 0 = one CTA per element group (orders != 7)
#endif
constexpr bool ax_persistent() { return SEMLAB_AX_PERSISTENT != 0; }

template <int ND>
constexpr int ax_min_blocks() {  // occupancy target: caps registers so ~20 warps/SM stay resident
  return ND >= 8 ? 10 : 16;
}

// IO: 0 global -> global with the owner-ordered Q^T; 1 local -> local (E-vectors); 2 global in,
// element-local out (the split path: k_gather_epi then sums in the reference order)
// GT: the geometric-factor storage type (double; float = the FP32 smoother's FP32-rounded factors,
// FP64 arithmetic)
template <int ND, int EPB, int IO, class EpiT, class GT = double>
__global__ void __launch_bounds__(EPB* ND* ND, ax_min_blocks<ND>())
    k_ax(const Slab sl, const DMat<ND> Dm, const double* __restrict__ u, const GT* __restrict__ geom,
         double* __restrict__ dep, unsigned* __restrict__ flags, unsigned* __restrict__ ticket, int ngroups,
         double* __restrict__ out_local, const EpiT epi) {
  constexpr int ND2 = ND * ND, NLOC = ND2 * ND, NT = EPB * ND2;
  constexpr int q = ND - 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* s_a = reinterpret_cast<double*>(smem_raw);
  double* s_b = s_a + EPB * NLOC;
  double* s_D = s_b + EPB * NLOC;
  __shared__ int s_grp;
  __shared__ unsigned s_epoch;
  const int tid = threadIdx.x;

  if (tid == 0) {
    int t;
    if (IO != 0) {
      t = blockIdx.x;
    } else {
      t = int(atomicAdd(ticket, 1u));
      if (t == ngroups - 1) atomicExch(ticket, 0u);  // every ticket of this launch is taken
    }
    s_grp = t;
  }
  // D to shared memory with compile-time indices (a per-thread index into the kernel parameter
  // would make the compiler copy the whole matrix to a local-memory stack frame in every thread)
  if (tid == 0) {
#pragma unroll
    for (int t = 0; t < ND2; ++t) s_D[t] = Dm.d[t];
  }
  __syncthreads();

  const int64_t nE = sl.elems();
  const int64_t e0 = int64_t(s_grp) * EPB;
  const int ne = int(nE - e0 < EPB ? nE - e0 : EPB);
  {  // stream the group's geometry (contiguous, 48 B/node) into L2 while u is loaded and
     // differentiated; phase 2 then reads it at L2 latency without holding shared memory
    const char* gbase = reinterpret_cast<const char*>(geom + e0 * 6 * NLOC);
    const int lines = (ne * 6 * NLOC * int(sizeof(GT)) + 127) / 128;
    for (int l = tid; l < lines; l += NT) asm volatile("prefetch.global.L2 [%0];" ::"l"(gbase + size_t(l) * 128));
  }
  if (tid == 0 && IO == 0) s_epoch = *reinterpret_cast<volatile unsigned*>(&flags[e0]);

  const int le = tid / ND2, ij = tid % ND2, i = ij % ND, j = ij / ND;
  const bool active = le < ne;
  const int64_t el = e0 + (active ? le : 0);
  const int ex = int(el % sl.Ex), ey = int((el / sl.Ex) % sl.Ey);
  const int ez = sl.ez0 + int(el / (int64_t(sl.Ex) * sl.Ey));
  const int64_t x = int64_t(ex) * q + i, y = int64_t(ey) * q + j, zb = int64_t(ez) * q;
  double* sa = s_a + le * NLOC;
  double* sb2 = s_b + le * NLOC;

  // phase 0: u column (i,j,:) into registers and the element block into smem
  double ureg[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) {  // unconditional loads (el is clamped to a valid element), then select
    const double raw = IO == 1 ? __ldg(&u[el * NLOC + k * ND2 + ij]) : __ldg(&u[sl.lidx(x, y, zb + k)]);
    const double v = (!active || (IO != 1 && sl.masked(x, y, zb + k))) ? 0.0 : raw;
    ureg[k] = v;
    sa[k * ND2 + ij] = v;
  }
  __syncthreads();

  // phase 1: ur, us, ut (sem_space.cpp:137-151)
  double ur[ND], us[ND], ut[ND];
  {
    double Di[ND], Dj[ND];
#pragma unroll
    for (int m = 0; m < ND; ++m) {
      Di[m] = s_D[i + ND * m];
      Dj[m] = s_D[j + ND * m];
    }
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      double dr = 0.0, ds = 0.0, dt = 0.0;
#pragma unroll
      for (int m = 0; m < ND; ++m) {
        dr = fma(Di[m], sa[k * ND2 + j * ND + m], dr);
        ds = fma(Dj[m], sa[k * ND2 + m * ND + i], ds);
        dt = fma(Dm.d[k + ND * m], ureg[m], dt);
      }
      ur[k] = dr;
      us[k] = ds;
      ut[k] = dt;
    }
  }

  // phase 2: geometric factors (sem_space.cpp:153-161), read from L2 (prefetched above)
  const GT* gg = geom + el * 6 * NLOC + ij;
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    // per-layer guarded loads: keeps the 6*ND geometry loads from all being hoisted at once
    // (that spills at the 96-register occupancy target); the geometry sits in L2 (prefetched)
    const int node = k * ND2;
    double g0 = 0, g1 = 0, g2 = 0, g3 = 0, g4 = 0, g5 = 0;
    if (active) {
      g0 = double(__ldcs(gg + 0 * NLOC + node));
      g1 = double(__ldcs(gg + 1 * NLOC + node));
      g2 = double(__ldcs(gg + 2 * NLOC + node));
      g3 = double(__ldcs(gg + 3 * NLOC + node));
      g4 = double(__ldcs(gg + 4 * NLOC + node));
      g5 = double(__ldcs(gg + 5 * NLOC + node));
    }
    const double r = ur[k], s = us[k], t = ut[k];
    ur[k] = g0 * r + g1 * s + g2 * t;
    us[k] = g1 * r + g3 * s + g4 * t;
    ut[k] = g2 * r + g4 * s + g5 * t;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    sa[k * ND2 + ij] = ur[k];
    sb2[k * ND2 + ij] = us[k];
  }
  __syncthreads();

  // phase 3: transposed contractions, interleaved in one accumulator (sem_space.cpp:163-174)
  double DiT[ND], DjT[ND];
#pragma unroll
  for (int m = 0; m < ND; ++m) {
    DiT[m] = s_D[m + ND * i];
    DjT[m] = s_D[m + ND * j];
  }
  double out[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < ND; ++m) {
      acc = fma(DiT[m], sa[k * ND2 + j * ND + m], acc);
      acc = fma(DjT[m], sb2[k * ND2 + m * ND + i], acc);
      acc = fma(Dm.d[m + ND * k], ut[m], acc);
    }
    out[k] = acc;
  }

  if (IO != 0) {
    if (active)
#pragma unroll
      for (int k = 0; k < ND; ++k) out_local[el * NLOC + k * ND2 + ij] = out[k];
    return;
  }

  // phase 4: deposit non-owned nodes, publish, wait for lower neighbours
  const bool ownx = (i < q) || (ex == sl.Ex - 1);
  const bool owny = (j < q) || (ey == sl.Ey - 1);
  const bool topz = (ez == sl.ez1 - 1);
  if (active) {
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      const bool own = ownx && owny && (k < q || topz);
      if (!own) dep[el * NLOC + k * ND2 + ij] = out[k];
    }
  }
  // CTA barrier then one gpu-scope release per element: the release is cumulative over the
  // deposits the barrier ordered before it (the CUTLASS semaphore pattern).
  __syncthreads();
  const unsigned target = s_epoch + 1u;
  if (tid < ne) st_release(&flags[e0 + tid], target);
  if (tid < 7 * EPB) {
    const int wl = tid / 7, combo = tid % 7 + 1;
    if (wl < ne) {
      const int64_t we = e0 + wl;
      const int wx = int(we % sl.Ex), wy = int((we / sl.Ex) % sl.Ey);
      const int wz = sl.ez0 + int(we / (int64_t(sl.Ex) * sl.Ey));
      const int a = combo & 1, b = (combo >> 1) & 1, c = (combo >> 2) & 1;
      if ((!a || wx > 0) && (!b || wy > 0) && (!c || wz > sl.ez0)) {
        const int64_t nb = we - a - int64_t(b) * sl.Ex - int64_t(c) * sl.Ex * sl.Ey;
        // relaxed spin: the deposits are read with ld.global.cg from L2 (the coherence point)
        // after the flag is observed, so no L1-invalidating acquire is needed
        while (ld_relaxed(&flags[nb]) < target) __nanosleep(32);
      }
    }
  }
  __syncthreads();
  if (!active) return;

  // phase 5: owned nodes summed in ascending element id (sem_space.cpp:113-117 order). All
  // deposit loads are issued up front (predicated, unrolled) so they cost one L2 round trip;
  // absent contributors add an exact 0.0, which leaves the reference's sum bitwise unchanged.
  const bool hx = (i == 0 && ex > 0), hy = (j == 0 && ey > 0), hz = (ez > sl.ez0);
  const int64_t LX = 1, LY = sl.Ex, LZ = int64_t(sl.Ex) * sl.Ey;
  const double* dbase = dep + el * NLOC + ij;
  const bool own0 = ownx && owny && hz;
  const double cz = ldcg_pred(dbase - LZ * NLOC + q * ND2, own0);
  const double cxz = ldcg_pred(dbase - (LZ + LX) * NLOC + q * ND2 + q, own0 && hx);
  const double cyz = ldcg_pred(dbase - (LZ + LY) * NLOC + q * ND2 + q * ND, own0 && hy);
  const double cxyz = ldcg_pred(dbase - (LZ + LY + LX) * NLOC + q * ND2 + q * ND + q, own0 && hx && hy);
  constexpr int KH = (ND + 1) / 2;  // two batches of layers bound the live registers
#pragma unroll
  for (int kb = 0; kb < ND; kb += KH) {
    double cx[KH], cy[KH], cxy[KH];
#pragma unroll
    for (int kk = 0; kk < KH; ++kk) {
      const int k = kb + kk;
      const bool own = k < ND && ownx && owny && (k < q || topz);
      cx[kk] = ldcg_pred(dbase - LX * NLOC + k * ND2 + q, own && hx);
      cy[kk] = ldcg_pred(dbase - LY * NLOC + k * ND2 + q * ND, own && hy);
      cxy[kk] = ldcg_pred(dbase - (LX + LY) * NLOC + k * ND2 + q * ND + q, own && hx && hy);
    }
#pragma unroll
    for (int kk = 0; kk < KH; ++kk) {
      const int k = kb + kk;
      if (k >= ND || !(ownx && owny && (k < q || topz))) continue;
      double acc = 0.0;
      if (k == 0) {  // (c=1): (b,a) = (1,1), (1,0), (0,1), (0,0)
        acc += cxyz;
        acc += cyz;
        acc += cxz;
        acc += cz;
      }
      acc += cxy[kk];  // (c=0): (1,1), (1,0), (0,1), then the element itself
      acc += cy[kk];
      acc += cx[kk];
      acc += out[k];
      const int64_t z = zb + k;
      epi(sl.lidx(x, y, z), sl.masked(x, y, z) ? 0.0 : acc);
    }
  }
}

// ------------------------------------------------------------------------ persistent Ax
// Same arithmetic and summation order as k_ax, restructured so no CTA idles on a neighbour or
// on HBM latency. A resident CTA loops over dynamic tickets (ascending element id):
//   * the element's 6 geometric-factor planes arrive in shared memory by ONE cp.async.bulk
//     (TMA engine, mbarrier completion) that was issued while the PREVIOUS element was in its
//     transposed contractions, so the 24 KB stream of each element overlaps a whole element of
//     compute; no registers or issue slots are spent on geometry loads;
//   * the next element's u rows are prefetched into L2 while this element is differentiated;
//   * the element deposits its non-owned nodes, writes the owned nodes with no lower
//     contributor (the 6^3 interior at p=7) at once, keeps its face-owned results in registers
//     and publishes its counter; only then does it finish ticket t-1's face-owned nodes, whose
//     lower neighbours have long been published.
// All lattice offsets are 32-bit (n_local < 2^31 is checked on the host); masking is
// precomputed per column (x,y) plus the two z end layers.
template <class GT>
__host__ __device__ constexpr int geom_bytes(int nloc) {
  return 6 * nloc * int(sizeof(GT));
}
__host__ __device__ constexpr int align128(int b) { return (b + 127) / 128 * 128; }

#ifndef SEMLAB_AXP_UPREFETCH
#define SEMLAB_AXP_UPREFETCH 1  // L2 prefetch of the next element's u rows
#endif

template <int ND>
constexpr int axp_minb() {  // resident CTAs per SM (shared memory allows no more at ND >= 9)
  return ND <= 8 ? SEMLAB_AXP_MINB : (ND == 9 ? 4 : 3);
}

template <int ND, class EpiT, class GT>
__global__ void __launch_bounds__(ND* ND, axp_minb<ND>())
    k_axp(const Slab sl, const DMat<ND> Dm, const double* __restrict__ u, const GT* __restrict__ geom,
          double* __restrict__ dep, unsigned* __restrict__ flags, unsigned* __restrict__ ticket, int total_tickets,
          const EpiT epi) {
  constexpr int ND2 = ND * ND, NLOC = ND2 * ND;
  constexpr int q = ND - 1;
  constexpr unsigned GB = unsigned(geom_bytes<GT>(NLOC));
  extern __shared__ __align__(128) unsigned char smem_raw[];
  GT* s_g = reinterpret_cast<GT*>(smem_raw);
  double* s_a = reinterpret_cast<double*>(smem_raw + align128(int(GB)));
  double* s_b = s_a + NLOC;
  double* s_D = s_b + NLOC;
  __shared__ uint64_t s_bar;
  __shared__ int s_tk[2];
  __shared__ unsigned s_epoch;
  const int tid = threadIdx.x;
  const int ij = tid, i = ij % ND, j = ij / ND;
  const int nE = int(sl.elems());
  const int Ex = sl.Ex, Ey = sl.Ey, LZ = Ex * Ey;
  const int Nx = int(sl.Nx), Ny = int(sl.Ny), Nz = int(sl.Nz), NxNy = Nx * Ny;
  const int zlo = int(sl.zlo);
  // D to shared memory with compile-time indices (a per-thread index into the kernel parameter
  // would make the compiler copy the whole matrix to a local-memory stack frame in every thread)
  if (tid == 0) {
#pragma unroll
    for (int t = 0; t < ND2; ++t) s_D[t] = Dm.d[t];
  }
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    const int t0 = int(atomicAdd(ticket, 1u));
    if (t0 == total_tickets - 1) atomicExch(ticket, 0u);
    s_tk[0] = t0;
    if (t0 < nE) {
      s_epoch = *reinterpret_cast<volatile unsigned*>(&flags[t0]);
      mbar_expect_tx(&s_bar, GB);
      bulk_g2s(s_g, geom + size_t(t0) * 6 * NLOC, GB, &s_bar);
    }
  }
  __syncthreads();
  const unsigned target = s_epoch + 1u;  // every element's counter equals s_epoch at launch
  unsigned phase = 0;
  int prev = -1;
  int buf = 0;
  double pprev[ND];  // face-owned results of ticket t-1, summed once its neighbours are in
#pragma unroll
  for (int k = 0; k < ND; ++k) pprev[k] = 0.0;

  // owned node (i,j,k) of element pe that has a lower contributor: sum in ascending element id
  auto finish_prev = [&](int pe) {
    const int ex = pe % Ex, ey = (pe / Ex) % Ey, ez = sl.ez0 + pe / LZ;
    if (tid < 7) {  // wait for the <= 7 lower neighbours of pe (released long ago, normally)
      const int a = (tid + 1) & 1, b = ((tid + 1) >> 1) & 1, c = ((tid + 1) >> 2) & 1;
      if ((!a || ex > 0) && (!b || ey > 0) && (!c || ez > sl.ez0)) {
        const int nb = pe - a - b * Ex - c * LZ;
        while (ld_relaxed(&flags[nb]) < target) {
        }
      }
    }
    __syncthreads();
    const bool hx = (i == 0 && ex > 0), hy = (j == 0 && ey > 0), hz = (ez > sl.ez0);
    const bool ownxy = ((i < q) || (ex == Ex - 1)) && ((j < q) || (ey == Ey - 1));
    const bool topz = (ez == sl.ez1 - 1);
    const int x = ex * q + i, y = ey * q + j, zb = ez * q;
    const int g0 = x + Nx * y + NxNy * (zb - zlo);
    const bool mxy = sl.dirichlet && (x == 0 || x == Nx - 1 || y == 0 || y == Ny - 1);
    const bool mz0 = sl.dirichlet && zb == 0, mzq = sl.dirichlet && zb + q == Nz - 1;
    const double* dbase = dep + size_t(pe) * NLOC + ij;
    const int oX = NLOC, oY = Ex * NLOC, oZ = LZ * NLOC;
    const bool own0 = ownxy && hz;
    const double cz = ldcg_pred(dbase - oZ + q * ND2, own0);
    const double cxz = ldcg_pred(dbase - (oZ + oX) + q * ND2 + q, own0 && hx);
    const double cyz = ldcg_pred(dbase - (oZ + oY) + q * ND2 + q * ND, own0 && hy);
    const double cxyz = ldcg_pred(dbase - (oZ + oY + oX) + q * ND2 + q * ND + q, own0 && hx && hy);
    constexpr int KH = (ND + 1) / 2;
#pragma unroll
    for (int kb = 0; kb < ND; kb += KH) {
      double cx[KH], cy[KH], cxy[KH];
#pragma unroll
      for (int kk = 0; kk < KH; ++kk) {
        const int k = kb + kk;
        const bool own = k < ND && ownxy && (k < q || topz);
        cx[kk] = ldcg_pred(dbase - oX + k * ND2 + q, own && hx);
        cy[kk] = ldcg_pred(dbase - oY + k * ND2 + q * ND, own && hy);
        cxy[kk] = ldcg_pred(dbase - (oX + oY) + k * ND2 + q * ND + q, own && hx && hy);
      }
#pragma unroll
      for (int kk = 0; kk < KH; ++kk) {
        const int k = kb + kk;
        if (k >= ND || !(ownxy && (k < q || topz))) continue;
        if (!(hx || hy || (k == 0 && hz))) continue;  // interior-owned: already written
        double acc = 0.0;
        if (k == 0) {  // (c=1): (b,a) = (1,1), (1,0), (0,1), (0,0)
          acc += cxyz;
          acc += cyz;
          acc += cxz;
          acc += cz;
        }
        acc += cxy[kk];  // (c=0): (1,1), (1,0), (0,1), then the element itself
        acc += cy[kk];
        acc += cx[kk];
        acc += pprev[k];
        const bool m = mxy || (k == 0 && mz0) || (k == q && mzq);
        epi(g0 + k * NxNy, m ? 0.0 : acc);
      }
    }
  };

  while (true) {
    const int el = s_tk[buf];
    if (el >= nE) break;
    if (tid == 0) {  // next ticket now, so its latency hides behind this element
      const int tn = int(atomicAdd(ticket, 1u));
      if (tn == total_tickets - 1) atomicExch(ticket, 0u);
      s_tk[buf ^ 1] = tn;
    }
    const int ex = el % Ex, ey = (el / Ex) % Ey, ez = sl.ez0 + el / LZ;
    const int x = ex * q + i, y = ey * q + j, zb = ez * q;
    const int g0 = x + Nx * y + NxNy * (zb - zlo);
    const bool mxy = sl.dirichlet && (x == 0 || x == Nx - 1 || y == 0 || y == Ny - 1);
    const bool mz0 = sl.dirichlet && zb == 0, mzq = sl.dirichlet && zb + q == Nz - 1;
    double ureg[ND];
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      const double raw = __ldg(u + g0 + k * NxNy);
      const bool m = mxy || (k == 0 && mz0) || (k == q && mzq);
      const double v = m ? 0.0 : raw;
      ureg[k] = v;
      s_a[k * ND2 + ij] = v;
    }
    __syncthreads();
#if SEMLAB_AXP_UPREFETCH
    {  // the next element's u rows (j', k') -> L2, one 64-byte row per thread
      const int tn = s_tk[buf ^ 1];
      if (tn < nE) {
        const int nx = tn % Ex, ny = (tn / Ex) % Ey, nz = sl.ez0 + tn / LZ;
        const int jj = tid % ND, kk = tid / ND;
        const double* row = u + (nx * q) + Nx * (ny * q + jj) + NxNy * (nz * q + kk - zlo);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(row));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(row + q));
      }
    }
#endif
    double ur[ND], us[ND], ut[ND];
    {
      double Di[ND], Dj[ND];
#pragma unroll
      for (int m = 0; m < ND; ++m) {
        Di[m] = s_D[i + ND * m];
        Dj[m] = s_D[j + ND * m];
      }
#pragma unroll
      for (int k = 0; k < ND; ++k) {
        double dr = 0.0, ds = 0.0, dt = 0.0;
#pragma unroll
        for (int m = 0; m < ND; ++m) {
          dr = fma(Di[m], s_a[k * ND2 + j * ND + m], dr);
          ds = fma(Dj[m], s_a[k * ND2 + m * ND + i], ds);
          dt = fma(Dm.d[k + ND * m], ureg[m], dt);
        }
        ur[k] = dr;
        us[k] = ds;
        ut[k] = dt;
      }
    }
    mbar_wait(&s_bar, phase);  // this element's geometry has landed in shared memory
    phase ^= 1u;
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      const GT* gk = s_g + k * ND2 + ij;
      const double g0v = double(gk[0 * NLOC]), g1 = double(gk[1 * NLOC]), g2 = double(gk[2 * NLOC]);
      const double g3 = double(gk[3 * NLOC]), g4 = double(gk[4 * NLOC]), g5 = double(gk[5 * NLOC]);
      const double r = ur[k], s = us[k], t = ut[k];
      ur[k] = g0v * r + g1 * s + g2 * t;
      us[k] = g1 * r + g3 * s + g4 * t;
      ut[k] = g2 * r + g4 * s + g5 * t;
    }
    __syncthreads();  // s_g and s_a are free
    if (tid == 0) {   // stream the next element's geometry while this one finishes
      const int tn = s_tk[buf ^ 1];
      if (tn < nE) {
        fence_proxy_async_shared();
        mbar_expect_tx(&s_bar, GB);
        bulk_g2s(s_g, geom + size_t(tn) * 6 * NLOC, GB, &s_bar);
      }
    }
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      s_a[k * ND2 + ij] = ur[k];
      s_b[k * ND2 + ij] = us[k];
    }
    __syncthreads();
    double pcur[ND];
    {
      double DiT[ND], DjT[ND];
#pragma unroll
      for (int m = 0; m < ND; ++m) {
        DiT[m] = s_D[m + ND * i];
        DjT[m] = s_D[m + ND * j];
      }
      const bool ownxy = ((i < q) || (ex == Ex - 1)) && ((j < q) || (ey == Ey - 1));
      const bool topz = (ez == sl.ez1 - 1);
      const bool hx = (i == 0 && ex > 0), hy = (j == 0 && ey > 0), hz = (ez > sl.ez0);
      double outk[ND];
#pragma unroll
      for (int k = 0; k < ND; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < ND; ++m) {
          acc = fma(DiT[m], s_a[k * ND2 + j * ND + m], acc);
          acc = fma(DjT[m], s_b[k * ND2 + m * ND + i], acc);
          acc = fma(Dm.d[m + ND * k], ut[m], acc);
        }
        outk[k] = acc;
      }
      // owned nodes with no lower contributor are final now: batched epilogue (all vector
      // loads first, then the stores); face-owned nodes wait in registers; the rest are deposited
      typename EpiT::In in[ND];
#pragma unroll
      for (int k = 0; k < ND; ++k) {
        const bool own = ownxy && (k < q || topz);
        if (own && !(hx || hy || (k == 0 && hz))) in[k] = epi.load(g0 + k * NxNy);
      }
      double* dl = dep + size_t(el) * NLOC + ij;
#pragma unroll
      for (int k = 0; k < ND; ++k) {
        const bool own = ownxy && (k < q || topz);
        pcur[k] = outk[k];
        if (!own) {
          dl[k * ND2] = outk[k];
        } else if (!(hx || hy || (k == 0 && hz))) {
          const bool m = mxy || (k == 0 && mz0) || (k == q && mzq);
          epi.store(g0 + k * NxNy, in[k], m ? 0.0 : outk[k]);
        }
      }
    }
    __syncthreads();
    if (tid == 0) st_release(&flags[el], target);
    if (prev >= 0) finish_prev(prev);
#pragma unroll
    for (int k = 0; k < ND; ++k) pprev[k] = pcur[k];
    prev = el;
    buf ^= 1;
  }
  if (prev >= 0) finish_prev(prev);
}

template <int ND, class GT, class EpiT>
int64_t axp_launch(const Slab& sl, const double* u, const GT* geom, const AxSync& sy, const EpiT& epi,
                   cudaStream_t s) {
  constexpr int NLOC = ND * ND * ND;
  const int64_t nE = sl.elems();
  if (nE == 0) return 0;
  if (sl.n_local() >= (int64_t(1) << 31) || nE * NLOC >= (int64_t(1) << 31))
    invalid("SemSpace: a rank's lattice must have < 2^31 nodes");
  const size_t smem = size_t(align128(geom_bytes<GT>(NLOC))) + (size_t(2) * NLOC + ND * ND) * sizeof(double);
  auto kern = k_axp<ND, EpiT, GT>;
  const int nctas = resident_ctas(kern, ND * ND, smem);
  const int grid = capped_grid(std::min<int64_t>(nctas, nE));
  kern<<<grid, ND * ND, smem, s>>>(sl, dmat<ND>(sl.q), u, geom, sy.dep, sy.flags, sy.ticket, int(nE + grid), epi);
  SB_LAUNCH_CHECK();
  return 1;
}

struct Cands {  // elements (along one axis) containing a lattice coordinate, ascending
  int n;
  int e[2];
  int loc[2];
};
__device__ __forceinline__ Cands cands(int64_t c, int q, int Eax, int lo_elem, int hi_elem) {
  // hi_elem = one past the last element layer available locally
  Cands r;
  int64_t e = c / q;
  const int l = int(c % q);
  if (l == 0 && e > 0) {
    r.n = 0;
    if (e - 1 >= lo_elem) { r.e[r.n] = int(e - 1); r.loc[r.n] = q; ++r.n; }
    if (e < hi_elem) { r.e[r.n] = int(e); r.loc[r.n] = 0; ++r.n; }
  } else {
    if (e == Eax) { e -= 1; }
    r.n = 1;
    r.e[0] = int(e);
    r.loc[0] = (e * q == c) ? 0 : int(c - e * q);
  }
  return r;
}

// ------------------------------------------------------------------------ warp-per-element Ax (p = 7)
// The p=7 operator on the FP64 tensor cores, in two launches with no inter-CTA waiting:
//
// k_axe: one warp per element (grid-stride, static order). Every contraction of
//   sem_space.cpp:137-174 is a stack of 8x8x8 products, i.e. two mma.m8n8k4.f64 (DMMA) each:
//     ur_k = U_k D^T, us_k = D U_k (per z-layer k), ut_(.,j,.) = D U_(.,j,.) (per y-row j),
//     out_k = Gr_k D + D^T Gs_k (+) D^T Gt_(.,j,.)
//   so an element costs 96 DMMA. A lane holds the nodes (k = 0..7, j = lane/4, i = 2(lane%4) +
//   {0,1}), the D fragments live in 4 registers, and the per-warp shared workspace (3 arrays of
//   8 z-layers) is padded and XOR-swizzled so every fragment access is conflict-free. The 216
//   interior nodes of the element have a single contributor: their epilogue (plain write,
//   residual, or the whole Chebyshev-Jacobi update) is applied right here. The 296 face nodes
//   go to a compact per-element face buffer (E x 296 doubles, 78 MB at E=32^3: written and read
//   back through L2). The next element's geometry and u rows are prefetched to L2 while this
//   one is computed, so every warp keeps a whole element of loads in flight.
// k_face_epi7: one thread per lattice node on an element face sums its 2-8 contributions from
//   the face buffer in ASCENDING element id (the order of the reference gather,
//   sem_space.cpp:40-52, 110-119), applies the Dirichlet mask and the epilogue. Results are
//   bitwise those of the one-kernel owner-ordered protocol this replaces, and deterministic.
namespace axw {
constexpr int PS = 72;  // z-layer stride (doubles): 64 + 8 so consecutive layers use opposite bank halves
constexpr int ARR = 8 * PS;
constexpr int FACE = 296;  // face nodes of a p=7 element: 2 x 64 (k = 0, 7) + 6 x 28 (rings)
__device__ __forceinline__ int sidx(int k, int j, int i) {  // swizzled workspace index
  return k * PS + j * 8 + 2 * ((i >> 1) ^ ((j >> 1) & 3)) + (i & 1);
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
// Face-buffer stores keep their lines in L2 (evict_last): the face gather reads them back right
// after, while the geometry streams past with evict-first loads, so the 78 MB buffer need not
// round-trip through HBM.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_l2_keep(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
// compact index of a face node (i, j, k) of an 8^3 element (at least one coordinate is 0 or 7)
__device__ __forceinline__ int face_idx(int i, int j, int k) {
  if (k == 0) return j * 8 + i;
  if (k == 7) return 64 + j * 8 + i;
  const int b = 128 + (k - 1) * 28;
  if (j == 0) return b + i;
  if (j == 7) return b + 8 + i;
  return b + 16 + 2 * (j - 1) + (i == 7 ? 1 : 0);
}
}  // namespace axw

#ifndef SEMLAB_AXW_WARPS
#define SEMLAB_AXW_WARPS 4  // warps (independent element pipelines) per CTA
#endif
#ifndef SEMLAB_AXW_GEOM_AHEAD
#define SEMLAB_AXW_GEOM_AHEAD 1  // FP32-factor layers loaded ahead of the one in use (2, 3 measured slower)
#endif
#ifndef SEMLAB_AXW_MINB
#define SEMLAB_AXW_MINB 3  // resident CTAs per SM
#endif

__host__ __device__ constexpr int axw_warp_doubles() { return 3 * axw::ARR; }  // per-warp shared memory in doubles

template <class GT>
struct GeomRaw;
template <>
struct GeomRaw<double> {
  using T = double2;
};
template <>
struct GeomRaw<float> {
  using T = float2;
};
__device__ __forceinline__ double2 ld_geom_raw(const double* p) { return __ldcs(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ float2 ld_geom_raw(const float* p) { return __ldcs(reinterpret_cast<const float2*>(p)); }
__device__ __forceinline__ double2 geom_to_d2(double2 v) { return v; }
__device__ __forceinline__ double2 geom_to_d2(float2 v) { return make_double2(double(v.x), double(v.y)); }

// GT = double: the operator itself (Krylov A). GT = float: the smoother's operator with the
// geometric factors rounded to FP32 (half the bytes; arithmetic stays FP64 on the DMMA path).
template <class EpiT, class GT>
__global__ void __launch_bounds__(32 * SEMLAB_AXW_WARPS, SEMLAB_AXW_MINB)
    k_axe(const Slab sl, const DMat<8> Dm, const double* __restrict__ u, const GT* __restrict__ geom,
          double* __restrict__ fb, const EpiT epi) {
  using namespace axw;
  constexpr int ND = 8, ND2 = 64, NLOC = 512, q = 7;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* sU = reinterpret_cast<double*>(smem_raw) + size_t(wid) * axw_warp_doubles();  // u, then Gr
  double* sS = sU + ARR;                                                               // Gs
  double* sT = sS + ARR;                                                               // ut, Gt, then D^T Gt
  const int gj = lane >> 2, gc = lane & 3;  // fragment row / column group
  const int j = gj, i0 = 2 * gc;            // this lane's nodes: (k, j, i0 + {0,1})
  // D fragments: Df[kc] = D(lane/4, lane%4 + 4kc), Dt[kc] = D(lane%4 + 4kc, lane/4)
  double Df[2], Dt[2];
#pragma unroll
  for (int kc = 0; kc < 2; ++kc) {
    Df[kc] = Dm.d[gj + ND * (gc + 4 * kc)];
    Dt[kc] = Dm.d[(gc + 4 * kc) + ND * gj];
  }
  const int nE = int(sl.elems());
  const int Ex = sl.Ex, Ey = sl.Ey, LZ = Ex * Ey;
  const int Nx = int(sl.Nx), Ny = int(sl.Ny), Nz = int(sl.Nz), NxNy = Nx * Ny;
  const int zlo = int(sl.zlo);
  const int stride = gridDim.x * SEMLAB_AXW_WARPS;

  auto prefetch = [&](int e) {  // element e's geometry (24 KB FP64 / 12 KB FP32) and u rows -> L2
    const char* gb = reinterpret_cast<const char*>(geom + size_t(e) * 6 * NLOC);
    constexpr int GL = 6 * NLOC * int(sizeof(GT)) / 128 / 32;  // 128-byte lines per lane
#pragma unroll
    for (int l = 0; l < GL; ++l) asm volatile("prefetch.global.L2 [%0];" ::"l"(gb + (l * 32 + lane) * 128));
    const int ex = e % Ex, ey = (e / Ex) % Ey, ez = sl.ez0 + e / LZ;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int row = lane * 2 + r, jj = row & 7, kk = row >> 3;
      const double* p = u + (ex * q) + Nx * (ey * q + jj) + NxNy * (ez * q + kk - zlo);
      asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(p + q));
    }
  };

  int el = blockIdx.x * SEMLAB_AXW_WARPS + wid;
  if (el < nE) prefetch(el);
  for (; el < nE; el += stride) {
    if (el + stride < nE) prefetch(el + stride);
    const int ex = el % Ex, ey = (el / Ex) % Ey, ez = sl.ez0 + el / LZ;
    const int y = ey * q + j, zb = ez * q;
    const int xb = ex * q + i0;
    const int g0 = xb + Nx * y + NxNy * (zb - zlo);
    const bool my = sl.dirichlet && (y == 0 || y == Ny - 1);
    const bool mx0 = my || (sl.dirichlet && (xb == 0 || xb == Nx - 1));
    const bool mx1 = my || (sl.dirichlet && (xb + 1 == Nx - 1));
    const bool mz0 = sl.dirichlet && zb == 0, mzq = sl.dirichlet && zb + q == Nz - 1;
    __syncwarp();  // the previous element's workspace reads are done
    // u: this lane's 16 nodes (masked, sem_space.cpp:199) -> swizzled workspace
    {
      double v[16];
#pragma unroll
      for (int k = 0; k < ND; ++k) {
        v[2 * k] = __ldg(u + g0 + k * NxNy);
        v[2 * k + 1] = __ldg(u + g0 + k * NxNy + 1);
      }
#pragma unroll
      for (int k = 0; k < ND; ++k) {
        const bool mz = (k == 0 && mz0) || (k == q && mzq);
        const double a = (mx0 || mz) ? 0.0 : v[2 * k], b = (mx1 || mz) ? 0.0 : v[2 * k + 1];
        *reinterpret_cast<double2*>(sU + sidx(k, j, i0)) = make_double2(a, b);
      }
    }
    __syncwarp();
    // ut: per y-row jj, (k, i) <- D (k, m) U(m, jj, i)
#pragma unroll
    for (int jj = 0; jj < ND; ++jj) {
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) dmma(c0, c1, Df[kc], sU[sidx(gc + 4 * kc, jj, gj)]);
      *reinterpret_cast<double2*>(sT + sidx(gj, jj, i0)) = make_double2(c0, c1);
    }
    __syncwarp();
    // per z-layer: ur, us (DMMA), ut (workspace), geometric factors, then Gr/Gs/Gt back out
    const GT* ge = geom + size_t(el) * 6 * NLOC + j * ND + i0;
    // geometry ring: GD layers in flight ahead of the one in use (FP32 factors stay packed in
    // registers until used, so the deeper ring costs fewer registers than FP64's one-ahead)
    constexpr int GD = std::is_same_v<GT, float> ? SEMLAB_AXW_GEOM_AHEAD : 1;
    typename GeomRaw<GT>::T gq[GD + 1][6];
#pragma unroll
    for (int a = 0; a < GD; ++a)
#pragma unroll
      for (int c = 0; c < 6; ++c) gq[a][c] = ld_geom_raw(ge + c * NLOC + a * ND2);
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      if (k + GD < ND) {
#pragma unroll
        for (int c = 0; c < 6; ++c) gq[(k + GD) % (GD + 1)][c] = ld_geom_raw(ge + c * NLOC + (k + GD) * ND2);
      }
      double2 gcur[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) gcur[c] = geom_to_d2(gq[k % (GD + 1)][c]);
      double r0 = 0.0, r1 = 0.0, s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) {
        dmma(r0, r1, sU[sidx(k, gj, gc + 4 * kc)], Df[kc]);
        dmma(s0, s1, Df[kc], sU[sidx(k, gc + 4 * kc, gj)]);
      }
      const double2 t2 = *reinterpret_cast<const double2*>(sT + sidx(k, j, i0));
      __syncwarp();  // every lane has read layer k of u before it is overwritten by Gr
      double gr[2], gs[2], gt[2];
      {
        const double rr[2] = {r0, r1}, ss[2] = {s0, s1}, tt[2] = {t2.x, t2.y};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double G0 = h ? gcur[0].y : gcur[0].x, G1 = h ? gcur[1].y : gcur[1].x;
          const double G2 = h ? gcur[2].y : gcur[2].x, G3 = h ? gcur[3].y : gcur[3].x;
          const double G4 = h ? gcur[4].y : gcur[4].x, G5 = h ? gcur[5].y : gcur[5].x;
          gr[h] = G0 * rr[h] + G1 * ss[h] + G2 * tt[h];
          gs[h] = G1 * rr[h] + G3 * ss[h] + G4 * tt[h];
          gt[h] = G2 * rr[h] + G4 * ss[h] + G5 * tt[h];
        }
      }
      *reinterpret_cast<double2*>(sU + sidx(k, j, i0)) = make_double2(gr[0], gr[1]);
      *reinterpret_cast<double2*>(sS + sidx(k, j, i0)) = make_double2(gs[0], gs[1]);
      *reinterpret_cast<double2*>(sT + sidx(k, j, i0)) = make_double2(gt[0], gt[1]);
    }
    __syncwarp();
    // out_k = Gr_k D + D^T Gs_k
    double o[16];
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) dmma(c0, c1, sU[sidx(k, gj, gc + 4 * kc)], Dt[kc]);
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) dmma(c0, c1, Dt[kc], sS[sidx(k, gc + 4 * kc, gj)]);
      o[2 * k] = c0;
      o[2 * k + 1] = c1;
    }
    // + D^T Gt per y-row (in place in the workspace: row jj is read and written only here)
#pragma unroll
    for (int jj = 0; jj < ND; ++jj) {
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) dmma(c0, c1, Dt[kc], sT[sidx(gc + 4 * kc, jj, gj)]);
      __syncwarp();
      *reinterpret_cast<double2*>(sT + sidx(gj, jj, i0)) = make_double2(c0, c1);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      const double2 t2 = *reinterpret_cast<const double2*>(sT + sidx(k, j, i0));
      o[2 * k] += t2.x;
      o[2 * k + 1] += t2.y;
    }
    // epilogue: interior nodes (one contributor) now, face nodes to the face buffer
    {
      const uint64_t keep = l2_evict_last_policy();
      const bool jface = (j == 0 || j == q);
      double* fe = fb + size_t(el) * FACE;
#pragma unroll
      for (int kb = 0; kb < ND; kb += 4) {
        typename EpiT::In in[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int k = kb + t / 2, i = i0 + t % 2;
          const bool face = jface || k == 0 || k == q || i == 0 || i == q;
          if (!face) in[t] = epi.load(g0 + k * NxNy + t % 2);
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int k = kb + t / 2, i = i0 + t % 2;
          const bool face = jface || k == 0 || k == q || i == 0 || i == q;
          const double v = o[2 * k + t % 2];
          if (face)
            st_l2_keep(fe + face_idx(i, j, k), v, keep);
          else
            epi.store(g0 + k * NxNy + t % 2, in[t], v);
        }
      }
    }
  }
}

// Face nodes of the slab: (a) planes z % q == 0, (b) z % q != 0 with y % q == 0, (c) z, y % q != 0
// with x % q == 0 — consecutive threads walk x in every family. Each node sums its contributors'
// face-buffer entries in ascending element id: the (lower, upper) candidates of z, then y, then
// x, all eight loads predicated and issued together.
struct Cand2 {  // the <= 2 elements along one axis containing a lattice coordinate (lower first)
  int e0, l0, e1, l1;
  bool v0, v1;
};
__device__ __forceinline__ Cand2 cand2(int c, int q, int lo_e, int hi_e) {
  Cand2 r;
  const int e = c / q, l = c - e * q;
  if (l == 0) {  // on an element boundary: lower element (local q), upper element (local 0)
    r.e0 = e - 1;
    r.l0 = q;
    r.v0 = e - 1 >= lo_e;
    r.e1 = e;
    r.l1 = 0;
    r.v1 = e < hi_e;
  } else {
    r.e0 = e;
    r.l0 = l;
    r.v0 = true;
    r.e1 = e;
    r.l1 = l;
    r.v1 = false;
  }
  return r;
}

// The split-path gather (low orders): one thread per lattice node of the slab, x along the
// threads and (y, z) from the block indices (32-bit, no divisions by runtime extents); the node
// sums its <= 8 contributors' element-local values in ascending element id (z, then y, then x
// candidates, lower first — sem_space.cpp:110-119), loads predicated and issued together; absent
// contributors add +0.0, so the sums are bitwise those of the candidate-list loops.
template <int ND, class EpiT>
__global__ void __launch_bounds__(128) k_gather_epi(const Slab sl, const double* __restrict__ loc, const EpiT epi) {
  constexpr int q = ND - 1, NLOC = ND * ND * ND;
  const int x = int(blockIdx.x * blockDim.x + threadIdx.x);
  if (x >= sl.Nx) return;
  const int y = int(blockIdx.y), z = sl.ez0 * q + int(blockIdx.z);
  const int64_t g = sl.lidx(x, y, z);
  if (sl.masked(x, y, z)) {
    epi(g, 0.0);
    return;
  }
  const Cand2 cx = cand2(x, q, 0, sl.Ex), cy = cand2(y, q, 0, sl.Ey), cz = cand2(z, q, sl.ez0, sl.ez1);
  double v[8];
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const bool on = (c ? cz.v1 : cz.v0) && (b ? cy.v1 : cy.v0) && (a ? cx.v1 : cx.v0);
        const int el = (a ? cx.e1 : cx.e0) + sl.Ex * ((b ? cy.e1 : cy.e0) + sl.Ey * ((c ? cz.e1 : cz.e0) - sl.ez0));
        const int li = (a ? cx.l1 : cx.l0) + ND * ((b ? cy.l1 : cy.l0) + ND * (c ? cz.l1 : cz.l0));
        v[c * 4 + b * 2 + a] = on ? __ldg(loc + int64_t(el) * NLOC + li) : 0.0;
      }
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc += v[k];
  epi(g, acc);
}

// One face lattice node (x, y, z) of family FAM: sum its contributors' face-buffer entries in
// ascending element id — the (lower, upper) candidates of z, then y, then x, the loads predicated
// and issued together — apply the Dirichlet mask and the epilogue. The family fixes which axes
// can split (FAM 0: z on an element face, x and y any; FAM 1: z interior, y on a face, x any;
// FAM 2: z and y interior, x on a face), so only the 8 / 4 / 2 possible contributors are formed
// and their face indices reduce to the closed forms of face_idx for that face.
// A face lattice node in flight: its contributors' face-buffer values (absent ones +0.0, padded
// to 8), its lattice index, the Dirichlet mask and the epilogue's inputs.
template <class EpiT>
struct FaceSite {
  double v[8];
  int64_t g;
  bool on, masked;
  typename EpiT::In in;
};

// Issue the loads of face node (x, y, z) of family FAM: its contributors' face-buffer entries in
// ascending element id — the (lower, upper) candidates of z, then y, then x — all predicated and
// issued together. The family fixes which axes can split (FAM 0: z on an element face, x and y
// any; FAM 1: z interior, y on a face, x any; FAM 2: z and y interior, x on a face), so only the
// 8 / 4 / 2 possible contributors are formed and their face indices reduce to closed forms.
template <int FAM, class EpiT>
__device__ __forceinline__ void face_load7(const Slab& sl, const double* __restrict__ fb, const EpiT& epi, int x,
                                           int y, int z, FaceSite<EpiT>& f) {
  using namespace axw;
  constexpr int q = 7;
  f.on = true;
  f.g = sl.lidx(x, y, z);
  f.masked = sl.masked(x, y, z);
#pragma unroll
  for (int c = 0; c < 8; ++c) f.v[c] = 0.0;
  if constexpr (FAM == 0) {
    const Cand2 cx = cand2(x, q, 0, sl.Ex), cy = cand2(y, q, 0, sl.Ey);
    const int ezu = z / q - sl.ez0;  // upper element layer (local k = 0); lower: ezu - 1 (k = q)
    const bool zv[2] = {ezu - 1 >= 0, ezu < sl.ez1 - sl.ez0};
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int aa = 0; aa < 2; ++aa) {
          const bool on = !f.masked && zv[c] && (bb ? cy.v1 : cy.v0) && (aa ? cx.v1 : cx.v0);
          const int ey = bb ? cy.e1 : cy.e0, ex = aa ? cx.e1 : cx.e0;
          const int el = ex + sl.Ex * (ey + sl.Ey * (ezu - 1 + c));
          const int fi = (c ? 0 : 64) + (bb ? cy.l1 : cy.l0) * 8 + (aa ? cx.l1 : cx.l0);
          f.v[c * 4 + bb * 2 + aa] = on ? __ldcs(fb + size_t(el) * FACE + fi) : 0.0;
        }
  } else {
    const int ez = z / q, k = z - ez * q;  // interior layer k = 1 .. q-1 of element layer ez
    const int zb = 128 + (k - 1) * 28;
    if constexpr (FAM == 1) {
      const Cand2 cx = cand2(x, q, 0, sl.Ex);
      const int eyu = y / q;  // upper element row (j = 0); lower: eyu - 1 (j = q)
      const bool yv[2] = {eyu - 1 >= 0, eyu < sl.Ey};
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int aa = 0; aa < 2; ++aa) {
          const bool on = !f.masked && yv[bb] && (aa ? cx.v1 : cx.v0);
          const int ex = aa ? cx.e1 : cx.e0;
          const int el = ex + sl.Ex * (eyu - 1 + bb + sl.Ey * (ez - sl.ez0));
          const int fi = zb + (bb ? 0 : 8) + (aa ? cx.l1 : cx.l0);
          f.v[bb * 2 + aa] = on ? __ldcs(fb + size_t(el) * FACE + fi) : 0.0;
        }
    } else {
      const int ey = y / q, j = y - ey * q;  // interior row j = 1 .. q-1
      const int exu = x / q;                  // upper element (i = 0); lower: exu - 1 (i = q)
      const bool xv[2] = {exu - 1 >= 0, exu < sl.Ex};
#pragma unroll
      for (int aa = 0; aa < 2; ++aa) {
        const int el = exu - 1 + aa + sl.Ex * (ey + sl.Ey * (ez - sl.ez0));
        const int fi = zb + 16 + 2 * (j - 1) + (aa ? 0 : 1);
        f.v[aa] = (!f.masked && xv[aa]) ? __ldcs(fb + size_t(el) * FACE + fi) : 0.0;
      }
    }
  }
  if (!f.masked) f.in = epi.load(f.g);
}

// Sum in ascending element id (absent contributors and the padding add +0.0: bitwise the sum
// over the present ones), apply the mask and the epilogue.
template <class EpiT>
__device__ __forceinline__ void face_finish7(const FaceSite<EpiT>& f, const EpiT& epi) {
  if (!f.on) return;
  if (f.masked) {
    epi(f.g, 0.0);
    return;
  }
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc += f.v[c];
  epi.store(f.g, f.in, acc);
}

// One launch for the three families: blockIdx.z enumerates the z planes of the slab
// (z = zb + zz, zz = 0 .. nzl q); blockIdx.y the rows of the plane's family; x along threads.
//   z % q == 0 (FAM 0): rows y = 0 .. Ny-1, threads over x
//   z % q != 0: rows 0 .. Ey  are FAM 1 (y = q row, threads over x);
//               rows Ey+1 .. 2Ey are FAM 2 (y in element row ey = row-Ey-1, threads over (i, y-1-q ey))
#ifndef SEMLAB_FACE_ROWS
#define SEMLAB_FACE_ROWS 2  // face rows per block step (loads of all in flight together; 3, 4 slower)
#endif
#ifndef SEMLAB_FACE_BLOCKS
#define SEMLAB_FACE_BLOCKS (148 * 64)  // face-pass blocks (each walks rows with stride gridDim.y)
#endif
template <class EpiT>
__global__ void __launch_bounds__(128) k_face_epi7(const Slab sl, const double* __restrict__ fb, const EpiT epi) {
  constexpr int q = 7;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  // compact row list: the Ny rows of each of the nzl+1 planes z % q == 0, then the 2 Ey + 1 face
  // rows of each of the 6 nzl planes between them; a block walks rows with stride gridDim.y
  const int ra = (sl.ez1 - sl.ez0 + 1) * sl.Ny, rb = 2 * sl.Ey + 1;
  const int rows = ra + (sl.ez1 - sl.ez0) * (q - 1) * rb;
  // one face row -> this thread's site in it (f.on = false past the row's end)
  auto load_row = [&](int r, FaceSite<EpiT>& f) {
    f.on = false;
    if (r < ra) {
      const int pz = r / sl.Ny, row = r - pz * sl.Ny;
      if (t < sl.Nx) face_load7<0>(sl, fb, epi, t, row, (sl.ez0 + pz) * q, f);
      return;
    }
    const int rr = r - ra, pl = rr / rb, row = rr - pl * rb;
    const int ez = pl / (q - 1), z = (sl.ez0 + ez) * q + 1 + (pl - ez * (q - 1));
    if (row <= sl.Ey) {
      if (t < sl.Nx) face_load7<1>(sl, fb, epi, t, row * q, z, f);
    } else {
      const int i = t / (q - 1), yi = t - i * (q - 1);
      if (i <= sl.Ex) face_load7<2>(sl, fb, epi, i * q, (row - sl.Ey - 1) * q + 1 + yi, z, f);
    }
  };
  // SEMLAB_FACE_ROWS rows per step: all their loads are in flight before any is summed
  constexpr int NR = SEMLAB_FACE_ROWS;
  const int gy = int(gridDim.y);
  for (int r = int(blockIdx.y); r < rows; r += NR * gy) {
    FaceSite<EpiT> f[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      f[k].on = false;
      if (r + k * gy < rows) load_row(r + k * gy, f[k]);
    }
#pragma unroll
    for (int k = 0; k < NR; ++k) face_finish7(f[k], epi);
  }
}

template <class EpiT, class GT>
int64_t axw_launch(const Slab& sl, const double* u, const GT* geom, const AxSync& sy, const EpiT& epi,
                   cudaStream_t s) {
  constexpr int NLOC = 512;
  const int64_t nE = sl.elems();
  if (nE == 0) return 0;
  if (sl.n_local() >= (int64_t(1) << 31) || nE * NLOC >= (int64_t(1) << 31))
    invalid("SemSpace: a rank's lattice must have < 2^31 nodes");
  constexpr int W = SEMLAB_AXW_WARPS;
  const size_t smem = size_t(W) * axw_warp_doubles() * sizeof(double);
  auto kern = k_axe<EpiT, GT>;
  const int nctas = resident_ctas(kern, 32 * W, smem);
  const int grid = capped_grid(std::min<int64_t>(nctas, (nE + W - 1) / W));
  kern<<<grid, 32 * W, smem, s>>>(sl, dmat<8>(sl.q), u, geom, sy.dep, epi);
  SB_LAUNCH_CHECK();
  const unsigned nzl = unsigned(sl.ez1 - sl.ez0);
  const unsigned bx = unsigned((std::max<int64_t>(sl.Nx, (sl.Ex + 1) * 6) + 127) / 128);
  const int64_t rows = int64_t(nzl + 1) * sl.Ny + int64_t(nzl) * 6 * (2 * sl.Ey + 1);
  const unsigned by = unsigned(std::min<int64_t>(rows, std::max<int64_t>(1, SEMLAB_FACE_BLOCKS / bx)));
  k_face_epi7<<<dim3(bx, by), 128, 0, s>>>(sl, sy.dep, epi);
  SB_LAUNCH_CHECK();
  return 2;
}

#ifndef SEMLAB_AX_DMMA
#define SEMLAB_AX_DMMA 1  // build-time A/B: 0 = the FP64-FMA persistent kernel at p = 7
#endif
constexpr bool ax_dmma() { return SEMLAB_AX_DMMA != 0; }

// Q^T of element-local results with an owner epilogue: each lattice node sums its <= 8
// contributors in ascending element id (sem_space.cpp:110-119 order), masked nodes get 0.
template <int ND, bool LOCAL, class EpiT, class GT = double>
int64_t ax_dispatch_nd(const Slab& sl, const double* u, const GT* geom, const AxSync& sy, double* out_local,
                       const EpiT& epi, cudaStream_t s) {
  if constexpr (!LOCAL && ND >= 8 && std::is_same_v<GT, double>) {
    if constexpr (ND == 8) {
      if (ax_dmma()) return axw_launch(sl, u, geom, sy, epi, s);
    }
    if (ax_persistent()) return axp_launch<ND>(sl, u, geom, sy, epi, s);
  }
  constexpr int EPB = epb<ND>();
  constexpr int NLOC = ND * ND * ND;
  const int64_t nE = sl.elems();
  if (nE == 0) return 0;
  const int ngroups = int((nE + EPB - 1) / EPB);
  const size_t smem = (size_t(EPB) * 2 * NLOC + ND * ND) * sizeof(double);
  // low orders: element-local Ax into the deposit buffer, then the ordered gather with the
  // epilogue (two fully parallel launches instead of CTAs idling on neighbour counters)
  constexpr int IO = LOCAL ? 1 : (ND <= SEMLAB_AX_SPLIT_ND ? 2 : 0);
  static_assert(std::is_same_v<GT, double> || IO == 2, "FP32 factors: the split path only");
  auto kern = k_ax<ND, EPB, IO, EpiT, GT>;
  smem_attr(kern, smem);
  kern<<<ngroups, EPB * ND * ND, smem, s>>>(sl, dmat<ND>(sl.q), u, geom, sy.dep, sy.flags, sy.ticket, ngroups,
                                           IO == 2 ? sy.dep : out_local, epi);
  SB_LAUNCH_CHECK();
  if constexpr (IO == 2) {
    const int64_t nzl = int64_t(sl.ez1 - sl.ez0) * sl.q + 1;
    if (sl.Ny > 65535 || nzl > 65535 || nE * NLOC >= (int64_t(1) << 31))
      invalid("SemSpace: lattice too large for the split-path gather");
    k_gather_epi<ND><<<dim3(unsigned((sl.Nx + 127) / 128), unsigned(sl.Ny), unsigned(nzl)), 128, 0, s>>>(sl, sy.dep,
                                                                                                         epi);
    SB_LAUNCH_CHECK();
    return 2;
  }
  return 1;
}

template <bool LOCAL, class EpiT>
int64_t ax_dispatch(const Slab& sl, const double* u, const double* geom, const AxSync& sy, double* out_local,
                    const EpiT& epi, cudaStream_t s) {
  switch (sl.q + 1) {
    case 2: return ax_dispatch_nd<2, LOCAL>(sl, u, geom, sy, out_local, epi, s);
    case 3: return ax_dispatch_nd<3, LOCAL>(sl, u, geom, sy, out_local, epi, s);
    case 4: return ax_dispatch_nd<4, LOCAL>(sl, u, geom, sy, out_local, epi, s);
    case 5: return ax_dispatch_nd<5, LOCAL>(sl, u, geom, sy, out_local, epi, s);
    case 6: return ax_dispatch_nd<6, LOCAL>(sl, u, geom, sy, out_local, epi, s);
    case 7: return ax_dispatch_nd<7, LOCAL>(sl, u, geom, sy, out_local, epi, s);
    case 8: return ax_dispatch_nd<8, LOCAL>(sl, u, geom, sy, out_local, epi, s);
    case 9: return ax_dispatch_nd<9, LOCAL>(sl, u, geom, sy, out_local, epi, s);
    case 10: return ax_dispatch_nd<10, LOCAL>(sl, u, geom, sy, out_local, epi, s);
    default: invalid("SemSpace: device kernels support orders 1..9, got " + std::to_string(sl.q));
  }
}

// ------------------------------------------------------------------------ diag
// sem_space.cpp:211-236 (local part; gathered by k_gather)
template <int ND>
__global__ void k_local_diag(const Slab sl, const DMat<ND> Dm, const double* __restrict__ geom,
                             double* __restrict__ out) {
  constexpr int NLOC = ND * ND * ND, ND2 = ND * ND;
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= sl.elems() * NLOC) return;
  const int64_t el = idx / NLOC;
  const int node = int(idx % NLOC);
  const int i = node % ND, j = (node / ND) % ND, k = node / ND2;
  const double* G = geom + el * 6 * NLOC;
  double acc = 0.0;
  for (int m = 0; m < ND; ++m) {
    const double a = Dm.d[m + ND * i], b = Dm.d[m + ND * j], c = Dm.d[m + ND * k];
    acc += a * a * G[0 * NLOC + m + ND * j + ND2 * k];
    acc += b * b * G[3 * NLOC + i + ND * m + ND2 * k];
    acc += c * c * G[5 * NLOC + i + ND * j + ND2 * m];
  }
  const double dii = Dm.d[i + ND * i], djj = Dm.d[j + ND * j], dkk = Dm.d[k + ND * k];
  acc += 2.0 * (dii * djj * G[1 * NLOC + node] + dii * dkk * G[2 * NLOC + node] + djj * dkk * G[4 * NLOC + node]);
  out[idx] = acc;
}

// ------------------------------------------------------------------------ Q, Q^T, QQ^T

__global__ void k_gather(const Slab sl, const double* __restrict__ loc, double* __restrict__ out) {
  const int q = sl.q, nd = q + 1;
  const int64_t nloc = int64_t(nd) * nd * nd;
  const int64_t zb = int64_t(sl.ez0) * q, nz = int64_t(sl.ez1 - sl.ez0) * q + 1;
  const int64_t total = sl.Nx * sl.Ny * nz;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t x = t % sl.Nx, y = (t / sl.Nx) % sl.Ny, z = zb + t / (sl.Nx * sl.Ny);
    const Cands cx = cands(x, q, sl.Ex, 0, sl.Ex), cy = cands(y, q, sl.Ey, 0, sl.Ey);
    const Cands cz = cands(z, q, sl.Ez, sl.ez0, sl.ez1);
    double acc = 0.0;
    for (int c = 0; c < cz.n; ++c)
      for (int b = 0; b < cy.n; ++b)
        for (int a = 0; a < cx.n; ++a) {
          const int64_t el = cx.e[a] + int64_t(sl.Ex) * (cy.e[b] + int64_t(sl.Ey) * (cz.e[c] - sl.ez0));
          acc += loc[el * nloc + cx.loc[a] + nd * (cy.loc[b] + nd * cz.loc[c])];
        }
    out[sl.lidx(x, y, z)] = acc;
  }
}

__global__ void k_scatter(const Slab sl, const double* __restrict__ glob, double* __restrict__ loc) {
  const int q = sl.q, nd = q + 1;
  const int64_t nloc = int64_t(nd) * nd * nd;
  const int64_t total = sl.elems() * nloc;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t el = t / nloc;
    const int node = int(t % nloc);
    const int i = node % nd, j = (node / nd) % nd, k = node / (nd * nd);
    const int ex = int(el % sl.Ex), ey = int((el / sl.Ex) % sl.Ey), ez = sl.ez0 + int(el / (int64_t(sl.Ex) * sl.Ey));
    loc[t] = glob[sl.lidx(int64_t(ex) * q + i, int64_t(ey) * q + j, int64_t(ez) * q + k)];
  }
}

__global__ void k_qqt(const Slab sl, const double* __restrict__ in, double* __restrict__ out) {
  const int q = sl.q, nd = q + 1;
  const int64_t nloc = int64_t(nd) * nd * nd;
  const int64_t total = sl.elems() * nloc;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t el = t / nloc;
    const int node = int(t % nloc);
    const int i = node % nd, j = (node / nd) % nd, k = node / (nd * nd);
    const int ex = int(el % sl.Ex), ey = int((el / sl.Ex) % sl.Ey), ez = sl.ez0 + int(el / (int64_t(sl.Ex) * sl.Ey));
    const Cands cx = cands(int64_t(ex) * q + i, q, sl.Ex, 0, sl.Ex);
    const Cands cy = cands(int64_t(ey) * q + j, q, sl.Ey, 0, sl.Ey);
    const Cands cz = cands(int64_t(ez) * q + k, q, sl.Ez, sl.ez0, sl.ez1);
    double acc = 0.0;
    for (int c = 0; c < cz.n; ++c)
      for (int b = 0; b < cy.n; ++b)
        for (int a = 0; a < cx.n; ++a) {
          const int64_t e2 = cx.e[a] + int64_t(sl.Ex) * (cy.e[b] + int64_t(sl.Ey) * (cz.e[c] - sl.ez0));
          acc += in[e2 * nloc + cx.loc[a] + nd * (cy.loc[b] + nd * cz.loc[c])];
        }
    out[t] = acc;
  }
}

__global__ void k_mask(const Slab sl, double* __restrict__ v) {
  const int64_t total = sl.n_local();
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t x = t % sl.Nx, y = (t / sl.Nx) % sl.Ny, z = sl.zlo + t / (sl.Nx * sl.Ny);
    if (sl.masked(x, y, z)) v[t] = 0.0;
  }
}

__global__ void k_invert_masked(const Slab sl, const double* __restrict__ in, double* __restrict__ out) {
  const int64_t total = sl.n_local();
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t x = t % sl.Nx, y = (t / sl.Nx) % sl.Ny, z = sl.zlo + t / (sl.Nx * sl.Ny);
    const double d = in[t];
    out[t] = (sl.masked(x, y, z) || d == 0.0) ? 0.0 : 1.0 / d;
  }
}

// ------------------------------------------------------------------------ reductions
// Deterministic: per-block partial sums in fixed order, the last block to finish reduces the
// partials in block order.
template <int K>
struct DotArgs {
  const double* a[K];
  const double* b[K];
};

template <int K>
__global__ void __launch_bounds__(256) k_dots(const DotArgs<K> args, int64_t n, double* __restrict__ out,
                                               double* __restrict__ partial, unsigned* __restrict__ counter) {
  __shared__ double sred[K * 8];
  __shared__ bool last;
  double v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = 0.0;
  for (int64_t t = int64_t(blockIdx.x) * 256 + threadIdx.x; t < n; t += int64_t(gridDim.x) * 256) {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = fma(args.a[k][t], args.b[k][t], v[k]);
  }
  block_sum<K, 256>(v, sred);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) partial[blockIdx.x * K + k] = v[k];
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();  // the whole last block reduces the partials (fixed strided shape)
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = 0.0;
  for (unsigned bidx = threadIdx.x; bidx < gridDim.x; bidx += 256)
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] += __ldcg(&partial[bidx * K + k]);
  block_sum<K, 256>(v, sred);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = v[k];
    *counter = 0u;
  }
}

template <class F>
__global__ void k_foreach(int64_t n, F f) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) f(t);
}

template <class F>
int64_t foreach(int64_t n, cudaStream_t s, F f) {
  if (n <= 0) return 0;
  k_foreach<<<grid1d(n, 256), 256, 0, s>>>(n, f);
  SB_LAUNCH_CHECK();
  return 1;
}

}  // namespace

// ------------------------------------------------------------------------ launchers
int64_t launch_geom(const Slab& sl, const double* X, double* geom, double* massw, unsigned long long* bad,
                    cudaStream_t s) {
  const int nd = sl.q + 1;
  const int64_t total = sl.elems() * nd * nd * nd;
  if (total == 0) return 0;
  const int blocks = int((total + 255) / 256);
  const auto& g = gll(sl.q);
#define SB_GEOM(ND)                                                              \
  case ND: {                                                                     \
    W1<ND> w;                                                                    \
    for (int t = 0; t < ND; ++t) w.w[t] = g.weights[t];                          \
    k_geom<ND><<<blocks, 256, 0, s>>>(sl, dmat<ND>(sl.q), w, X, geom, massw, bad); \
    break;                                                                       \
  }
  switch (nd) {
    SB_GEOM(2) SB_GEOM(3) SB_GEOM(4) SB_GEOM(5) SB_GEOM(6) SB_GEOM(7) SB_GEOM(8) SB_GEOM(9) SB_GEOM(10)
    default: invalid("SemSpace: device kernels support orders 1..9");
  }
#undef SB_GEOM
  SB_LAUNCH_CHECK();
  return 1;
}

int64_t launch_ax(const Slab& sl, const double* u, const double* geom, const AxSync& sy, Epi epi, const EpiArgs& a,
                  cudaStream_t s) {
  switch (epi) {
    case Epi::Write: return ax_dispatch<false>(sl, u, geom, sy, nullptr, EWrite{a.w}, s);
    case Epi::Residual: return ax_dispatch<false>(sl, u, geom, sy, nullptr, EResidual{a.w, a.b}, s);
    case Epi::ChebJacStep:
      return ax_dispatch<false>(sl, u, geom, sy, nullptr, EChebJacStep{a.x, a.r, a.d, a.inv, a.c1, a.c2}, s);
    case Epi::ChebJacInit:
      return ax_dispatch<false>(sl, u, geom, sy, nullptr, EChebJacInit{a.r, a.d, a.b, a.inv, a.c1}, s);
  }
  return 0;
}

template <int ND>
int64_t ax_g32_split(const Slab& sl, const double* u, const float* g, const AxSync& sy, Epi epi, const EpiArgs& a,
                     cudaStream_t s) {
  switch (epi) {
    case Epi::Write: return ax_dispatch_nd<ND, false>(sl, u, g, sy, nullptr, EWrite{a.w}, s);
    case Epi::Residual: return ax_dispatch_nd<ND, false>(sl, u, g, sy, nullptr, EResidual{a.w, a.b}, s);
    case Epi::ChebJacStep:
      return ax_dispatch_nd<ND, false>(sl, u, g, sy, nullptr, EChebJacStep{a.x, a.r, a.d, a.inv, a.c1, a.c2}, s);
    case Epi::ChebJacInit:
      return ax_dispatch_nd<ND, false>(sl, u, g, sy, nullptr, EChebJacInit{a.r, a.d, a.b, a.inv, a.c1}, s);
  }
  return 0;
}

bool ax_g32_supported(int q) { return q == 7 || (q >= 1 && q + 1 <= SEMLAB_AX_SPLIT_ND); }

int64_t launch_ax_g32(const Slab& sl, const double* u, const float* geom32, const AxSync& sy, Epi epi,
                      const EpiArgs& a, cudaStream_t s) {
  if (!ax_g32_supported(sl.q))
    invalid("launch_ax_g32: FP32 geometry is implemented for order 7 and the split-path orders");
  if (sl.q != 7) {
    switch (sl.q + 1) {
      case 2: return ax_g32_split<2>(sl, u, geom32, sy, epi, a, s);
      case 3: return ax_g32_split<3>(sl, u, geom32, sy, epi, a, s);
      case 4: return ax_g32_split<4>(sl, u, geom32, sy, epi, a, s);
      case 5: return ax_g32_split<5>(sl, u, geom32, sy, epi, a, s);
      case 6: return ax_g32_split<6>(sl, u, geom32, sy, epi, a, s);
      default: invalid("launch_ax_g32: unsupported order");
    }
  }
  switch (epi) {
    case Epi::Write: return axw_launch(sl, u, geom32, sy, EWrite{a.w}, s);
    case Epi::Residual: return axw_launch(sl, u, geom32, sy, EResidual{a.w, a.b}, s);
    case Epi::ChebJacStep:
      return axw_launch(sl, u, geom32, sy, EChebJacStep{a.x, a.r, a.d, a.inv, a.c1, a.c2}, s);
    case Epi::ChebJacInit: return axw_launch(sl, u, geom32, sy, EChebJacInit{a.r, a.d, a.b, a.inv, a.c1}, s);
  }
  return 0;
}

int64_t launch_ax_local(const Slab& sl, const double* uloc, const double* geom, double* out, cudaStream_t s) {
  return ax_dispatch<true>(sl, uloc, geom, AxSync{}, out, EWrite{nullptr}, s);
}

int64_t launch_local_diag(const Slab& sl, const double* geom, double* out, cudaStream_t s) {
  const int nd = sl.q + 1;
  const int64_t total = sl.elems() * nd * nd * nd;
  if (total == 0) return 0;
  const int blocks = int((total + 255) / 256);
#define SB_DIAG(ND) \
  case ND: k_local_diag<ND><<<blocks, 256, 0, s>>>(sl, dmat<ND>(sl.q), geom, out); break;
  switch (nd) {
    SB_DIAG(2) SB_DIAG(3) SB_DIAG(4) SB_DIAG(5) SB_DIAG(6) SB_DIAG(7) SB_DIAG(8) SB_DIAG(9) SB_DIAG(10)
    default: invalid("SemSpace: device kernels support orders 1..9");
  }
#undef SB_DIAG
  SB_LAUNCH_CHECK();
  return 1;
}

int64_t launch_gather(const Slab& sl, const double* loc, double* glob, cudaStream_t s) {
  const int64_t total = sl.Nx * sl.Ny * (int64_t(sl.ez1 - sl.ez0) * sl.q + 1);
  k_gather<<<grid1d(total, 256), 256, 0, s>>>(sl, loc, glob);
  SB_LAUNCH_CHECK();
  return 1;
}
int64_t launch_scatter(const Slab& sl, const double* glob, double* loc, cudaStream_t s) {
  const int64_t total = sl.elems() * int64_t(sl.q + 1) * (sl.q + 1) * (sl.q + 1);
  k_scatter<<<grid1d(total, 256), 256, 0, s>>>(sl, glob, loc);
  SB_LAUNCH_CHECK();
  return 1;
}
int64_t launch_qqt(const Slab& sl, const double* in, double* out, cudaStream_t s) {
  const int64_t total = sl.elems() * int64_t(sl.q + 1) * (sl.q + 1) * (sl.q + 1);
  k_qqt<<<grid1d(total, 256), 256, 0, s>>>(sl, in, out);
  SB_LAUNCH_CHECK();
  return 1;
}
int64_t launch_mask(const Slab& sl, double* v, cudaStream_t s) {
  k_mask<<<grid1d(sl.n_local(), 256), 256, 0, s>>>(sl, v);
  SB_LAUNCH_CHECK();
  return 1;
}
int64_t launch_invert_masked(const Slab& sl, const double* in, double* out, cudaStream_t s) {
  k_invert_masked<<<grid1d(sl.n_local(), 256), 256, 0, s>>>(sl, in, out);
  SB_LAUNCH_CHECK();
  return 1;
}

int64_t launch_fill(double* d, int64_t n, double v, cudaStream_t s) {
  return foreach(n, s, [=] __device__(int64_t t) { d[t] = v; });
}
int64_t launch_copy(double* dst, const double* src, int64_t n, cudaStream_t s) {
  if (n > 0) SB_CUDA(cudaMemcpyAsync(dst, src, size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
  return 0;
}
int64_t launch_to_f32(const double* in, float* out, int64_t n, cudaStream_t s) {
  return foreach(n, s, [=] __device__(int64_t t) { out[t] = float(in[t]); });
}

int64_t launch_axpby(double* y, double a, const double* x, double b, int64_t n, cudaStream_t s) {
  return foreach(n, s, [=] __device__(int64_t t) { y[t] = a * x[t] + b * y[t]; });
}
int64_t launch_mul(double* y, const double* a, const double* x, int64_t n, cudaStream_t s) {
  return foreach(n, s, [=] __device__(int64_t t) { y[t] = a[t] * x[t]; });
}
int64_t launch_sub(double* y, const double* a, const double* b, int64_t n, cudaStream_t s) {
  return foreach(n, s, [=] __device__(int64_t t) { y[t] = a[t] - b[t]; });
}
int64_t launch_add_planes(double* y, const double* a, const double* b, int64_t n, cudaStream_t s) {
  return foreach(n, s, [=] __device__(int64_t t) { y[t] = a[t] + b[t]; });
}
int64_t launch_div(double* y, const double* x, double a, int64_t n, cudaStream_t s) {
  return foreach(n, s, [=] __device__(int64_t t) { y[t] = x[t] / a; });
}
int64_t launch_cheb_init(double* r, double* d, double theta, int64_t n, cudaStream_t s) {
  return foreach(n, s, [=] __device__(int64_t t) { d[t] = r[t] / theta; });
}
int64_t launch_cheb_step(double* x, double* r, double* d, const double* sad, double c1, double c2, int64_t n,
                         cudaStream_t s) {
  return foreach(n, s, [=] __device__(int64_t t) {
    const double dg = d[t];
    x[t] += dg;
    const double rg = r[t] - sad[t];
    r[t] = rg;
    d[t] = c1 * dg + c2 * rg;
  });
}
int64_t launch_cheb_jac_zero_init(const double* b, const double* inv, double* r, double* d, double theta, int64_t n,
                                  cudaStream_t s) {
  return foreach(n, s, [=] __device__(int64_t t) {
    const double rg = inv[t] * b[t];
    r[t] = rg;
    d[t] = rg / theta;
  });
}

int64_t launch_dots(int K, const double* const* a, const double* const* b, int64_t n, double* out,
                    const DotScratch& ws, cudaStream_t s) {
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>(kMaxDotBlocks, (n + 255) / 256)));
#define SB_DOTS(KK)                                                                             \
  case KK: {                                                                                    \
    DotArgs<KK> d;                                                                              \
    for (int k = 0; k < KK; ++k) { d.a[k] = a[k]; d.b[k] = b[k]; }                              \
    k_dots<KK><<<blocks, 256, 0, s>>>(d, n, out, ws.partial, ws.counter);                       \
    break;                                                                                      \
  }
  switch (K) {
    SB_DOTS(1) SB_DOTS(2) SB_DOTS(3) SB_DOTS(4)
    default: invalid("launch_dots: K must be 1..4");
  }
#undef SB_DOTS
  SB_LAUNCH_CHECK();
  return 1;
}

}  // namespace sb
