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
#include <cstdlib>

#include "device.cuh"
#include "host_math.hpp"
#include "kernels.hpp"

#ifndef SEMLAB_AX_BATCH_EPI
#define SEMLAB_AX_BATCH_EPI 1  // owner epilogue: issue all vector loads before the stores
#endif
#ifndef SEMLAB_AXP_MINB
#define SEMLAB_AXP_MINB 8  // resident CTAs per SM the persistent Ax is register-capped for
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
// SEMLAB_AX_PERSISTENT=0 selects the one-CTA-per-element kernel (kept for A/B measurement).
bool ax_persistent() {
  static const bool on = [] {
    const char* e = std::getenv("SEMLAB_AX_PERSISTENT");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int ND>
constexpr int ax_min_blocks() {  // occupancy target: caps registers so ~20 warps/SM stay resident
  return ND >= 8 ? 10 : 16;
}

template <int ND, int EPB, bool LOCAL, class EpiT>
__global__ void __launch_bounds__(EPB* ND* ND, ax_min_blocks<ND>())
    k_ax(const Slab sl, const DMat<ND> Dm, const double* __restrict__ u, const double* __restrict__ geom,
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
    if (LOCAL) {
      t = blockIdx.x;
    } else {
      t = int(atomicAdd(ticket, 1u));
      if (t == ngroups - 1) atomicExch(ticket, 0u);  // every ticket of this launch is taken
    }
    s_grp = t;
  }
  for (int t = tid; t < ND2; t += NT) s_D[t] = Dm.d[t];
  __syncthreads();

  const int64_t nE = sl.elems();
  const int64_t e0 = int64_t(s_grp) * EPB;
  const int ne = int(nE - e0 < EPB ? nE - e0 : EPB);
  {  // stream the group's geometry (contiguous, 48 B/node) into L2 while u is loaded and
     // differentiated; phase 2 then reads it at L2 latency without holding shared memory
    const char* gbase = reinterpret_cast<const char*>(geom + e0 * 6 * NLOC);
    const int lines = (ne * 6 * NLOC * int(sizeof(double)) + 127) / 128;
    for (int l = tid; l < lines; l += NT) asm volatile("prefetch.global.L2 [%0];" ::"l"(gbase + size_t(l) * 128));
  }
  if (tid == 0 && !LOCAL) s_epoch = *reinterpret_cast<volatile unsigned*>(&flags[e0]);

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
    const double raw = LOCAL ? __ldg(&u[el * NLOC + k * ND2 + ij]) : __ldg(&u[sl.lidx(x, y, zb + k)]);
    const double v = (!active || (!LOCAL && sl.masked(x, y, zb + k))) ? 0.0 : raw;
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
  const double* gg = geom + el * 6 * NLOC + ij;
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    // per-layer guarded loads: keeps the 6*ND geometry loads from all being hoisted at once
    // (that spills at the 96-register occupancy target); the geometry sits in L2 (prefetched)
    const int node = k * ND2;
    double g0 = 0, g1 = 0, g2 = 0, g3 = 0, g4 = 0, g5 = 0;
    if (active) {
      g0 = __ldcs(gg + 0 * NLOC + node);
      g1 = __ldcs(gg + 1 * NLOC + node);
      g2 = __ldcs(gg + 2 * NLOC + node);
      g3 = __ldcs(gg + 3 * NLOC + node);
      g4 = __ldcs(gg + 4 * NLOC + node);
      g5 = __ldcs(gg + 5 * NLOC + node);
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

  if (LOCAL) {
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
// Same arithmetic and summation order as k_ax, restructured so no CTA idles on a neighbour:
// a resident CTA loops over dynamic tickets; for ticket t it computes the element, deposits
// the non-owned nodes, writes the owned nodes that have no lower contributor (the 6^3 interior
// of a p=7 element) right away and publishes its counter; only then does it finish ticket t-1's
// owned face nodes, whose lower neighbours have long been published. The next ticket is taken,
// and its geometry prefetched to L2, before the current element is computed.
template <int ND, class EpiT>
__global__ void __launch_bounds__(ND* ND, SEMLAB_AXP_MINB)
    k_axp(const Slab sl, const DMat<ND> Dm, const double* __restrict__ u, const double* __restrict__ geom,
          double* __restrict__ dep, unsigned* __restrict__ flags, unsigned* __restrict__ ticket, int total_tickets,
          const EpiT epi) {
  constexpr int ND2 = ND * ND, NLOC = ND2 * ND, NT = ND2;
  constexpr int q = ND - 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* s_a = reinterpret_cast<double*>(smem_raw);
  double* s_b = s_a + NLOC;
  double* s_D = s_b + NLOC;
  double* s_out[2] = {s_D + ND2, s_D + ND2 + NLOC};  // per-element results awaiting completion
  __shared__ int s_tk[2];
  __shared__ unsigned s_epoch;
  const int tid = threadIdx.x;
  const int ij = tid, i = ij % ND, j = ij / ND;
  const int64_t nE = sl.elems();
  const int64_t LX = 1, LY = sl.Ex, LZ = int64_t(sl.Ex) * sl.Ey;
  for (int t = tid; t < ND2; t += NT) s_D[t] = Dm.d[t];
  if (tid == 0) {
    const int t0 = int(atomicAdd(ticket, 1u));
    if (t0 == total_tickets - 1) atomicExch(ticket, 0u);
    s_tk[0] = t0;
    if (t0 < nE) s_epoch = *reinterpret_cast<volatile unsigned*>(&flags[t0]);
  }
  __syncthreads();
  const unsigned target = s_epoch + 1u;  // every element's counter equals s_epoch at launch
  int64_t prev = -1;
  int buf = 0;

  auto coords = [&](int64_t el, int& ex, int& ey, int& ez) {
    ex = int(el % sl.Ex);
    ey = int((el / sl.Ex) % sl.Ey);
    ez = sl.ez0 + int(el / LZ);
  };
  // owned node (i,j,k) of element (ex,ey,ez) has no contributor below it
  auto finish_prev = [&](int64_t pe, const double* pout) {
    int ex, ey, ez;
    coords(pe, ex, ey, ez);
    if (tid < 7) {  // wait for the <= 7 lower neighbours of pe (released long ago, normally)
      const int a = (tid + 1) & 1, b = ((tid + 1) >> 1) & 1, c = ((tid + 1) >> 2) & 1;
      if ((!a || ex > 0) && (!b || ey > 0) && (!c || ez > sl.ez0)) {
        const int64_t nb = pe - a * LX - b * LY - c * LZ;
        while (ld_relaxed(&flags[nb]) < target) {
        }
      }
    }
    __syncthreads();
    const bool hx = (i == 0 && ex > 0), hy = (j == 0 && ey > 0), hz = (ez > sl.ez0);
    const bool ownx = (i < q) || (ex == sl.Ex - 1), owny = (j < q) || (ey == sl.Ey - 1);
    const bool topz = (ez == sl.ez1 - 1);
    const int64_t x = int64_t(ex) * q + i, y = int64_t(ey) * q + j, zb = int64_t(ez) * q;
    const double* dbase = dep + pe * NLOC + ij;
    const bool own0 = ownx && owny && hz;
    const double cz = ldcg_pred(dbase - LZ * NLOC + q * ND2, own0);
    const double cxz = ldcg_pred(dbase - (LZ + LX) * NLOC + q * ND2 + q, own0 && hx);
    const double cyz = ldcg_pred(dbase - (LZ + LY) * NLOC + q * ND2 + q * ND, own0 && hy);
    const double cxyz = ldcg_pred(dbase - (LZ + LY + LX) * NLOC + q * ND2 + q * ND + q, own0 && hx && hy);
    constexpr int KH = (ND + 1) / 2;
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
        acc += pout[k * ND2 + ij];
        const int64_t z = zb + k;
        epi(sl.lidx(x, y, z), sl.masked(x, y, z) ? 0.0 : acc);
      }
    }
  };

  while (true) {
    const int64_t el = s_tk[buf];
    if (el >= nE) break;
    if (tid == 0) {  // next ticket now, so its latency hides behind this element
      const int tn = int(atomicAdd(ticket, 1u));
      if (tn == total_tickets - 1) atomicExch(ticket, 0u);
      s_tk[buf ^ 1] = tn;
    }
    {  // this element's geometry -> L2
      const char* gbase = reinterpret_cast<const char*>(geom + el * 6 * NLOC);
      constexpr int lines = (6 * NLOC * int(sizeof(double)) + 127) / 128;
      for (int l = tid; l < lines; l += NT) asm volatile("prefetch.global.L2 [%0];" ::"l"(gbase + size_t(l) * 128));
    }
    int ex, ey, ez;
    coords(el, ex, ey, ez);
    const int64_t x = int64_t(ex) * q + i, y = int64_t(ey) * q + j, zb = int64_t(ez) * q;
    double ureg[ND];
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      const double raw = __ldg(&u[sl.lidx(x, y, zb + k)]);
      const double v = sl.masked(x, y, zb + k) ? 0.0 : raw;
      ureg[k] = v;
      s_a[k * ND2 + ij] = v;
    }
    __syncthreads();
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
    const double* gg = geom + el * 6 * NLOC + ij;
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      const int node = k * ND2;
      double g0, g1, g2, g3, g4, g5;
      if (el >= 0) {  // always true: keeps per-layer load batches (bounded registers)
        g0 = __ldcs(gg + 0 * NLOC + node);
        g1 = __ldcs(gg + 1 * NLOC + node);
        g2 = __ldcs(gg + 2 * NLOC + node);
        g3 = __ldcs(gg + 3 * NLOC + node);
        g4 = __ldcs(gg + 4 * NLOC + node);
        g5 = __ldcs(gg + 5 * NLOC + node);
      } else {
        g0 = g1 = g2 = g3 = g4 = g5 = 0.0;
      }
      const double r = ur[k], s = us[k], t = ut[k];
      ur[k] = g0 * r + g1 * s + g2 * t;
      us[k] = g1 * r + g3 * s + g4 * t;
      ut[k] = g2 * r + g4 * s + g5 * t;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      s_a[k * ND2 + ij] = ur[k];
      s_b[k * ND2 + ij] = us[k];
    }
    __syncthreads();
    double* cur_out = s_out[buf];
    {
      double DiT[ND], DjT[ND];
#pragma unroll
      for (int m = 0; m < ND; ++m) {
        DiT[m] = s_D[m + ND * i];
        DjT[m] = s_D[m + ND * j];
      }
      const bool ownx = (i < q) || (ex == sl.Ex - 1), owny = (j < q) || (ey == sl.Ey - 1);
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
      // loads first, then the stores); face-owned nodes wait in smem; the rest are deposited
      typename EpiT::In in[ND];
#if SEMLAB_AX_BATCH_EPI
#pragma unroll
      for (int k = 0; k < ND; ++k) {
        const bool own = ownx && owny && (k < q || topz);
        if (own && !(hx || hy || (k == 0 && hz))) in[k] = epi.load(sl.lidx(x, y, zb + k));
      }
#endif
#pragma unroll
      for (int k = 0; k < ND; ++k) {
        const bool own = ownx && owny && (k < q || topz);
        if (!own) {
          dep[el * NLOC + k * ND2 + ij] = outk[k];
        } else if (hx || hy || (k == 0 && hz)) {
          cur_out[k * ND2 + ij] = outk[k];  // owned face node: summed once the neighbours are in
        } else {
          const int64_t z = zb + k;
#if !SEMLAB_AX_BATCH_EPI
          in[k] = epi.load(sl.lidx(x, y, z));
#endif
          epi.store(sl.lidx(x, y, z), in[k], sl.masked(x, y, z) ? 0.0 : outk[k]);
        }
      }
    }
    __syncthreads();
    if (tid == 0) st_release(&flags[el], target);
    if (prev >= 0) finish_prev(prev, s_out[buf ^ 1]);
    prev = el;
    buf ^= 1;
    __syncthreads();
  }
  if (prev >= 0) finish_prev(prev, s_out[buf ^ 1]);
}

template <int ND, class EpiT>
int64_t axp_launch(const Slab& sl, const double* u, const double* geom, const AxSync& sy, const EpiT& epi,
                   cudaStream_t s) {
  constexpr int NLOC = ND * ND * ND;
  const int64_t nE = sl.elems();
  if (nE == 0) return 0;
  const size_t smem = (size_t(4) * NLOC + ND * ND) * sizeof(double);
  auto kern = k_axp<ND, EpiT>;
  static int nctas = 0;  // resident CTAs: occupancy x SMs (per instantiation)
  if (nctas == 0) {
    SB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0, dev = 0, sms = 0;
    SB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, ND * ND, smem));
    SB_CUDA(cudaGetDevice(&dev));
    SB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    nctas = std::max(1, per_sm * sms);
  }
  const int grid = int(std::min<int64_t>(nctas, nE));
  kern<<<grid, ND * ND, smem, s>>>(sl, dmat<ND>(sl.q), u, geom, sy.dep, sy.flags, sy.ticket, int(nE + grid), epi);
  SB_LAUNCH_CHECK();
  return 1;
}

template <int ND, bool LOCAL, class EpiT>
int64_t ax_dispatch_nd(const Slab& sl, const double* u, const double* geom, const AxSync& sy, double* out_local,
                       const EpiT& epi, cudaStream_t s) {
  if constexpr (!LOCAL && ND >= 8) {
    if (ax_persistent()) return axp_launch<ND>(sl, u, geom, sy, epi, s);
  }
  constexpr int EPB = epb<ND>();
  constexpr int NLOC = ND * ND * ND;
  const int64_t nE = sl.elems();
  if (nE == 0) return 0;
  const int ngroups = int((nE + EPB - 1) / EPB);
  const size_t smem = (size_t(EPB) * 2 * NLOC + ND * ND) * sizeof(double);
  auto kern = k_ax<ND, EPB, LOCAL, EpiT>;
  static bool configured = false;  // per instantiation
  if (!configured) {
    SB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    configured = true;
  }
  kern<<<ngroups, EPB * ND * ND, smem, s>>>(sl, dmat<ND>(sl.q), u, geom, sy.dep, sy.flags, sy.ticket, ngroups,
                                           out_local, epi);
  SB_LAUNCH_CHECK();
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
