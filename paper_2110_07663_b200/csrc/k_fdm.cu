// Overlapping Schwarz smoother kernels (sm_100a), replacing SchwarzSmoother::apply and
// fdm_solve (schwarz.cpp:228-289).
//
// Several elements per CTA (order+3 = P per direction; boundary boxes are smaller and padded
// with zero S rows). Each element's extended box is extracted from the global lattice vector
// straight into shared memory (sites outside the element core in more than one direction are
// zero-filled, schwarz.cpp:255-265). The three forward transforms S_x^T, S_y^T, S_z^T, the
// scaling by inv_D = 1/(lx_i + ly_j + lz_k) (recomputed from the 3P eigenvalues instead of
// streaming the P^3 table, schwarz.cpp:92-108) and the backward transforms run as line passes:
// every thread keeps R lines of the box in registers and reads S as 2-wide vectors (one shared
// load feeds 2R FMAs), so the passes are FMA-bound rather than shared-memory-bound.
// RAS: the element writes exactly the lattice nodes it owns (lowest element whose core holds
// the node, schwarz.cpp:114-127) — a race-free owner write that carries the whole Chebyshev
// vector update. ASM: per-element boxes go to a buffer and every node sums the boxes covering it
// in ascending element id (the reference's order) times 1/count (schwarz.cpp:269-287).
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_set>

#include "device.cuh"
#include "kernels_fdm.hpp"

#ifndef SEMLAB_RASW_GATHER_UNROLL
#define SEMLAB_RASW_GATHER_UNROLL 2  // z-columns of the box gathered per lane per batch
#endif
#ifndef SEMLAB_RASW_OWNER_U
#define SEMLAB_RASW_OWNER_U 4  // owned sites per lane per batch of the owner write
#endif
constexpr int kGatherUnroll = SEMLAB_RASW_GATHER_UNROLL;
#ifndef SEMLAB_RASW_MINB
#define SEMLAB_RASW_MINB 5  // resident 4-warp CTAs per SM the warp-per-element RAS is register-capped for
#endif

#ifndef SEMLAB_RAS_SMALLP_MINB
#define SEMLAB_RAS_SMALLP_MINB 7  // p = 3 level (P = 6): 7 CTAs/SM of the CTA RAS kernel (3% faster than 5 despite 12 B of spills)
#endif
#ifndef SEMLAB_RASW_MINP
#define SEMLAB_RASW_MINP 8  // warp-per-element RAS from box size P = p + 3 >= this (p >= 3)
#endif
#ifndef SEMLAB_RASW_FFMA2
#define SEMLAB_RASW_FFMA2 1  // packed FP32 FMA (sm_100 FFMA2) in the FDM line passes
#endif

namespace sb {

namespace {

struct Box1D {  // extended-box geometry of one element along one axis (schwarz.cpp:155-169)
  int n, lo, gl, gr, own_lo, own_hi;  // own_*: box indices this element owns (RAS, inclusive)
};

__device__ __forceinline__ Box1D box1d(int e_d, int E_d, int q, bool dirichlet) {
  Box1D b;
  const bool left_int = e_d > 0;
  const bool right_int = e_d < E_d - 1;
  const int i0 = (!left_int && dirichlet) ? 1 : 0;
  const int i1 = (!right_int && dirichlet) ? q - 1 : q;
  b.gl = left_int ? 1 : 0;
  b.gr = right_int ? 1 : 0;
  b.n = (i1 - i0 + 1) + b.gl + b.gr;
  b.lo = e_d * q + i0 - b.gl;
  const int first = left_int ? 1 : i0;  // the left face node is owned by the left neighbour
  b.own_lo = first - i0 + b.gl;
  b.own_hi = i1 - i0 + b.gl;
  return b;
}

__device__ __forceinline__ bool ghost(const Box1D& b, int a) { return (b.gl && a == 0) || (b.gr && a == b.n - 1); }

template <int P, class T>
struct Shape {
  static constexpr int R = sizeof(T) == 4 ? 4 : 2;  // lines per thread
  static constexpr int P2 = P * P, P3 = P2 * P;
  static constexpr int TPE = (P2 + R - 1) / R;  // threads per element
  static constexpr int NT = 128;
  static constexpr int EPC = NT / TPE;  // elements per CTA
  static constexpr int SPE = 2 * P3 + 3 * P2 + 3 * P + 2;  // smem T per element (even, 8B aligned)
  static constexpr size_t smem() { return size_t(EPC) * SPE * sizeof(T); }
};

// 1/s for the FP32 smoother: hardware approximation plus one Newton step (within 1 ulp of the
// rounded quotient; s = lx + ly + lz > 0 is a normal number), three instructions instead of the
// special-case-checking IEEE sequence
__device__ __forceinline__ float rcp(float s) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(s));
  return fmaf(r, fmaf(-s, r, 1.0f), r);
}
__device__ __forceinline__ double rcp(double s) { return 1.0 / s; }

// One line pass along axis AX: for the thread's R lines, out = M^T in (FWD) or M in (!FWD);
// MID: forward z, scale by inv_D, backward z in registers.
template <int P, class T, int AX, int KIND /*0 fwd, 1 bwd, 2 mid*/>
__device__ __forceinline__ void line_pass(const T* __restrict__ src, T* __restrict__ dst, const T* __restrict__ S,
                                          const T* __restrict__ L, int ti) {
  using Sh = Shape<P, T>;
  constexpr int R = Sh::R, P2 = Sh::P2, TPE = Sh::TPE;
  T in[R][P], out[R][P];
  int base[R];
  constexpr int stride = AX == 0 ? 1 : (AX == 1 ? P : P2);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int l = ti + TPE * r;
    const int u = l % P, v = l / P;
    base[r] = AX == 0 ? (v * P2 + u * P) : (AX == 1 ? (v * P2 + u) : (v * P + u));
    const bool ok = l < P2;
#pragma unroll
    for (int m = 0; m < P; ++m) in[r][m] = ok ? src[base[r] + m * stride] : T(0);
  }
  auto fwd = [&](const T* M, T(&x)[R][P], T(&y)[R][P]) {  // y[o] = sum_a M(a,o) x[a]
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int o = 0; o < P; ++o) y[r][o] = T(0);
#pragma unroll
    for (int a = 0; a < P; ++a) {
      if constexpr (P % 2 == 0 && sizeof(T) == 4 && SEMLAB_RASW_FFMA2) {
        // packed FP32 (FFMA2): the (o, o+1) output pair shares x_a; same per-output order
#pragma unroll
        for (int o = 0; o < P; o += 2) {
          const float2 s2 = *reinterpret_cast<const float2*>(M + a * P + o);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const float2 acc = __ffma2_rn(s2, make_float2(x[r][a], x[r][a]), make_float2(y[r][o], y[r][o + 1]));
            y[r][o] = acc.x;
            y[r][o + 1] = acc.y;
          }
        }
      } else if constexpr (P % 2 == 0) {
#pragma unroll
        for (int o = 0; o < P; o += 2) {
          T s0, s1;
          if constexpr (sizeof(T) == 4) {
            const float2 s = *reinterpret_cast<const float2*>(M + a * P + o);
            s0 = s.x;
            s1 = s.y;
          } else {
            const double2 s = *reinterpret_cast<const double2*>(M + a * P + o);
            s0 = s.x;
            s1 = s.y;
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {
            y[r][o] = fma(s0, x[r][a], y[r][o]);
            y[r][o + 1] = fma(s1, x[r][a], y[r][o + 1]);
          }
        }
      } else {
#pragma unroll
        for (int o = 0; o < P; ++o) {
          const T s = M[a * P + o];
#pragma unroll
          for (int r = 0; r < R; ++r) y[r][o] = fma(s, x[r][a], y[r][o]);
        }
      }
    }
  };
  auto bwd = [&](const T* M, T(&x)[R][P], T(&y)[R][P]) {  // y[a] = sum_o M(a,o) x[o]
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int a = 0; a < P; ++a) y[r][a] = T(0);
#pragma unroll
    for (int a = 0; a < P; ++a) {
      if constexpr (P % 2 == 0 && sizeof(T) == 4 && SEMLAB_RASW_FFMA2) {
        // packed FP32: even and odd o accumulate in the two halves, summed at the end (the
        // order of k_rasw's backward pass)
        float2 a2[R];
#pragma unroll
        for (int r = 0; r < R; ++r) a2[r] = make_float2(0.f, 0.f);
#pragma unroll
        for (int o = 0; o < P; o += 2) {
          const float2 s2 = *reinterpret_cast<const float2*>(M + a * P + o);
#pragma unroll
          for (int r = 0; r < R; ++r) a2[r] = __ffma2_rn(s2, make_float2(x[r][o], x[r][o + 1]), a2[r]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) y[r][a] = a2[r].x + a2[r].y;
      } else if constexpr (P % 2 == 0) {
#pragma unroll
        for (int o = 0; o < P; o += 2) {
          T s0, s1;
          if constexpr (sizeof(T) == 4) {
            const float2 s = *reinterpret_cast<const float2*>(M + a * P + o);
            s0 = s.x;
            s1 = s.y;
          } else {
            const double2 s = *reinterpret_cast<const double2*>(M + a * P + o);
            s0 = s.x;
            s1 = s.y;
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {
            y[r][a] = fma(s0, x[r][o], y[r][a]);
            y[r][a] = fma(s1, x[r][o + 1], y[r][a]);
          }
        }
      } else {
#pragma unroll
        for (int o = 0; o < P; ++o) {
          const T s = M[a * P + o];
#pragma unroll
          for (int r = 0; r < R; ++r) y[r][a] = fma(s, x[r][o], y[r][a]);
        }
      }
    }
  };
  if (KIND == 0) {
    fwd(S, in, out);
  } else if (KIND == 1) {
    bwd(S, in, out);
  } else {
    fwd(S, in, out);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int l = ti + TPE * r;
      const int a = l % P, b = (l / P) % P;
      const T lab = L[0 * P + a] + L[1 * P + b];
#pragma unroll
      for (int c = 0; c < P; ++c) out[r][c] = out[r][c] * rcp(lab + L[2 * P + c]);
    }
    bwd(S, out, in);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int m = 0; m < P; ++m) out[r][m] = in[r][m];
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int l = ti + TPE * r;
    if (l < P2)
#pragma unroll
      for (int m = 0; m < P; ++m) dst[base[r] + m * stride] = out[r][m];
  }
}

// Block of EPC elements: load factors + boxes (from the lattice vector or from a box array),
// run the five line passes. Result left in the element's tmp buffer.
template <int P, class T, bool FROM_BOXES>
__device__ __forceinline__ void fdm_block(const Slab& sl, const T* __restrict__ S, const T* __restrict__ L,
                                          const double* __restrict__ src, int64_t e_first, int64_t nE, T* smem,
                                          Box1D (*bx)[3]) {
  using Sh = Shape<P, T>;
  constexpr int P2 = Sh::P2, P3 = Sh::P3, EPC = Sh::EPC, SPE = Sh::SPE, TPE = Sh::TPE;
  const int tid = threadIdx.x;
  if (!FROM_BOXES && tid < EPC) {
    const int64_t el = e_first + tid;
    if (el < nE) {
      const int ex = int(el % sl.Ex), ey = int((el / sl.Ex) % sl.Ey);
      const int ez = sl.ez0 + int(el / (int64_t(sl.Ex) * sl.Ey));
      const bool dir = sl.dirichlet != 0;
      bx[tid][0] = box1d(ex, sl.Ex, sl.q, dir);
      bx[tid][1] = box1d(ey, sl.Ey, sl.q, dir);
      bx[tid][2] = box1d(ez, sl.Ez, sl.q, dir);
    }
  }
  // factors: S (3 P^2) and lambda (3 P) of each element; all loads issued before the stores
  {
    constexpr int NF = 3 * P2 + 3 * P, ITER = (EPC * NF + Sh::NT - 1) / Sh::NT;
    T v[ITER];
#pragma unroll
    for (int it = 0; it < ITER; ++it) {
      const int t = tid + it * Sh::NT;
      const int e = t / NF, w = t % NF;
      const int64_t el = e_first + e;
      const bool ok = t < EPC * NF && el < nE;
      v[it] = !ok ? T(0) : (w < 3 * P2 ? __ldg(S + el * 3 * P2 + w) : __ldg(L + el * 3 * P + (w - 3 * P2)));
    }
#pragma unroll
    for (int it = 0; it < ITER; ++it) {
      const int t = tid + it * Sh::NT;
      if (t < EPC * NF) smem[(t / NF) * SPE + 2 * P3 + t % NF] = v[it];
    }
  }
  __syncthreads();
  // extraction by box rows (b,c): the P loads of a row are independent and issued together
  for (int rr = tid; rr < EPC * P2; rr += Sh::NT) {
    const int e = rr / P2, w = rr % P2, b = w % P, c = w / P;
    const int64_t el = e_first + e;
    T v[P];
    if (FROM_BOXES) {
#pragma unroll
      for (int a = 0; a < P; ++a) v[a] = el < nE ? T(src[el * P3 + w * P + a]) : T(0);
    } else {
      const Box1D &X = bx[e][0], &Y = bx[e][1], &Z = bx[e][2];
      const bool row_ok = el < nE && b < Y.n && c < Z.n;
      const int gyz = row_ok ? int(ghost(Y, b)) + int(ghost(Z, c)) : 2;
      const double* rowp = src + (row_ok ? sl.lidx(X.lo, Y.lo + b, Z.lo + c) : 0);
      // unconditional loads from always-valid (clamped) addresses, then select: no branch
      // per load, so all P loads of the row are in flight together
#pragma unroll
      for (int a = 0; a < P; ++a) {
        const bool ok = row_ok && a < X.n && gyz + int(ghost(X, a)) <= 1;
        const double val = __ldg(rowp + (a < X.n ? a : 0));
        v[a] = ok ? T(val) : T(0);
      }
    }
#pragma unroll
    for (int a = 0; a < P; ++a) smem[e * SPE + w * P + a] = v[a];
  }
  __syncthreads();
  const int e = tid / TPE, ti = tid % TPE;
  const bool act = e < EPC && e_first + e < nE;
  T* box = smem + (act ? e : 0) * SPE;
  T* tmp = box + P3;
  const T* Se = box + 2 * P3;
  const T* Le = Se + 3 * P2;
  if (act) line_pass<P, T, 0, 0>(box, tmp, Se + 0 * P2, Le, ti);
  __syncthreads();
  if (act) line_pass<P, T, 1, 0>(tmp, box, Se + 1 * P2, Le, ti);
  __syncthreads();
  if (act) line_pass<P, T, 2, 2>(box, tmp, Se + 2 * P2, Le, ti);
  __syncthreads();
  if (act) line_pass<P, T, 1, 1>(tmp, box, Se + 1 * P2, Le, ti);
  __syncthreads();
  if (act) line_pass<P, T, 0, 1>(box, tmp, Se + 0 * P2, Le, ti);
  __syncthreads();
}

// ---------------------------------------------------------------- RAS (+ fused Chebyshev update)
template <int P, class T>
constexpr int ras_minb() {  // CTAs per SM the CTA kernel is register-capped for
  return sizeof(T) == 4 ? (P <= 7 ? SEMLAB_RAS_SMALLP_MINB : 3) : 1;
}

template <int P, class T, int MODE>
__global__ void __launch_bounds__(128, ras_minb<P, T>()) k_ras(const Slab sl, const T* __restrict__ S, const T* __restrict__ L,
                                             const double* __restrict__ r, RasEpi epi) {
  using Sh = Shape<P, T>;
  constexpr int P2 = Sh::P2, P3 = Sh::P3, EPC = Sh::EPC, SPE = Sh::SPE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  __shared__ Box1D bx[EPC][3];
  const int64_t nE = sl.elems();
  const int64_t e_first = int64_t(blockIdx.x) * EPC;
  fdm_block<P, T, false>(sl, S, L, r, e_first, nE, smem, bx);
  // owner write: sites flattened with a (x) fastest so a warp's accesses are contiguous runs;
  // U sites per thread per round with every vector load issued before any use
  // at most q owned sites per direction, q + 1 at a Neumann domain face (its face node is kept)
  constexpr int U = 4;
  const int Q = sl.dirichlet ? P - 3 : P - 2, Q3 = Q * Q * Q;
  for (int base = threadIdx.x; base < EPC * Q3; base += Sh::NT * U) {
    int64_t g[U];
    bool ok[U];
    double z[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = base + u * Sh::NT;
      const int e = t / Q3, w = t % Q3;
      const int a = w % Q, b = (w / Q) % Q, c = w / (Q * Q);
      ok[u] = false;
      g[u] = 0;  // a valid address for the unconditional loads below
      z[u] = 0.0;
      if (t < EPC * Q3 && e_first + e < nE) {
        const Box1D &X = bx[e][0], &Y = bx[e][1], &Z = bx[e][2];
        if (a <= X.own_hi - X.own_lo && b <= Y.own_hi - Y.own_lo && c <= Z.own_hi - Z.own_lo) {
          const int aa = X.own_lo + a, bb = Y.own_lo + b, cc = Z.own_lo + c;
          ok[u] = true;
          g[u] = sl.lidx(X.lo + aa, Y.lo + bb, Z.lo + cc);
          z[u] = double(smem[e * SPE + P3 + cc * P2 + bb * P + aa]);
        }
      }
    }
    if (MODE == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ok[u]) epi.out[g[u]] = z[u];
    } else if (MODE == 1) {  // Chebyshev init: r = S t, d = r / theta  (chebyshev.cpp:82-84)
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ok[u]) {
          epi.r[g[u]] = z[u];
          epi.d[g[u]] = z[u] * epi.c2;  // c2 = 1 / theta (FP64 division per node was 11% of the stalls)
        }
    } else {  // Chebyshev step: x += d; r -= S A d; d = c1 d + c2 r  (chebyshev.cpp:86-92)
      double dv[U], rv[U], xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        dv[u] = epi.d[g[u]];
        rv[u] = epi.r[g[u]];
        xv[u] = epi.x[g[u]];
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ok[u]) {
          const double x1 = xv[u] + dv[u];
          const double rg = rv[u] - z[u];
          const double dn = epi.c1 * dv[u] + epi.c2 * rg;
          if (MODE == 3) {  // last step: the final x += d fused, r and d are dead afterwards
            epi.x[g[u]] = x1 + dn;
          } else {
            epi.x[g[u]] = x1;
            epi.r[g[u]] = rg;
            epi.d[g[u]] = dn;
          }
        }
    }
  }
}

// ---------------------------------------------------------------- RAS, one warp per element
// Same arithmetic (and summation order) as k_ras, organised so no CTA barrier couples elements:
// each warp owns one element at a time in a grid-stride loop and synchronises with __syncwarp
// only, so the gather, the FMA passes and the owner write of different warps overlap freely.
// Gather and owner write walk the box / owned sites with x fastest across the lanes (coalesced
// runs); the line passes stream the input lines from shared memory (accumulators in registers,
// ~100 registers) so five CTAs of four warps fit per SM.
template <int P, class T>
struct WShape {
  static constexpr int P2 = P * P, P3 = P2 * P;
  static constexpr int R = (P2 + 31) / 32;  // lines per lane
  static constexpr int WPC = 4;             // warps (elements in flight) per CTA
  static constexpr int NT = 32 * WPC;
  static constexpr int SPE = (2 * P3 + 3 * P2 + 3 * P + 3) / 4 * 4;  // box, tmp, S, L (16B multiple)
  static constexpr size_t smem() { return size_t(WPC) * SPE * sizeof(T); }
};

template <int P, int AX>
__device__ __forceinline__ int wline_base(int l) {
  constexpr int P2 = P * P;
  const int u = l % P, v = l / P;
  return AX == 0 ? (v * P2 + u * P) : (AX == 1 ? (v * P2 + u) : (v * P + u));
}

template <int P, class T>
__device__ __forceinline__ void load_pair(const T* M, T& s0, T& s1) {
  if constexpr (sizeof(T) == 4) {
    const float2 v = *reinterpret_cast<const float2*>(M);
    s0 = v.x;
    s1 = v.y;
  } else {
    const double2 v = *reinterpret_cast<const double2*>(M);
    s0 = v.x;
    s1 = v.y;
  }
}

// forward transform along AX: y[o] = sum_a M(a,o) x[a], x streamed from src, y in registers
template <int P, class T, int AX>
__device__ __forceinline__ void wfwd(const T* __restrict__ src, const T* __restrict__ M, const int (&base)[WShape<P, T>::R],
                                     T (&y)[WShape<P, T>::R][P]) {
  constexpr int R = WShape<P, T>::R;
  constexpr int stride = AX == 0 ? 1 : (AX == 1 ? P : P * P);
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int o = 0; o < P; ++o) y[r][o] = T(0);
#pragma unroll 2  // bounded: a full unroll hoists every S load and spills
  for (int a = 0; a < P; ++a) {
    T xa[R];
#pragma unroll
    for (int r = 0; r < R; ++r) xa[r] = src[base[r] + a * stride];
    if constexpr (P % 2 == 0 && sizeof(T) == 4 && SEMLAB_RASW_FFMA2) {
      // packed FP32 (FFMA2): the (o, o+1) output pair shares x_a; same per-output order as below
#pragma unroll
      for (int o = 0; o < P; o += 2) {
        const float2 s2 = *reinterpret_cast<const float2*>(M + a * P + o);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float2 acc = __ffma2_rn(s2, make_float2(xa[r], xa[r]), make_float2(y[r][o], y[r][o + 1]));
          y[r][o] = acc.x;
          y[r][o + 1] = acc.y;
        }
      }
    } else if constexpr (P % 2 == 0) {
#pragma unroll
      for (int o = 0; o < P; o += 2) {
        T s0, s1;
        load_pair<P, T>(M + a * P + o, s0, s1);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          y[r][o] = fma(s0, xa[r], y[r][o]);
          y[r][o + 1] = fma(s1, xa[r], y[r][o + 1]);
        }
      }
    } else {
#pragma unroll
      for (int o = 0; o < P; ++o) {
        const T sv = M[a * P + o];
#pragma unroll
        for (int r = 0; r < R; ++r) y[r][o] = fma(sv, xa[r], y[r][o]);
      }
    }
  }
}

// backward transform along AX: dst[a] = sum_o M(a,o) x[o], x in registers, rows written as formed
template <int P, class T, int AX>
__device__ __forceinline__ void wbwd(const T (&x)[WShape<P, T>::R][P], const T* __restrict__ M,
                                     const int (&base)[WShape<P, T>::R], const bool (&ok)[WShape<P, T>::R],
                                     T* __restrict__ dst) {
  constexpr int R = WShape<P, T>::R;
  constexpr int stride = AX == 0 ? 1 : (AX == 1 ? P : P * P);
#pragma unroll 2
  for (int a = 0; a < P; ++a) {
    T acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = T(0);
    if constexpr (P % 2 == 0 && sizeof(T) == 4 && SEMLAB_RASW_FFMA2) {
      // packed FP32: even and odd o accumulate in the two halves, summed at the end
      float2 a2[R];
#pragma unroll
      for (int r = 0; r < R; ++r) a2[r] = make_float2(0.f, 0.f);
#pragma unroll
      for (int o = 0; o < P; o += 2) {
        const float2 s2 = *reinterpret_cast<const float2*>(M + a * P + o);
#pragma unroll
        for (int r = 0; r < R; ++r) a2[r] = __ffma2_rn(s2, make_float2(x[r][o], x[r][o + 1]), a2[r]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = a2[r].x + a2[r].y;
    } else if constexpr (P % 2 == 0) {
#pragma unroll
      for (int o = 0; o < P; o += 2) {
        T s0, s1;
        load_pair<P, T>(M + a * P + o, s0, s1);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          acc[r] = fma(s0, x[r][o], acc[r]);
          acc[r] = fma(s1, x[r][o + 1], acc[r]);
        }
      }
    } else {
#pragma unroll
      for (int o = 0; o < P; ++o) {
        const T sv = M[a * P + o];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = fma(sv, x[r][o], acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (ok[r]) dst[base[r] + a * stride] = acc[r];
  }
}

template <int P, class T, int AX>
__device__ __forceinline__ void wbases(int lane, int (&base)[WShape<P, T>::R], bool (&ok)[WShape<P, T>::R]) {
#pragma unroll
  for (int r = 0; r < WShape<P, T>::R; ++r) {
    const int l = lane + 32 * r;
    ok[r] = l < P * P;
    base[r] = ok[r] ? wline_base<P, AX>(l) : 0;  // idle lines read a valid address, never write
  }
}

#ifndef SEMLAB_RASW_PF
#define SEMLAB_RASW_PF 0  // L2 prefetch of the next element's box rows and factors
#endif

template <int P, class T, int MODE>
__global__ void __launch_bounds__(WShape<P, T>::NT, sizeof(T) == 4 ? SEMLAB_RASW_MINB : 2)
    k_rasw(const Slab sl, const T* __restrict__ S, const T* __restrict__ L, const double* __restrict__ rin,
           RasEpi epi) {
  using W = WShape<P, T>;
  constexpr int P2 = W::P2, P3 = W::P3, R = W::R, SPE = W::SPE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T* box = reinterpret_cast<T*>(smem_raw) + warp * SPE;
  T* tmp = box + P3;
  T* Se = tmp + P3;
  T* Le = Se + 3 * P2;
  const int nE = int(sl.elems());
  const bool dir = sl.dirichlet != 0;
  for (int el = blockIdx.x * W::WPC + warp; el < nE; el += gridDim.x * W::WPC) {
    const int ex = el % sl.Ex, ey = (el / sl.Ex) % sl.Ey, ez = sl.ez0 + el / (sl.Ex * sl.Ey);
    const Box1D X = box1d(ex, sl.Ex, sl.q, dir), Y = box1d(ey, sl.Ey, sl.q, dir), Z = box1d(ez, sl.Ez, sl.q, dir);
#if SEMLAB_RASW_PF
    {  // the next element's extended-box rows (and factors) -> L2 while this element is solved
      const int en = el + gridDim.x * W::WPC;
      if (en < nE) {
        const int nx = en % sl.Ex, ny = (en / sl.Ex) % sl.Ey, nz = sl.ez0 + en / (sl.Ex * sl.Ey);
        const Box1D NX = box1d(nx, sl.Ex, sl.q, dir), NY = box1d(ny, sl.Ey, sl.q, dir), NZ = box1d(nz, sl.Ez, sl.q, dir);
        const double* nc = rin + sl.lidx(NX.lo, NY.lo, NZ.lo);
        const int64_t NXY = sl.Nx * sl.Ny;
        for (int rw = lane; rw < NY.n * NZ.n; rw += 32) {
          const double* p = nc + (rw % NY.n) * sl.Nx + (rw / NY.n) * NXY;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(p + NX.n - 1));
        }
        if (lane < (3 * P2 * int(sizeof(T)) + 127) / 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(S + int64_t(en) * 3 * P2) + lane * 128));
      }
    }
#endif
    __syncwarp();  // the previous element's owner write has finished reading tmp
    {  // factors: S (3 P^2) and lambda (3 P), all loads issued before the stores
      constexpr int NF = 3 * P2 + 3 * P, IT = (NF + 31) / 32;
      T v[IT];
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const int w = lane + 32 * it;
        v[it] = w < 3 * P2 ? __ldg(S + int64_t(el) * 3 * P2 + w)
                           : (w < NF ? __ldg(L + int64_t(el) * 3 * P + (w - 3 * P2)) : T(0));
      }
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const int w = lane + 32 * it;
        if (w < NF) Se[w] = v[it];
      }
    }
    {  // gather the extended box by z-columns: lane = (a, b) pair, loop over c, so the x/y
       // validity and the column address are fixed per pair and the z test is a bit mask; sites
       // outside the core in more than one direction (and outside a smaller boundary box) are zero
       // (schwarz.cpp:255-265)
      unsigned zin = 0, zcore = 0;  // c < Z.n; c < Z.n and not a z ghost
#pragma unroll
      for (int c = 0; c < P; ++c) {
        zin |= unsigned(c < Z.n) << c;
        zcore |= unsigned(c < Z.n && !ghost(Z, c)) << c;
      }
      const int64_t NXY = sl.Nx * sl.Ny;
      const double* corner = rin + sl.lidx(X.lo, Y.lo, Z.lo);
#pragma unroll kGatherUnroll
      for (int r = 0; r < R; ++r) {
        const int l = min(lane + 32 * r, P2 - 1);  // lanes past the last pair redo it (same values)
        const int a = l % P, b = l / P;
        const bool okab = a < X.n && b < Y.n;
        const int gab = int(ghost(X, a)) + int(ghost(Y, b));
        const unsigned m = !okab ? 0u : (gab == 0 ? zin : (gab == 1 ? zcore : 0u));
        const double* col = corner + a + b * sl.Nx;
        double v[P];
#pragma unroll
        for (int c = 0; c < P; ++c) v[c] = __ldg((m >> c) & 1u ? col + c * NXY : rin);
#pragma unroll
        for (int c = 0; c < P; ++c) box[c * P2 + l] = (m >> c) & 1u ? T(v[c]) : T(0);
      }
    }
    __syncwarp();
    int base[R];
    bool okl[R];
    T y[R][P];
    wbases<P, T, 0>(lane, base, okl);
    wfwd<P, T, 0>(box, Se + 0 * P2, base, y);  // x forward: box -> tmp
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (okl[r])
#pragma unroll
        for (int o = 0; o < P; ++o) tmp[base[r] + o] = y[r][o];
    __syncwarp();
    wbases<P, T, 1>(lane, base, okl);
    wfwd<P, T, 1>(tmp, Se + 1 * P2, base, y);  // y forward: tmp -> box
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (okl[r])
#pragma unroll
        for (int o = 0; o < P; ++o) box[base[r] + o * P] = y[r][o];
    __syncwarp();
    wbases<P, T, 2>(lane, base, okl);
    wfwd<P, T, 2>(box, Se + 2 * P2, base, y);  // z forward, scale by inv_D, z backward: box -> tmp
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int l = lane + 32 * r;
      const int a = l % P, b = (l / P) % P;
      const T lab = Le[0 * P + a] + Le[1 * P + b];
#pragma unroll
      for (int c = 0; c < P; ++c) y[r][c] = y[r][c] * rcp(lab + Le[2 * P + c]);
    }
    wbwd<P, T, 2>(y, Se + 2 * P2, base, okl, tmp);
    __syncwarp();
    wbases<P, T, 1>(lane, base, okl);  // y backward: tmp -> box
    {
      constexpr int stride = P;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int m = 0; m < P; ++m) y[r][m] = tmp[base[r] + m * stride];
    }
    wbwd<P, T, 1>(y, Se + 1 * P2, base, okl, box);
    __syncwarp();
    wbases<P, T, 0>(lane, base, okl);  // x backward: box -> tmp
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int m = 0; m < P; ++m) y[r][m] = box[base[r] + m];
    wbwd<P, T, 0>(y, Se + 0 * P2, base, okl, tmp);
    __syncwarp();
    // owner write by z-columns: lane = (a, b) over the owned face (QA x QA, power of two so the
    // split is a shift), U consecutive c per round with every vector load issued before the stores
    const int na = X.own_hi - X.own_lo + 1, nb = Y.own_hi - Y.own_lo + 1, nc = Z.own_hi - Z.own_lo + 1;
    constexpr int QA = (P - 2) <= 4 ? 4 : ((P - 2) <= 8 ? 8 : 16);
    constexpr int U = SEMLAB_RASW_OWNER_U;
    const int64_t NXY = sl.Nx * sl.Ny;
#pragma unroll 1
    for (int pr = lane; pr < QA * QA; pr += 32) {
      const int oa = pr % QA, ob = pr / QA;
      if (oa >= na || ob >= nb) continue;
      const int aa = X.own_lo + oa, bb = Y.own_lo + ob;
      const int64_t g0 = sl.lidx(X.lo + aa, Y.lo + bb, Z.lo + Z.own_lo);
      const T* zt = tmp + Z.own_lo * P2 + bb * P + aa;
#pragma unroll 1
      for (int c0 = 0; c0 < nc; c0 += U) {
        int64_t g[U];
        bool ok[U];
        double z[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = c0 + u;
          ok[u] = c < nc;
          g[u] = ok[u] ? g0 + c * NXY : g0;
          z[u] = ok[u] ? double(zt[c * P2]) : 0.0;
        }
        if (MODE == 0) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (ok[u]) epi.out[g[u]] = z[u];
        } else if (MODE == 1) {  // Chebyshev init: r = S t, d = r / theta  (chebyshev.cpp:82-84)
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (ok[u]) {
              epi.r[g[u]] = z[u];
              epi.d[g[u]] = z[u] * epi.c2;  // c2 = 1 / theta (FP64 division per node was 11% of the stalls)
            }
        } else {  // Chebyshev step: x += d; r -= S A d; d = c1 d + c2 r  (chebyshev.cpp:86-92)
          double dv[U], rv[U], xv[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            dv[u] = epi.d[g[u]];
            rv[u] = epi.r[g[u]];
            xv[u] = epi.x[g[u]];
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (ok[u]) {
              const double x1 = xv[u] + dv[u];
              const double rg = rv[u] - z[u];
              const double dn = epi.c1 * dv[u] + epi.c2 * rg;
              if (MODE == 3) {  // last step: the final x += d fused, r and d are dead afterwards
                epi.x[g[u]] = x1 + dn;
              } else {
                epi.x[g[u]] = x1;
                epi.r[g[u]] = rg;
                epi.d[g[u]] = dn;
              }
            }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- ASM boxes + deterministic sum
template <int P, class T>
__global__ void __launch_bounds__(128, sizeof(T) == 4 ? 3 : 1) k_asm_boxes(const Slab sl, const T* __restrict__ S, const T* __restrict__ L,
                                                   const double* __restrict__ r, T* __restrict__ boxes) {
  using Sh = Shape<P, T>;
  constexpr int P3 = Sh::P3, EPC = Sh::EPC, SPE = Sh::SPE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  __shared__ Box1D bx[EPC][3];
  const int64_t nE = sl.elems();
  const int64_t e_first = int64_t(blockIdx.x) * EPC;
  fdm_block<P, T, false>(sl, S, L, r, e_first, nE, smem, bx);
  for (int t = threadIdx.x; t < EPC * P3; t += Sh::NT) {
    const int e = t / P3, w = t % P3;
    if (e_first + e < nE) boxes[(e_first + e) * P3 + w] = smem[e * SPE + P3 + w];
  }
}

// out[g] = (1/count) * sum over elements whose participating box covers g, ascending id.
// On a z-slab the sum also covers the ghost planes, and on the exchange planes (zb-1, zb, zb+1
// below an internal boundary; zt-1, zt, zt+1 above one) it writes the raw local sum to out and
// the local count to cnt[plane][x + Nx y] (planes 0..2 bottom, 3..5 top) for asm_exchange.
template <int P, class T>
__global__ void k_asm_sum(const Slab sl, const T* __restrict__ boxes, double* __restrict__ out,
                          double* __restrict__ cnt) {
  constexpr int P2 = P * P, P3 = P2 * P;
  const int q = sl.q;
  const bool dir = sl.dirichlet != 0;
  const int64_t zb = int64_t(sl.ez0) * q, zt = int64_t(sl.ez1) * q;
  const int64_t z0 = zb - sl.nranks_below, nz = zt + sl.nranks_above - z0 + 1;
  const int64_t total = sl.Nx * sl.Ny * nz;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t x = t % sl.Nx, y = (t / sl.Nx) % sl.Ny, z = z0 + t / (sl.Nx * sl.Ny);
    int ce[3][3], ca[3][3], cg[3][3], cn[3] = {0, 0, 0};
    const int64_t coord[3] = {x, y, z};
    const int Ed[3] = {sl.Ex, sl.Ey, sl.Ez};
    const int lo_e[3] = {0, 0, sl.ez0}, hi_e[3] = {sl.Ex, sl.Ey, sl.ez1};
    for (int d = 0; d < 3; ++d) {
      const int base = int(coord[d] / q);
      for (int e = base - 1; e <= base + 1; ++e) {
        if (e < lo_e[d] || e >= hi_e[d]) continue;
        const Box1D b = box1d(e, Ed[d], q, dir);
        const int a = int(coord[d]) - b.lo;
        if (a < 0 || a >= b.n) continue;
        ce[d][cn[d]] = e;
        ca[d][cn[d]] = a;
        cg[d][cn[d]] = ghost(b, a) ? 1 : 0;
        ++cn[d];
      }
    }
    double acc = 0.0;
    int count = 0;
    for (int k = 0; k < cn[2]; ++k)
      for (int j = 0; j < cn[1]; ++j)
        for (int i = 0; i < cn[0]; ++i) {
          if (cg[0][i] + cg[1][j] + cg[2][k] > 1) continue;
          const int64_t el = ce[0][i] + int64_t(sl.Ex) * (ce[1][j] + int64_t(sl.Ey) * (ce[2][k] - sl.ez0));
          acc += double(boxes[el * P3 + ca[2][k] * P2 + ca[1][j] * P + ca[0][i]]);
          ++count;
        }
    int plane = -1;
    if (sl.nranks_below && z <= zb + 1) plane = int(z - (zb - 1));
    if (sl.nranks_above && z >= zt - 1) plane = 3 + int(z - (zt - 1));
    if (plane >= 0) {
      out[sl.lidx(x, y, z)] = acc;
      cnt[int64_t(plane) * sl.Nx * sl.Ny + x + sl.Nx * y] = double(count);
    } else {
      out[sl.lidx(x, y, z)] = count > 0 ? acc * (1.0 / double(count)) : 0.0;
    }
  }
}

// ASM on slabs, after the exchange: plane = lower partial + upper partial over the summed counts
// (both ranks form the interface plane in the same order: bitwise identical copies).
__global__ void k_asm_combine(double* __restrict__ v, const double* __restrict__ lo_sum,
                              const double* __restrict__ lo_cnt, const double* __restrict__ hi_sum,
                              const double* __restrict__ hi_cnt, int64_t P) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < P; t += int64_t(gridDim.x) * blockDim.x) {
    const double c = lo_cnt[t] + hi_cnt[t];
    v[t] = c > 0.0 ? (lo_sum[t] + hi_sum[t]) * (1.0 / c) : 0.0;
  }
}

// fdm_solve on given boxes (API / tests), FP64 in/out
template <int P, class T>
__global__ void __launch_bounds__(128, sizeof(T) == 4 ? 3 : 1) k_fdm_boxes(const Slab sl, const T* __restrict__ S, const T* __restrict__ L,
                                                   const double* __restrict__ in, double* __restrict__ outb) {
  using Sh = Shape<P, T>;
  constexpr int P3 = Sh::P3, EPC = Sh::EPC, SPE = Sh::SPE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  __shared__ Box1D bx[EPC][3];
  const int64_t nE = sl.elems();
  const int64_t e_first = int64_t(blockIdx.x) * EPC;
  fdm_block<P, T, true>(sl, S, L, in, e_first, nE, smem, bx);
  for (int t = threadIdx.x; t < EPC * P3; t += Sh::NT) {
    const int e = t / P3, w = t % P3;
    if (e_first + e < nE) outb[(e_first + e) * P3 + w] = double(smem[e * SPE + P3 + w]);
  }
}

template <class K>
void prep(K kern, size_t smem) {
  smem_attr(kern, smem);
}

#ifndef SEMLAB_RAS_WARP
#define SEMLAB_RAS_WARP 1  // build-time A/B (tools/build_variant*.sh): 0 = CTA-per-group RAS for every order
#endif
constexpr bool ras_warp() { return SEMLAB_RAS_WARP != 0; }

template <class T>
struct Launch {
  // warp-per-element RAS for the large boxes (SEMLAB_RAS_WARP=0 selects the CTA-per-group kernel)
  template <int P, int MODE>
  static void rasw(const Slab& sl, const T* S, const T* L, const double* r, const RasEpi& e, cudaStream_t s) {
    using W = WShape<P, T>;
    auto kern = k_rasw<P, T, MODE>;
    const int nctas = resident_ctas(kern, W::NT, W::smem());
    const int64_t need = (sl.elems() + W::WPC - 1) / W::WPC;
    kern<<<capped_grid(std::min<int64_t>(need, nctas)), W::NT, W::smem(), s>>>(sl, S, L, r, e);
  }
  template <int P>
  static void ras(const Slab& sl, const T* S, const T* L, const double* r, int mode, const RasEpi& e, cudaStream_t s) {
    if (sizeof(T) == 4 && P >= SEMLAB_RASW_MINP && ras_warp() && sl.elems() < (int64_t(1) << 31)) {
      if (mode == 0) rasw<P, 0>(sl, S, L, r, e, s);
      else if (mode == 1) rasw<P, 1>(sl, S, L, r, e, s);
      else if (mode == 2) rasw<P, 2>(sl, S, L, r, e, s);
      else rasw<P, 3>(sl, S, L, r, e, s);
      return;
    }
    using Sh = Shape<P, T>;
    const int grid = int((sl.elems() + Sh::EPC - 1) / Sh::EPC);
    if (mode == 0) {
      prep(k_ras<P, T, 0>, Sh::smem());
      k_ras<P, T, 0><<<grid, Sh::NT, Sh::smem(), s>>>(sl, S, L, r, e);
    } else if (mode == 1) {
      prep(k_ras<P, T, 1>, Sh::smem());
      k_ras<P, T, 1><<<grid, Sh::NT, Sh::smem(), s>>>(sl, S, L, r, e);
    } else if (mode == 2) {
      prep(k_ras<P, T, 2>, Sh::smem());
      k_ras<P, T, 2><<<grid, Sh::NT, Sh::smem(), s>>>(sl, S, L, r, e);
    } else {
      prep(k_ras<P, T, 3>, Sh::smem());
      k_ras<P, T, 3><<<grid, Sh::NT, Sh::smem(), s>>>(sl, S, L, r, e);
    }
  }
  template <int P>
  static void asm_(const Slab& sl, const T* S, const T* L, const double* r, void* boxes, double* out, double* cnt,
                   cudaStream_t s) {
    using Sh = Shape<P, T>;
    const int grid = int((sl.elems() + Sh::EPC - 1) / Sh::EPC);
    prep(k_asm_boxes<P, T>, Sh::smem());
    k_asm_boxes<P, T><<<grid, Sh::NT, Sh::smem(), s>>>(sl, S, L, r, static_cast<T*>(boxes));
    const int64_t total = sl.Nx * sl.Ny * (int64_t(sl.ez1 - sl.ez0) * sl.q + 1 + sl.nranks_below + sl.nranks_above);
    k_asm_sum<P, T><<<int(std::min<int64_t>((total + 255) / 256, 148 * 32)), 256, 0, s>>>(
        sl, static_cast<const T*>(boxes), out, cnt);
  }
  template <int P>
  static void boxes(const Slab& sl, const T* S, const T* L, const double* in, double* out, cudaStream_t s) {
    using Sh = Shape<P, T>;
    const int grid = int((sl.elems() + Sh::EPC - 1) / Sh::EPC);
    prep(k_fdm_boxes<P, T>, Sh::smem());
    k_fdm_boxes<P, T><<<grid, Sh::NT, Sh::smem(), s>>>(sl, S, L, in, out);
  }
};

#define SB_FDM_SWITCH(P_, CALL)                                              \
  switch (P_) {                                                               \
    case 5: CALL(5); break;                                                   \
    case 6: CALL(6); break;                                                   \
    case 7: CALL(7); break;                                                   \
    case 8: CALL(8); break;                                                   \
    case 9: CALL(9); break;                                                   \
    case 10: CALL(10); break;                                                 \
    case 11: CALL(11); break;                                                 \
    case 12: CALL(12); break;                                                 \
    default: invalid("SchwarzSmoother: device kernels support orders 2..9"); \
  }

}  // namespace

int64_t launch_ras(const Slab& sl, int precision, const void* S, const void* L, const double* r, int mode,
                   const RasEpi& e, cudaStream_t s) {
  if (sl.elems() == 0) return 0;
  const int P = sl.q + 3;
  if (precision == 32) {
#define C32(PP) Launch<float>::ras<PP>(sl, static_cast<const float*>(S), static_cast<const float*>(L), r, mode, e, s)
    SB_FDM_SWITCH(P, C32)
#undef C32
  } else {
#define C64(PP) Launch<double>::ras<PP>(sl, static_cast<const double*>(S), static_cast<const double*>(L), r, mode, e, s)
    SB_FDM_SWITCH(P, C64)
#undef C64
  }
  SB_LAUNCH_CHECK();
  return 1;
}

int64_t launch_asm(const Slab& sl, int precision, const void* S, const void* L, const double* r, void* boxes,
                   double* out, double* cnt, cudaStream_t s) {
  if (sl.elems() == 0) return 0;
  const int P = sl.q + 3;
  if (precision == 32) {
#define C32(PP) Launch<float>::asm_<PP>(sl, static_cast<const float*>(S), static_cast<const float*>(L), r, boxes, out, cnt, s)
    SB_FDM_SWITCH(P, C32)
#undef C32
  } else {
#define C64(PP) Launch<double>::asm_<PP>(sl, static_cast<const double*>(S), static_cast<const double*>(L), r, boxes, out, cnt, s)
    SB_FDM_SWITCH(P, C64)
#undef C64
  }
  SB_LAUNCH_CHECK();
  return 2;
}

int64_t launch_fdm_boxes(const Slab& sl, int precision, const void* S, const void* L, const double* in, double* out,
                         cudaStream_t s) {
  if (sl.elems() == 0) return 0;
  const int P = sl.q + 3;
  if (precision == 32) {
#define C32(PP) Launch<float>::boxes<PP>(sl, static_cast<const float*>(S), static_cast<const float*>(L), in, out, s)
    SB_FDM_SWITCH(P, C32)
#undef C32
  } else {
#define C64(PP) Launch<double>::boxes<PP>(sl, static_cast<const double*>(S), static_cast<const double*>(L), in, out, s)
    SB_FDM_SWITCH(P, C64)
#undef C64
  }
  SB_LAUNCH_CHECK();
  return 1;
}

int64_t launch_asm_combine(double* v, const double* lo_sum, const double* lo_cnt, const double* hi_sum,
                           const double* hi_cnt, int64_t P, cudaStream_t s) {
  k_asm_combine<<<int(std::min<int64_t>((P + 255) / 256, 148 * 8)), 256, 0, s>>>(v, lo_sum, lo_cnt, hi_sum, hi_cnt, P);
  SB_LAUNCH_CHECK();
  return 1;
}

}  // namespace sb
