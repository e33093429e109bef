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

#ifndef SEMLAB_RASW_OWNER_U
#define SEMLAB_RASW_OWNER_U 4  // owned sites per lane per batch of the owner write
#endif
#ifndef SEMLAB_RASW_MINB
#define SEMLAB_RASW_MINB 3  // resident 4-warp CTAs per SM (3 x 74.6 KB of shared memory at P = 10)
#endif

#ifndef SEMLAB_RAS_SMALLP_MINB
#define SEMLAB_RAS_SMALLP_MINB 5  // p = 3 level (P = 6): 5 CTAs/SM of the CTA RAS kernel
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
      if constexpr (P % 2 == 0) {
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
      if constexpr (P % 2 == 0) {
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
// Warp-per-element RAS (FP32 FDM), the p >= 5 boxes (P = p + 3 >= 8). Line passes with a fixed
// lane -> line map: lane = (u, w0) with u = lane % P, w0 = lane / P (G = 32 / P groups, P*G lanes
// busy); the lane owns the lines w = w0 + G r (r < R = ceil(P / G)) of every pass, so all its
// shared-memory addresses are one base register plus compile-time offsets. Per input value a
// line pass costs one shared load and P scalar FFMA (FFMA issues at twice the flop rate of FFMA2
// on this part: tools/peak_bench.cu); the factor rows are read as 16-byte broadcasts. The z pass
// keeps its lines in registers through the forward transform, the inv_D scaling and the
// backward transform. The next element's extended box (FP64, as stored) and factors arrive by
// cp.async one element ahead.
template <int P>
struct LShape {
  static constexpr int P2 = P * P, P3 = P2 * P;
  static constexpr int G = 32 / P;             // lane groups
  static constexpr int R = (P + G - 1) / G;    // lines per lane per pass
  static constexpr int SP = (P + 3) / 4 * 4;   // factor row stride (16-byte rows)
  static constexpr int FAC = 3 * P * SP + 3 * SP;  // S_x, S_y, S_z rows, then lambda_x, _y, _z
  static constexpr int WPC = 4;                // warps (elements in flight) per CTA
  static constexpr int NT = 32 * WPC;
  // per warp (floats): FP64 staging of the box, the FP32 box and tmp, the factors double-buffered
  static constexpr int SPE = 2 * P3 + 2 * P3 + 2 * FAC;
  static constexpr size_t smem() { return size_t(WPC) * SPE * sizeof(float); }
};

// P entries of a 16-byte aligned factor row (broadcast loads)
template <int P>
__device__ __forceinline__ void load_row(const float* __restrict__ row, float (&s)[P]) {
  constexpr int SP = LShape<P>::SP;
  float v[SP];
#pragma unroll
  for (int q4 = 0; q4 < SP / 4; ++q4) {
    const float4 t = *reinterpret_cast<const float4*>(row + 4 * q4);
    v[4 * q4] = t.x;
    v[4 * q4 + 1] = t.y;
    v[4 * q4 + 2] = t.z;
    v[4 * q4 + 3] = t.w;
  }
#pragma unroll
  for (int o = 0; o < P; ++o) s[o] = v[o];
}

// forward transform of the lane's R lines: y[r][o] = sum_a M(a, o) src[base + OFF r + STEP a]
template <int P, int OFF, int STEP, class SrcT>
__device__ __forceinline__ void lfwd(const SrcT* __restrict__ src, const float* __restrict__ M,
                                     float (&y)[LShape<P>::R][P]) {
  constexpr int R = LShape<P>::R, SP = LShape<P>::SP;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int o = 0; o < P; ++o) y[r][o] = 0.f;
#pragma unroll
  for (int a = 0; a < P; ++a) {
    float xa[R];
#pragma unroll
    for (int r = 0; r < R; ++r) xa[r] = float(src[OFF * r + STEP * a]);
    float sr[P];
    load_row<P>(M + a * SP, sr);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int o = 0; o < P; ++o) y[r][o] = fmaf(sr[o], xa[r], y[r][o]);
  }
}

// backward transform: out[r][a] = sum_o M(a, o) x[r][o], written to dst[OFF r + STEP a]
template <int P, int OFF, int STEP>
__device__ __forceinline__ void lbwd(const float (&x)[LShape<P>::R][P], const float* __restrict__ M,
                                     const bool (&ok)[LShape<P>::R], float* __restrict__ dst) {
  constexpr int R = LShape<P>::R, SP = LShape<P>::SP;
#pragma unroll
  for (int a = 0; a < P; ++a) {
    float sr[P];
    load_row<P>(M + a * SP, sr);
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      acc[r] = 0.f;
#pragma unroll
      for (int o = 0; o < P; ++o) acc[r] = fmaf(sr[o], x[r][o], acc[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (ok[r]) dst[OFF * r + STEP * a] = acc[r];
  }
}

template <int P>
__device__ __forceinline__ void lstore(const float (&y)[LShape<P>::R][P], const bool (&ok)[LShape<P>::R],
                                       float* __restrict__ dst, int off, int step) {
#pragma unroll
  for (int r = 0; r < LShape<P>::R; ++r)
    if (ok[r])
#pragma unroll
      for (int o = 0; o < P; ++o) dst[off * r + step * o] = y[r][o];
}

template <int P, int MODE>
__global__ void __launch_bounds__(LShape<P>::NT, SEMLAB_RASW_MINB)
    k_rasw(const Slab sl, const float* __restrict__ S, const float* __restrict__ L, const double* __restrict__ rin,
           RasEpi epi) {
  using W = LShape<P>;
  constexpr int P2 = W::P2, P3 = W::P3, G = W::G, R = W::R, SP = W::SP, SPE = W::SPE, FAC = W::FAC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* stage = reinterpret_cast<double*>(reinterpret_cast<float*>(smem_raw) + warp * SPE);
  float* box = reinterpret_cast<float*>(stage + P3);
  float* tmp = box + P3;
  float* fac0 = tmp + P3;  // factors of even / odd iterations of this warp's element loop
  const int nE = int(sl.elems());
  const bool dir = sl.dirichlet != 0;
  const int64_t NXY = sl.Nx * sl.Ny;
  const int stride = gridDim.x * W::WPC;
  // line map of this lane (idle lanes past P*G shadow lane 0 and never store)
  const bool lane_on = lane < P * G;
  const int u = lane_on ? lane % P : 0, w0 = lane_on ? lane / P : 0;
  bool ok[R];
#pragma unroll
  for (int r = 0; r < R; ++r) ok[r] = lane_on && (w0 + G * r < P);

  // Asynchronous loads of element e: the factor rows (padded to SP) and lambdas into fac, the
  // extended box (FP64) into the staging buffer. Sites outside the box, and sites outside the
  // element core in more than one direction (schwarz.cpp:255-265), are zero-filled by the copy
  // itself (src-size 0). The box is gathered by z-columns: lane = (a, b) pair.
  auto issue = [&](int e, float* fac) {
    const int ex = e % sl.Ex, ey = (e / sl.Ex) % sl.Ey, ez = sl.ez0 + e / (sl.Ex * sl.Ey);
    const Box1D X = box1d(ex, sl.Ex, sl.q, dir), Y = box1d(ey, sl.Ey, sl.q, dir), Z = box1d(ez, sl.Ez, sl.q, dir);
    const float* se = S + int64_t(e) * 3 * P2;
    for (int w = lane; w < 3 * P2; w += 32) {
      const int d = w / P2, rem = w - d * P2, ra = rem / P, o = rem - ra * P;
      cp_async4(fac + d * P * SP + ra * SP + o, se + w);
    }
    if (lane < 3 * P) {
      const int d = lane / P;
      cp_async4(fac + 3 * P * SP + d * SP + (lane - d * P), L + int64_t(e) * 3 * P + lane);
    }
    unsigned zin = 0, zcore = 0;  // c < Z.n; c < Z.n and not a z ghost
#pragma unroll
    for (int c = 0; c < P; ++c) {
      zin |= unsigned(c < Z.n) << c;
      zcore |= unsigned(c < Z.n && !ghost(Z, c)) << c;
    }
    const double* corner = rin + sl.lidx(X.lo, Y.lo, Z.lo);
#pragma unroll 1
    for (int l = lane; l < P2; l += 32) {
      const int a = l % P, b = l / P;
      const bool okab = a < X.n && b < Y.n;
      const int gab = int(ghost(X, a)) + int(ghost(Y, b));
      const unsigned m = !okab ? 0u : (gab == 0 ? zin : (gab == 1 ? zcore : 0u));
      const double* col = corner + a + b * sl.Nx;
#pragma unroll
      for (int c = 0; c < P; ++c) {
        const bool on = (m >> c) & 1u;
        cp_async8(stage + c * P2 + l, on ? col + c * NXY : rin, on);
      }
    }
    cp_async_commit();
  };
  int el = blockIdx.x * W::WPC + warp;
  if (el < nE) issue(el, fac0);
  for (int it = 0; el < nE; el += stride, ++it) {
    const float* Sx = fac0 + (it & 1) * FAC;
    const float* Sy = Sx + P * SP;
    const float* Sz = Sy + P * SP;
    const float* Lm = Sz + P * SP;  // lambda_x at Lm, lambda_y at Lm + SP, lambda_z at Lm + 2 SP
    const int ex = el % sl.Ex, ey = (el / sl.Ex) % sl.Ey, ez = sl.ez0 + el / (sl.Ex * sl.Ey);
    const Box1D X = box1d(ex, sl.Ex, sl.q, dir), Y = box1d(ey, sl.Ey, sl.q, dir), Z = box1d(ez, sl.Ez, sl.q, dir);
    cp_async_wait_all();
    __syncwarp();  // this element's box and factors are in shared memory for every lane
    float y[R][P];
    // x forward: lines (b, c) = (u, w): staged FP64 box -> tmp
    lfwd<P, G * P2, 1>(stage + P * u + P2 * w0, Sx, y);
    lstore<P>(y, ok, tmp + P * u + P2 * w0, G * P2, 1);
    __syncwarp();  // the staging buffer and the other factor buffer are free: prefetch the next element
    if (el + stride < nE) issue(el + stride, fac0 + ((it + 1) & 1) * FAC);
    // y forward: lines (a, c) = (u, w): tmp -> box
    lfwd<P, G * P2, P>(tmp + u + P2 * w0, Sy, y);
    lstore<P>(y, ok, box + u + P2 * w0, G * P2, P);
    __syncwarp();
    // z: lines (a, b) = (u, w): forward, scale by inv_D = 1 / (lx_a + ly_b + lz_c), backward
    lfwd<P, G * P, P2>(box + u + P * w0, Sz, y);
    {
      float lz[P];
      load_row<P>(Lm + 2 * SP, lz);
      const float lx = Lm[u];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float lab = lx + Lm[SP + min(w0 + G * r, P - 1)];
#pragma unroll
        for (int o = 0; o < P; ++o) {
          float inv;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(lab + lz[o]));
          y[r][o] *= inv;
        }
      }
    }
    lbwd<P, G * P, P2>(y, Sz, ok, tmp + u + P * w0);
    __syncwarp();
    // y backward: lines (a, c): tmp -> box
    {
      const float* src = tmp + u + P2 * w0;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int o = 0; o < P; ++o) y[r][o] = src[G * P2 * r + P * o];
    }
    lbwd<P, G * P2, P>(y, Sy, ok, box + u + P2 * w0);
    __syncwarp();
    // x backward: lines (b, c): box -> tmp
    {
      const float* src = box + P * u + P2 * w0;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int o = 0; o < P; ++o) y[r][o] = src[G * P2 * r + o];
    }
    lbwd<P, G * P2, 1>(y, Sx, ok, tmp + P * u + P2 * w0);
    __syncwarp();
    // owner write by z-columns: lane = (a, b) over the owned face (QA x QA, power of two so the
    // split is a shift), U consecutive c per round with every vector load issued before the stores
    const int na = X.own_hi - X.own_lo + 1, nb = Y.own_hi - Y.own_lo + 1, nc = Z.own_hi - Z.own_lo + 1;
    constexpr int QA = (P - 2) <= 4 ? 4 : ((P - 2) <= 8 ? 8 : 16);
    constexpr int U = SEMLAB_RASW_OWNER_U;
#pragma unroll 1
    for (int pr = lane; pr < QA * QA; pr += 32) {
      const int oa = pr % QA, ob = pr / QA;
      if (oa >= na || ob >= nb) continue;
      const int aa = X.own_lo + oa, bb = Y.own_lo + ob;
      const int64_t g0 = sl.lidx(X.lo + aa, Y.lo + bb, Z.lo + Z.own_lo);
      const float* zt = tmp + Z.own_lo * P2 + bb * P + aa;
#pragma unroll 1
      for (int c0 = 0; c0 < nc; c0 += U) {
        int64_t g[U];
        bool okc[U];
        double z[U];
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
          const int c = c0 + uu;
          okc[uu] = c < nc;
          g[uu] = okc[uu] ? g0 + c * NXY : g0;
          z[uu] = okc[uu] ? double(zt[c * P2]) : 0.0;
        }
        if (MODE == 0) {
#pragma unroll
          for (int uu = 0; uu < U; ++uu)
            if (okc[uu]) epi.out[g[uu]] = z[uu];
        } else if (MODE == 1) {  // Chebyshev init: r = S t, d = r / theta  (chebyshev.cpp:82-84)
#pragma unroll
          for (int uu = 0; uu < U; ++uu)
            if (okc[uu]) {
              epi.r[g[uu]] = z[uu];
              epi.d[g[uu]] = z[uu] * epi.c2;  // c2 = 1 / theta
            }
        } else {  // Chebyshev step: x += d; r -= S A d; d = c1 d + c2 r  (chebyshev.cpp:86-92)
          double dv[U], rv[U], xv[U];
#pragma unroll
          for (int uu = 0; uu < U; ++uu) {
            dv[uu] = epi.d[g[uu]];
            rv[uu] = epi.r[g[uu]];
            xv[uu] = epi.x[g[uu]];
          }
#pragma unroll
          for (int uu = 0; uu < U; ++uu)
            if (okc[uu]) {
              const double x1 = xv[uu] + dv[uu];
              const double rg = rv[uu] - z[uu];
              const double dn = epi.c1 * dv[uu] + epi.c2 * rg;
              if (MODE == 3) {  // last step: the final x += d fused, r and d are dead afterwards
                epi.x[g[uu]] = x1 + dn;
              } else {
                epi.x[g[uu]] = x1;
                epi.r[g[uu]] = rg;
                epi.d[g[uu]] = dn;
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

// out[g] = (1/count) * sum over elements whose participating box covers g, ascending id
template <int P, class T>
__global__ void k_asm_sum(const Slab sl, const T* __restrict__ boxes, double* __restrict__ out) {
  constexpr int P2 = P * P, P3 = P2 * P;
  const int q = sl.q;
  const bool dir = sl.dirichlet != 0;
  const int64_t z0 = int64_t(sl.ez0) * q, nz = int64_t(sl.ez1 - sl.ez0) * q + 1;
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
    out[sl.lidx(x, y, z)] = count > 0 ? acc * (1.0 / double(count)) : 0.0;
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

bool ras_warp() {
  static const bool on = [] {
    const char* e = std::getenv("SEMLAB_RAS_WARP");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class T>
struct Launch {
  // warp-per-element RAS for the large boxes (SEMLAB_RAS_WARP=0 selects the CTA-per-group kernel)
  template <int P, int MODE>
  static void rasw(const Slab& sl, const float* S, const float* L, const double* r, const RasEpi& e, cudaStream_t s) {
    using W = LShape<P>;
    auto kern = k_rasw<P, MODE>;
    const int nctas = resident_ctas(kern, W::NT, W::smem());
    const int64_t need = (sl.elems() + W::WPC - 1) / W::WPC;
    kern<<<capped_grid(std::min<int64_t>(need, nctas)), W::NT, W::smem(), s>>>(sl, S, L, r, e);
  }
  template <int P>
  static void ras(const Slab& sl, const T* S, const T* L, const double* r, int mode, const RasEpi& e, cudaStream_t s) {
    if constexpr (sizeof(T) == 4 && P >= SEMLAB_RASW_MINP) {
      if (ras_warp() && sl.elems() < (int64_t(1) << 31)) {
        if (mode == 0) rasw<P, 0>(sl, S, L, r, e, s);
        else if (mode == 1) rasw<P, 1>(sl, S, L, r, e, s);
        else if (mode == 2) rasw<P, 2>(sl, S, L, r, e, s);
        else rasw<P, 3>(sl, S, L, r, e, s);
        return;
      }
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
  static void asm_(const Slab& sl, const T* S, const T* L, const double* r, void* boxes, double* out, cudaStream_t s) {
    using Sh = Shape<P, T>;
    const int grid = int((sl.elems() + Sh::EPC - 1) / Sh::EPC);
    prep(k_asm_boxes<P, T>, Sh::smem());
    k_asm_boxes<P, T><<<grid, Sh::NT, Sh::smem(), s>>>(sl, S, L, r, static_cast<T*>(boxes));
    const int64_t total = sl.Nx * sl.Ny * (int64_t(sl.ez1 - sl.ez0) * sl.q + 1);
    k_asm_sum<P, T><<<int(std::min<int64_t>((total + 255) / 256, 148 * 32)), 256, 0, s>>>(
        sl, static_cast<const T*>(boxes), out);
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
                   double* out, cudaStream_t s) {
  if (sl.elems() == 0) return 0;
  const int P = sl.q + 3;
  if (precision == 32) {
#define C32(PP) Launch<float>::asm_<PP>(sl, static_cast<const float*>(S), static_cast<const float*>(L), r, boxes, out, s)
    SB_FDM_SWITCH(P, C32)
#undef C32
  } else {
#define C64(PP) Launch<double>::asm_<PP>(sl, static_cast<const double*>(S), static_cast<const double*>(L), r, boxes, out, s)
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

}  // namespace sb
