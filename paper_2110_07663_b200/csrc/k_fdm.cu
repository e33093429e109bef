// Overlapping Schwarz smoother kernels (sm_100a), replacing SchwarzSmoother::apply and
// fdm_solve (schwarz.cpp:228-289).
//
// One CTA per element. The extended box (order+3 per direction, padded; boundary elements are
// smaller and padded with zero S rows) is extracted from the global lattice vector straight into
// shared memory (sites outside the element core in more than one direction are zero-filled,
// schwarz.cpp:255-265), transformed by S_x^T, S_y^T, S_z^T (one register-resident line per
// thread, S broadcast from shared memory), scaled by inv_D = 1/(lx_i + ly_j + lz_k) recomputed
// from the 3*(order+3) eigenvalues (schwarz.cpp:92-108; saves the (order+3)^3 table), and
// transformed back. RAS: the element writes exactly the lattice nodes it owns (lowest element
// whose core holds the node, schwarz.cpp:114-127) — a race-free owner write that can carry the
// whole Chebyshev vector update. ASM: per-element boxes are written out and summed per node in
// ascending element id (deterministic, the reference's order) then weighted by 1/count.
#include "device.cuh"
#include "kernels_fdm.hpp"

namespace sb {

namespace {

struct Box1D {  // extended-box geometry of one element along one axis (schwarz.cpp:155-169)
  int n, lo, gl, gr, own_lo, own_hi;  // own_*: box indices this element owns (RAS, inclusive)
};

__device__ __forceinline__ Box1D box1d(int e_d, int E_d, int q, bool dirichlet, int has_lower_rank,
                                       int has_upper_rank) {
  // has_*_rank: the neighbour element along this axis lives on another rank (z only)
  Box1D b;
  const bool left_int = e_d > 0 || has_lower_rank;
  const bool right_int = e_d < E_d - 1 || has_upper_rank;
  const int i0 = (!left_int && dirichlet) ? 1 : 0;
  const int i1 = (!right_int && dirichlet) ? q - 1 : q;
  b.gl = left_int ? 1 : 0;
  b.gr = right_int ? 1 : 0;
  b.n = (i1 - i0 + 1) + b.gl + b.gr;
  b.lo = e_d * q + i0 - b.gl;
  // owned element-local indices: [max(i0, left_int ? 1 : 0), i1]; box index a = i - i0 + gl
  const int first = left_int ? 1 : i0;
  b.own_lo = first - i0 + b.gl;
  b.own_hi = i1 - i0 + b.gl;
  return b;
}

__device__ __forceinline__ bool ghost(const Box1D& b, int a) { return (b.gl && a == 0) || (b.gr && a == b.n - 1); }

// out[a'] = sum_a M(a, a') in[a]  (transpose=true: S^T)  or  out[a] = sum_a' M(a, a') in[a'] (S)
template <int P, class T, bool TRANS>
__device__ __forceinline__ void line(const T* __restrict__ M /* P x P row-major M(a,a')=M[a*P+a'] */,
                                     const T (&in)[P], T (&out)[P]) {
#pragma unroll
  for (int o = 0; o < P; ++o) out[o] = T(0);
#pragma unroll
  for (int a = 0; a < P; ++a) {
#pragma unroll
    for (int o = 0; o < P; ++o) {
      if (TRANS)
        out[o] = fma(M[a * P + o], in[a], out[o]);
      else
        out[a] = fma(M[a * P + o], in[o], out[a]);
    }
  }
}

// Apply the box solve in shared memory: box[c][b][a] (P^3, stride P) -> box (in place via tmp).
template <int P, class T>
__device__ void fdm_box(T* __restrict__ box, T* __restrict__ tmp, const T* __restrict__ sS, const T* __restrict__ sL,
                        int tid, int nthreads) {
  constexpr int P2 = P * P;
  T in[P], out[P];
  // x: S_x^T along a, lines (b,c)
  for (int l = tid; l < P2; l += nthreads) {
    const int b = l % P, c = l / P;
#pragma unroll
    for (int a = 0; a < P; ++a) in[a] = box[c * P2 + b * P + a];
    line<P, T, true>(sS + 0 * P2, in, out);
#pragma unroll
    for (int a = 0; a < P; ++a) tmp[c * P2 + b * P + a] = out[a];
  }
  __syncthreads();
  // y: S_y^T along b, lines (a,c)
  for (int l = tid; l < P2; l += nthreads) {
    const int a = l % P, c = l / P;
#pragma unroll
    for (int b = 0; b < P; ++b) in[b] = tmp[c * P2 + b * P + a];
    line<P, T, true>(sS + 1 * P2, in, out);
#pragma unroll
    for (int b = 0; b < P; ++b) box[c * P2 + b * P + a] = out[b];
  }
  __syncthreads();
  // z: S_z^T along c, scale by inv_D, then S_z back (lines (a,b))
  for (int l = tid; l < P2; l += nthreads) {
    const int a = l % P, b = l / P;
#pragma unroll
    for (int c = 0; c < P; ++c) in[c] = box[c * P2 + b * P + a];
    line<P, T, true>(sS + 2 * P2, in, out);
    const T lab = sL[0 * P + a] + sL[1 * P + b];
#pragma unroll
    for (int c = 0; c < P; ++c) out[c] = out[c] / (lab + sL[2 * P + c]);
    line<P, T, false>(sS + 2 * P2, out, in);
#pragma unroll
    for (int c = 0; c < P; ++c) box[c * P2 + b * P + a] = in[c];
  }
  __syncthreads();
  // y back
  for (int l = tid; l < P2; l += nthreads) {
    const int a = l % P, c = l / P;
#pragma unroll
    for (int b = 0; b < P; ++b) in[b] = box[c * P2 + b * P + a];
    line<P, T, false>(sS + 1 * P2, in, out);
#pragma unroll
    for (int b = 0; b < P; ++b) tmp[c * P2 + b * P + a] = out[b];
  }
  __syncthreads();
  // x back
  for (int l = tid; l < P2; l += nthreads) {
    const int b = l % P, c = l / P;
#pragma unroll
    for (int a = 0; a < P; ++a) in[a] = tmp[c * P2 + b * P + a];
    line<P, T, false>(sS + 0 * P2, in, out);
#pragma unroll
    for (int a = 0; a < P; ++a) box[c * P2 + b * P + a] = out[a];
  }
  __syncthreads();
}

template <int P, class T>
__device__ __forceinline__ void load_factors(const T* __restrict__ S, const T* __restrict__ L, int64_t el, T* sS, T* sL,
                                             int tid, int nthreads) {
  const T* Se = S + el * 3 * P * P;
  for (int t = tid; t < 3 * P * P; t += nthreads) sS[t] = Se[t];
  const T* Le = L + el * 3 * P;
  for (int t = tid; t < 3 * P; t += nthreads) sL[t] = Le[t];
}

// ---------------------------------------------------------------- RAS (+ fused Chebyshev update)
template <int P, class T, int MODE>
__global__ void __launch_bounds__(128) k_ras(const Slab sl, const T* __restrict__ S, const T* __restrict__ L,
                                             const double* __restrict__ r, RasEpi epi) {
  constexpr int P2 = P * P, P3 = P2 * P;
  __shared__ T sS[3 * P2];
  __shared__ T sL[3 * P];
  __shared__ T box[P3];
  __shared__ T tmp[P3];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t el = blockIdx.x;
  const int q = sl.q;
  const int ex = int(el % sl.Ex), ey = int((el / sl.Ex) % sl.Ey), ez = sl.ez0 + int(el / (int64_t(sl.Ex) * sl.Ey));
  const bool dir = sl.dirichlet != 0;
  const Box1D bx = box1d(ex, sl.Ex, q, dir, 0, 0);
  const Box1D by = box1d(ey, sl.Ey, q, dir, 0, 0);
  const Box1D bz = box1d(ez, sl.Ez, q, dir, 0, 0);
  load_factors<P, T>(S, L, el, sS, sL, tid, nt);
  for (int t = tid; t < P3; t += nt) {
    const int a = t % P, b = (t / P) % P, c = t / P2;
    T v = T(0);
    if (a < bx.n && b < by.n && c < bz.n) {
      const int out = int(ghost(bx, a)) + int(ghost(by, b)) + int(ghost(bz, c));
      if (out <= 1) v = T(r[sl.lidx(bx.lo + a, by.lo + b, bz.lo + c)]);
    }
    box[t] = v;
  }
  __syncthreads();
  fdm_box<P, T>(box, tmp, sS, sL, tid, nt);
  const int wa = bx.own_hi - bx.own_lo + 1, wb = by.own_hi - by.own_lo + 1, wc = bz.own_hi - bz.own_lo + 1;
  for (int t = tid; t < wa * wb * wc; t += nt) {
    const int a = bx.own_lo + t % wa, b = by.own_lo + (t / wa) % wb, c = bz.own_lo + t / (wa * wb);
    const int64_t g = sl.lidx(bx.lo + a, by.lo + b, bz.lo + c);
    const double z = double(box[c * P2 + b * P + a]);
    if (MODE == 0) {
      epi.out[g] = z;
    } else if (MODE == 1) {  // Chebyshev init: r = S t, d = r / theta  (chebyshev.cpp:82-84)
      epi.r[g] = z;
      epi.d[g] = z / epi.c1;
    } else {  // Chebyshev step: x += d; r -= S A d; d = c1 d + c2 r  (chebyshev.cpp:86-92)
      const double dg = epi.d[g];
      epi.x[g] += dg;
      const double rg = epi.r[g] - z;
      epi.r[g] = rg;
      epi.d[g] = epi.c1 * dg + epi.c2 * rg;
    }
  }
}

// ---------------------------------------------------------------- ASM boxes + deterministic sum
template <int P, class T>
__global__ void __launch_bounds__(128) k_asm_boxes(const Slab sl, const T* __restrict__ S, const T* __restrict__ L,
                                                   const double* __restrict__ r, T* __restrict__ boxes) {
  constexpr int P2 = P * P, P3 = P2 * P;
  __shared__ T sS[3 * P2];
  __shared__ T sL[3 * P];
  __shared__ T box[P3];
  __shared__ T tmp[P3];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t el = blockIdx.x;
  const int q = sl.q;
  const int ex = int(el % sl.Ex), ey = int((el / sl.Ex) % sl.Ey), ez = sl.ez0 + int(el / (int64_t(sl.Ex) * sl.Ey));
  const bool dir = sl.dirichlet != 0;
  const Box1D bx = box1d(ex, sl.Ex, q, dir, 0, 0), by = box1d(ey, sl.Ey, q, dir, 0, 0), bz = box1d(ez, sl.Ez, q, dir, 0, 0);
  load_factors<P, T>(S, L, el, sS, sL, tid, nt);
  for (int t = tid; t < P3; t += nt) {
    const int a = t % P, b = (t / P) % P, c = t / P2;
    T v = T(0);
    if (a < bx.n && b < by.n && c < bz.n) {
      const int out = int(ghost(bx, a)) + int(ghost(by, b)) + int(ghost(bz, c));
      if (out <= 1) v = T(r[sl.lidx(bx.lo + a, by.lo + b, bz.lo + c)]);
    }
    box[t] = v;
  }
  __syncthreads();
  fdm_box<P, T>(box, tmp, sS, sL, tid, nt);
  for (int t = tid; t < P3; t += nt) boxes[el * P3 + t] = box[t];
}

// out[g] = w(g) * sum over elements whose participating box covers g (ascending id), w = 1/count
template <int P, class T>
__global__ void k_asm_sum(const Slab sl, const T* __restrict__ boxes, double* __restrict__ out) {
  constexpr int P2 = P * P, P3 = P2 * P;
  const int q = sl.q;
  const bool dir = sl.dirichlet != 0;
  const int64_t z0 = int64_t(sl.ez0) * q, nz = int64_t(sl.ez1 - sl.ez0) * q + 1;
  const int64_t total = sl.Nx * sl.Ny * nz;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t x = t % sl.Nx, y = (t / sl.Nx) % sl.Ny, z = z0 + t / (sl.Nx * sl.Ny);
    // candidate elements per axis: at most two boxes cover a lattice coordinate
    int ce[3][3], ca[3][3], cg[3][3], cn[3] = {0, 0, 0};
    const int64_t coord[3] = {x, y, z};
    const int Ed[3] = {sl.Ex, sl.Ey, sl.Ez};
    const int lo_e[3] = {0, 0, sl.ez0}, hi_e[3] = {sl.Ex, sl.Ey, sl.ez1};
    for (int d = 0; d < 3; ++d) {
      const int base = int(coord[d] / q);
      for (int e = base - 1; e <= base + 1; ++e) {
        if (e < lo_e[d] || e >= hi_e[d]) continue;
        const Box1D b = box1d(e, Ed[d], q, dir, 0, 0);
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
__global__ void __launch_bounds__(128) k_fdm_boxes(const T* __restrict__ S, const T* __restrict__ L,
                                                   const double* __restrict__ in, double* __restrict__ outb) {
  constexpr int P2 = P * P, P3 = P2 * P;
  __shared__ T sS[3 * P2];
  __shared__ T sL[3 * P];
  __shared__ T box[P3];
  __shared__ T tmp[P3];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t el = blockIdx.x;
  load_factors<P, T>(S, L, el, sS, sL, tid, nt);
  for (int t = tid; t < P3; t += nt) box[t] = T(in[el * P3 + t]);
  __syncthreads();
  fdm_box<P, T>(box, tmp, sS, sL, tid, nt);
  for (int t = tid; t < P3; t += nt) outb[el * P3 + t] = double(box[t]);
}

template <class T>
struct Launch {
  template <int P>
  static void ras(const Slab& sl, const T* S, const T* L, const double* r, int mode, const RasEpi& e, cudaStream_t s) {
    const int grid = int(sl.elems());
    if (mode == 0) k_ras<P, T, 0><<<grid, 128, 0, s>>>(sl, S, L, r, e);
    else if (mode == 1) k_ras<P, T, 1><<<grid, 128, 0, s>>>(sl, S, L, r, e);
    else k_ras<P, T, 2><<<grid, 128, 0, s>>>(sl, S, L, r, e);
  }
  template <int P>
  static void asm_(const Slab& sl, const T* S, const T* L, const double* r, void* boxes, double* out, cudaStream_t s) {
    k_asm_boxes<P, T><<<int(sl.elems()), 128, 0, s>>>(sl, S, L, r, static_cast<T*>(boxes));
    const int64_t total = sl.Nx * sl.Ny * (int64_t(sl.ez1 - sl.ez0) * sl.q + 1);
    k_asm_sum<P, T><<<int(std::min<int64_t>((total + 255) / 256, 148 * 32)), 256, 0, s>>>(
        sl, static_cast<const T*>(boxes), out);
  }
  template <int P>
  static void boxes(int64_t E, const T* S, const T* L, const double* in, double* out, cudaStream_t s) {
    k_fdm_boxes<P, T><<<int(E), 128, 0, s>>>(S, L, in, out);
  }
};

#define SB_FDM_SWITCH(P_, CALL)                                                     \
  switch (P_) {                                                                      \
    case 4: CALL(4); break;                                                          \
    case 5: CALL(5); break;                                                          \
    case 6: CALL(6); break;                                                          \
    case 7: CALL(7); break;                                                          \
    case 8: CALL(8); break;                                                          \
    case 9: CALL(9); break;                                                          \
    case 10: CALL(10); break;                                                        \
    case 11: CALL(11); break;                                                        \
    case 12: CALL(12); break;                                                        \
    default: invalid("SchwarzSmoother: device kernels support orders 1..9");        \
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

int64_t launch_fdm_boxes(int q, int64_t E, int precision, const void* S, const void* L, const double* in, double* out,
                         cudaStream_t s) {
  if (E == 0) return 0;
  const int P = q + 3;
  if (precision == 32) {
#define C32(PP) Launch<float>::boxes<PP>(E, static_cast<const float*>(S), static_cast<const float*>(L), in, out, s)
    SB_FDM_SWITCH(P, C32)
#undef C32
  } else {
#define C64(PP) Launch<double>::boxes<PP>(E, static_cast<const double*>(S), static_cast<const double*>(L), in, out, s)
    SB_FDM_SWITCH(P, C64)
#undef C64
  }
  SB_LAUNCH_CHECK();
  return 1;
}

}  // namespace sb
