// Shared internals of libsemlab_b200: error model, slab geometry, device buffers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace sb {

// Status codes of include/semlab_b200.h.
enum Code { kOk = 0, kInval = 1, kNumeric = 2, kCuda = 3, kNccl = 4 };

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
// std::invalid_argument / std::runtime_error of the reference map onto these two.
[[noreturn]] inline void invalid(const std::string& msg) { fail(kInval, msg); }
[[noreturn]] inline void numeric(const std::string& msg) { fail(kNumeric, msg); }

#define SB_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t err_ = (call);                                                             \
    if (err_ != cudaSuccess)                                                               \
      ::sb::fail(::sb::kCuda, std::string(#call) + ": " + cudaGetErrorString(err_) + " (" + \
                                  __FILE__ + ":" + std::to_string(__LINE__) + ")");        \
  } while (0)

// NCCL status -> sb::Error (kNccl); needs <nccl.h> in the including translation unit.
#define SB_NCCL(call)                                                                  \
  do {                                                                                 \
    ncclResult_t r_ = (call);                                                          \
    if (r_ != ncclSuccess) ::sb::fail(::sb::kNccl, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// Check the last launch (launch-configuration errors surface immediately; asynchronous
// faults surface at the next synchronising call).
#define SB_LAUNCH_CHECK() SB_CUDA(cudaGetLastError())

// One-time launch configuration (cudaFuncSetAttribute, occupancy-derived grid sizes) cached per
// (device, kernel): function attributes belong to a device's context, so a value computed on one
// GPU is never reused on another.
int per_device_once(const void* key, const std::function<int()>& init);

// Test/debug cap on the grid of the grid-stride (persistent) kernels: with a cap of 1-2 CTAs every
// warp runs many elements, which forces the multi-element paths of k_axw / k_rasw at small E.
// 0 = no cap (the default). Set through semlab_debug_set_grid_cap().
int grid_cap();
// Resident CTAs of a kernel over the whole device (occupancy x SMs), with its dynamic shared memory
// attribute set; cached per (device, kernel).
template <class K>
int resident_ctas(K kern, int threads, size_t smem) {
  return per_device_once(reinterpret_cast<const void*>(kern), [&] {
    if (smem > 48 * 1024)
      SB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0, dev = 0, sms = 0;
    SB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    SB_CUDA(cudaGetDevice(&dev));
    SB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return per_sm > 0 ? per_sm * sms : sms;
  });
}
// Sets a kernel's dynamic shared memory attribute once per device.
template <class K>
void smem_attr(K kern, size_t smem) {
  per_device_once(reinterpret_cast<const char*>(kern) + 1, [&] {  // key distinct from resident_ctas'
    SB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    return 1;
  });
}
// Test/debug: false forces GMRES to the reference's x += M (V y) form (semlab_debug_set_gmres_form).
bool gmres_flexible_allowed();
inline int capped_grid(int64_t grid) {
  const int c = grid_cap();
  return int(c > 0 && grid > c ? c : grid);
}

// Geometry of this rank's z-slab of the structured element grid, passed by value to kernels.
// Elements: e = ex + Ex (ey + Ey ez) globally (mesh.hpp:58-60); this rank owns element layers
// ez in [ez0, ez1). Lattice: x-fastest global index (sem_space.hpp:44-49); local vectors hold
// global planes z in [zlo, zlo + nzl), i.e. the slab's planes [ez0 q, ez1 q] plus one ghost
// plane across each internal slab boundary (the Schwarz halo, schwarz.cpp:159-168).
struct Slab {
  int q;            // polynomial order
  int Ex, Ey, Ez;   // global element counts
  int ez0, ez1;     // owned element layers
  int64_t Nx, Ny, Nz;  // global lattice points per axis
  int64_t zlo, nzl;    // local planes: global z of local plane 0, plane count
  int dirichlet;       // BcMode::Dirichlet
  int nranks_below, nranks_above;  // 1 if a neighbour slab exists below / above

  __host__ __device__ int64_t elems() const { return int64_t(Ex) * Ey * (ez1 - ez0); }
  __host__ __device__ int64_t n_local() const { return Nx * Ny * nzl; }
  __host__ __device__ int64_t lidx(int64_t x, int64_t y, int64_t z) const {
    return x + Nx * (y + Ny * (z - zlo));
  }
  __host__ __device__ bool masked(int64_t x, int64_t y, int64_t z) const {
    return dirichlet && (x == 0 || x == Nx - 1 || y == 0 || y == Ny - 1 || z == 0 || z == Nz - 1);
  }
  // Planes this rank owns for reductions: [ez0 q, ez1 q), plus the global top plane.
  __host__ __device__ int64_t own_z0() const { return int64_t(ez0) * q; }
  __host__ __device__ int64_t own_z1() const { return int64_t(ez1) * q + (ez1 == Ez ? 1 : 0); }
};

inline Slab make_slab(int q, int Ex, int Ey, int Ez, int rank, int nranks, bool dirichlet) {
  Slab s{};
  s.q = q;
  s.Ex = Ex;
  s.Ey = Ey;
  s.Ez = Ez;
  s.ez0 = int((int64_t(rank) * Ez) / nranks);
  s.ez1 = int((int64_t(rank + 1) * Ez) / nranks);
  s.Nx = int64_t(Ex) * q + 1;
  s.Ny = int64_t(Ey) * q + 1;
  s.Nz = int64_t(Ez) * q + 1;
  s.nranks_below = s.ez0 > 0 ? 1 : 0;
  s.nranks_above = s.ez1 < Ez ? 1 : 0;
  s.zlo = int64_t(s.ez0) * q - s.nranks_below;
  const int64_t zhi = int64_t(s.ez1) * q + s.nranks_above;
  s.nzl = zhi - s.zlo + 1;
  s.dirichlet = dirichlet ? 1 : 0;
  return s;
}

// Owning device buffer (cudaMalloc/cudaFree), move-only.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) SB_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void zero(cudaStream_t s) { if (n) SB_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s)); }
  void download(T* h, size_t count, cudaStream_t s) const {
    SB_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    SB_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  T* get() const { return p; }
};

}  // namespace sb
