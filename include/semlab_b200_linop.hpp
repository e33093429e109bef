// semlab_b200_linop.hpp — the binding a maintainer of the reference adds to keep existing semlab
// code (its Eigen types, LinOp closures and its own krylov.cpp gmres_solve) and swap only the heavy
// operators for B200 ones. Wraps any C-ABI operator handle (semlab_op: apply_A, a Schwarz
// smoother, the pMG V-cycle, ...) as a reference semlab::LinOp (types.hpp:13). Each application
// copies the host vector to the device and back (one PCIe round trip per operator call); use the
// device-resident API (semlab_b200.hpp / the C-ABI) for the production solve.
//
// Requires the reference's <semlab/types.hpp> (Eigen) and this repo's include/semlab_b200.h.
// Built and run against the reference's own gmres_solve by tests/test_ref_binding_gpu.py.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>

#include "semlab/types.hpp"
#include "semlab_b200.h"

inline semlab::LinOp b200_linop(semlab_op op, int64_t n) {
  struct Buf {
    double* in = nullptr;
    double* out = nullptr;
    ~Buf() {
      cudaFree(in);
      cudaFree(out);
    }
  };
  auto buf = std::make_shared<Buf>();
  if (cudaMalloc(&buf->in, size_t(n) * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&buf->out, size_t(n) * sizeof(double)) != cudaSuccess)
    throw std::runtime_error("b200_linop: cudaMalloc failed");
  return [op, n, buf](const Eigen::VectorXd& in, Eigen::VectorXd& out) {
    if (in.size() != n) throw std::invalid_argument("b200_linop: vector length differs from the operator's n");
    out.resize(n);
    cudaMemcpy(buf->in, in.data(), size_t(n) * sizeof(double), cudaMemcpyHostToDevice);
    if (semlab_op_apply(op, buf->in, buf->out) != SEMLAB_OK) throw std::runtime_error(semlab_last_error());
    cudaMemcpy(out.data(), buf->out, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost);
  };
}
