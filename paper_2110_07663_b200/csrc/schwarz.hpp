// SchwarzSmoother host object (setup on the host, apply on the device).
#pragma once

#include "kernels_fdm.hpp"
#include "objects.hpp"

struct semlab_schwarz_s {
  semlab_space space = nullptr;
  int mode = SEMLAB_SCHWARZ_RAS;
  int precision = 32;
  int P = 0;
  sb::DevBuf<unsigned char> S, L, boxes;
  sb::DevBuf<double> cnt, xch;  // ASM on slabs: local counts (6 planes) and received sums/counts (8 planes)
  void asm_exchange(double* z);
  std::vector<double> hlen;  // 3 per local element
  std::vector<double> hlam;  // 3*P per local element (padded with 1)
  std::vector<int> hn;       // 3 per local element

  void build();
  // SchwarzSmoother::apply (schwarz.cpp:242-289): z = sum_e W_e R_e^T Abar_e^-1 R_e r.
  void apply(const double* r, double* z);
  // RAS with a fused owner epilogue (used by the Chebyshev driver).
  void ras(const double* r, int mode, const sb::RasEpi& e);
};
