// p-multigrid hierarchy (RESTATED: pmg.cpp is missing in the reference; SPEC.md:308-373,
// PAPER.md Alg. 1) and its coarse solvers: exact (dense inverse) or aggregation AMG
// (setup restated from amg.cpp:12-129, V-cycle on the device).
#pragma once

#include <vector>

#include "kernels_mg.hpp"
#include "objects.hpp"
#include "schwarz.hpp"
#include "solvers.hpp"

namespace sb {

struct HostCsr {  // row-major sparse, columns ascending within a row
  int64_t n = 0, m = 0;
  std::vector<int64_t> ptr;
  std::vector<int> idx;
  std::vector<double> val;
  double coeff(int64_t i, int64_t j) const;
};

// Free-dof block of the assembled operator of a Dirichlet space (row/col = free index).
HostCsr assemble_free_matrix(semlab_space sp);

struct AmgLevelHost {
  HostCsr A;
  std::vector<double> inv_diag;
  std::vector<int> agg;  // empty on the coarsest level
  int n_agg = 0;
};

// AmgHierarchy::build (amg.cpp:69-129) with the default AmgOptions (amg.hpp:16-25).
std::vector<AmgLevelHost> amg_build(const HostCsr& A, double theta = 0.25, int max_levels = 25,
                                    int max_coarse_size = 200);
std::vector<int> amg_aggregate(const HostCsr& A, double theta, int& n_agg);
// Dense SPD inverse (Cholesky), column-major; false if not positive definite.
bool dense_spd_inverse(int64_t n, std::vector<double>& M);
int device_spd_inverse(semlab_ctx ctx, int64_t n, const std::vector<double>& M, DevBuf<double>& inv);

struct CoarseSolver {
  semlab_space sp = nullptr;
  int mode = SEMLAB_COARSE_DIRECT;
  int64_t nfree = 0;
  DevBuf<double> rf, zf;
  // direct
  DevBuf<double> Minv;
  // amg
  struct Lev {
    int64_t n = 0, nc = 0;
    DevBuf<int64_t> ptr, aptr;
    DevBuf<int> idx, agg, amem;
    DevBuf<double> val, inv_diag, r, z, t;
  };
  std::vector<Lev> lev;
  DevBuf<double> coarse_inv;
  int64_t coarse_n = 0;
  double omega = 0.9;
  DevBuf<double> gsend, grecv, rfull, zfull;  // distributed gather of the coarse residual
  bool neumann = false;  // singular coarse problem: solve on the zero-mean subspace
  void build(semlab_space space, int mode);
  void build_amg(semlab_space space, const HostCsr& A);  // AMG hierarchy of a given matrix
  void solve(const double* r_full, double* z_full);
  void solve_dist(semlab_space dist_space, const double* r_loc, double* z_loc);
  void amg_cycle(int l, const double* r, double* z);
};

}  // namespace sb

struct semlab_pmg_s {
  semlab_ctx ctx = nullptr;
  semlab_mesh mesh = nullptr;
  std::vector<int> orders;
  int smoother = SEMLAB_SMOOTHER_JACOBI, cheb_order = 2, precision = 32, coarse_mode = SEMLAB_COARSE_DIRECT;
  int bc = SEMLAB_BC_DIRICHLET, cycle_mode = SEMLAB_CYCLE_STANDARD;
  bool plain() const { return smoother == SEMLAB_SMOOTHER_RAS_PLAIN || smoother == SEMLAB_SMOOTHER_ASM_PLAIN; }
  double lmin = 0.1, lmax = 1.1;
  struct Level {
    semlab_space sp = nullptr;
    semlab_schwarz sch = nullptr;
    semlab_op A = nullptr, S = nullptr;
    semlab_cheby cheb = nullptr;
    double lam = 0.0;
    sb::DevBuf<double> b, x, r, t;
  };
  std::vector<Level> lv;
  std::vector<sb::Jmat> J;  // J[l]: level l+1 (coarse) -> level l (fine)
  sb::DevBuf<double> tA, tB;  // transfer scratch
  sb::CoarseSolver coarse;
  semlab_space coarse_full = nullptr;  // whole-mesh p=1 space for the redundant coarse solve
  ~semlab_pmg_s();
  void build();
  void prolong(int l, const double* coarse_v, double* fine_v, bool add = false);  // add: fine_v += P coarse_v
  void restrict_(int l, const double* fine_v, double* coarse_v, const double* sub_from = nullptr);  // Pᵀ (sub_from - fine_v) if given
  void vcycle(const double* b, double* z);
  void cycle(int l);
  void cycle_additive(int l);
  void run_body();  // cycle(0) or cycle_additive(0)
  void smooth(int l, bool x_is_zero);  // x_l <- smoother(b_l, x_l)
  void run_cycle();  // cycle(0), replayed as a captured CUDA graph after one eager call
  cudaGraphExec_t graph_exec = nullptr;
  int graph_state = 0;  // 0 not run, 1 warmed up, 2 captured, -1 eager only
  int64_t graph_launches = 0;
};
