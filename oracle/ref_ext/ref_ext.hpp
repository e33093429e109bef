// ORACLE TEST INFRASTRUCTURE — restated missing pieces on top of the reference's semlab API.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "semlab/amg.hpp"
#include "semlab/chebyshev.hpp"
#include "semlab/gll.hpp"
#include "semlab/krylov.hpp"
#include "semlab/mesh.hpp"
#include "semlab/schwarz.hpp"
#include "semlab/sem_space.hpp"

namespace semlab_ref {

semlab::FieldVector jacobi_inverse_diag(const semlab::SemSpace& s);
semlab::FieldVector build_rhs(const semlab::SemSpace& s, std::uint64_t seed);

struct Transfer {
  const semlab::SemSpace* f;
  const semlab::SemSpace* c;
  Eigen::MatrixXd J;
  Transfer(const semlab::SemSpace& fine, const semlab::SemSpace& coarse);
  semlab::FieldVector prolong(const semlab::FieldVector& uc) const;
  semlab::FieldVector restrict_(const semlab::FieldVector& rf) const;
};

class CoarseSolve {
 public:
  CoarseSolve(const semlab::SemSpace& s, const std::string& mode);  // Neumann space: zero-mean solve
  semlab::FieldVector solve(const semlab::FieldVector& r) const;
  const semlab::AmgHierarchy* amg() const { return amg_.get(); }

 private:
  const semlab::SemSpace* sp;
  std::string mode_;
  std::vector<Eigen::Index> free_;
  semlab::CsrMatrix A_;
  Eigen::LDLT<Eigen::MatrixXd> ldlt_;
  std::unique_ptr<semlab::AmgHierarchy> amg_;
};

class Pmg {
 public:
  // smoother: "jacobi" | "ras" | "asm" (Chebyshev-accelerated) | "ras_plain" | "asm_plain";
  // additive: the additive V-cycle without post-smoothing
  Pmg(const semlab::HexMesh& mesh, const std::vector<int>& orders, const std::string& smoother, int eta, double lmin,
      double lmax, const std::string& coarse, semlab::BcMode bc = semlab::BcMode::Dirichlet, bool additive = false);
  semlab::FieldVector vcycle(const semlab::FieldVector& b) const { return additive_ ? cycle_additive(0, b) : cycle(0, b); }
  semlab::LinOp as_linop() const;
  struct Level {
    semlab::LinOp A, S;
    std::unique_ptr<semlab::SchwarzSmoother> sch;
    std::unique_ptr<semlab::ChebyshevSmoother> cheb;
    double lam = 0.0;
  };
  std::vector<std::unique_ptr<semlab::SemSpace>> spaces;
  std::vector<Level> levels;
  std::vector<std::unique_ptr<Transfer>> transfers;

 private:
  semlab::FieldVector cycle(size_t l, const semlab::FieldVector& b) const;
  semlab::FieldVector cycle_additive(size_t l, const semlab::FieldVector& b) const;
  semlab::FieldVector smooth(size_t l, const semlab::FieldVector& b, const semlab::FieldVector* x) const;
  bool plain_ = false, additive_ = false;
  std::unique_ptr<CoarseSolve> coarse_;
};

semlab::GmresStats pcg_solve(const semlab::LinOp& A, const semlab::LinOp& M, const semlab::FieldVector& b,
                             semlab::FieldVector& x, double tol, int max_iters);

}  // namespace semlab_ref
