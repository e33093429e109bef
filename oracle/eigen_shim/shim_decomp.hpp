// ORACLE TEST INFRASTRUCTURE — decompositions and sparse matrices of the Eigen-API shim.
#pragma once

#include <complex>
#include <map>
#include <numeric>

namespace Eigen {

namespace shim {

// cyclic Jacobi for a symmetric n x n matrix (column-major): A = Q diag Q^T
inline void sym_jacobi(Index n, std::vector<double>& A, std::vector<double>& Q) {
  Q.assign(size_t(n * n), 0.0);
  for (Index i = 0; i < n; ++i) Q[size_t(i + n * i)] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (Index i = 0; i < n; ++i)
      for (Index j = 0; j < n; ++j) {
        tot += A[size_t(i + n * j)] * A[size_t(i + n * j)];
        if (i != j) off += A[size_t(i + n * j)] * A[size_t(i + n * j)];
      }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (Index p = 0; p < n - 1; ++p)
      for (Index q = p + 1; q < n; ++q) {
        const double apq = A[size_t(p + n * q)];
        if (apq == 0.0) continue;
        const double theta = (A[size_t(q + n * q)] - A[size_t(p + n * p)]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (Index k = 0; k < n; ++k) {
          const double akp = A[size_t(k + n * p)], akq = A[size_t(k + n * q)];
          A[size_t(k + n * p)] = c * akp - s * akq;
          A[size_t(k + n * q)] = s * akp + c * akq;
        }
        for (Index k = 0; k < n; ++k) {
          const double apk = A[size_t(p + n * k)], aqk = A[size_t(q + n * k)];
          A[size_t(p + n * k)] = c * apk - s * aqk;
          A[size_t(q + n * k)] = s * apk + c * aqk;
        }
        for (Index k = 0; k < n; ++k) {
          const double qkp = Q[size_t(k + n * p)], qkq = Q[size_t(k + n * q)];
          Q[size_t(k + n * p)] = c * qkp - s * qkq;
          Q[size_t(k + n * q)] = s * qkp + c * qkq;
        }
      }
  }
}

// Francis double-shift QR eigenvalues of a general real matrix (row-major working copy).
inline std::vector<std::complex<double>> eigenvalues_general(Index n, std::vector<double> a /* row-major */) {
  auto A = [&](Index i, Index j) -> double& { return a[size_t(i * n + j)]; };
  for (Index m = 1; m < n - 1; ++m) {  // reduce to Hessenberg
    double x = 0.0;
    Index i = m;
    for (Index j = m; j < n; ++j)
      if (std::abs(A(j, m - 1)) > std::abs(x)) { x = A(j, m - 1); i = j; }
    if (i != m) {
      for (Index j = m - 1; j < n; ++j) std::swap(A(i, j), A(m, j));
      for (Index j = 0; j < n; ++j) std::swap(A(j, i), A(j, m));
    }
    if (x != 0.0)
      for (i = m + 1; i < n; ++i) {
        double y = A(i, m - 1);
        if (y != 0.0) {
          y /= x;
          A(i, m - 1) = y;
          for (Index j = m; j < n; ++j) A(i, j) -= y * A(m, j);
          for (Index j = 0; j < n; ++j) A(j, m) += y * A(j, i);
        }
      }
  }
  for (Index i = 2; i < n; ++i)
    for (Index j = 0; j < i - 1; ++j) A(i, j) = 0.0;
  std::vector<double> wr(size_t(n), 0.0), wi(size_t(n), 0.0);
  double anorm = 0.0;
  for (Index i = 0; i < n; ++i)
    for (Index j = std::max<Index>(i - 1, 0); j < n; ++j) anorm += std::abs(A(i, j));
  Index nn = n - 1, l = 0;
  double t = 0.0, p = 0, q = 0, r = 0, s = 0, w = 0, x = 0, y = 0, z = 0;
  auto sign = [](double aa, double bb) { return bb >= 0.0 ? std::abs(aa) : -std::abs(aa); };
  while (nn >= 0) {
    int its = 0;
    do {
      for (l = nn; l >= 1; l--) {
        s = std::abs(A(l - 1, l - 1)) + std::abs(A(l, l));
        if (s == 0.0) s = anorm;
        if (std::abs(A(l, l - 1)) + s == s) { A(l, l - 1) = 0.0; break; }
      }
      x = A(nn, nn);
      if (l == nn) {
        wr[size_t(nn)] = x + t;
        wi[size_t(nn--)] = 0.0;
      } else {
        y = A(nn - 1, nn - 1);
        w = A(nn, nn - 1) * A(nn - 1, nn);
        if (l == nn - 1) {
          p = 0.5 * (y - x);
          q = p * p + w;
          z = std::sqrt(std::abs(q));
          x += t;
          if (q >= 0.0) {
            z = p + sign(z, p);
            wr[size_t(nn - 1)] = wr[size_t(nn)] = x + z;
            if (z != 0.0) wr[size_t(nn)] = x - w / z;
            wi[size_t(nn - 1)] = wi[size_t(nn)] = 0.0;
          } else {
            wr[size_t(nn - 1)] = wr[size_t(nn)] = x + p;
            wi[size_t(nn - 1)] = -(wi[size_t(nn)] = z);
          }
          nn -= 2;
        } else {
          if (its == 60) throw std::runtime_error("EigenSolver shim: no convergence");
          if (its == 10 || its == 20) {
            t += x;
            for (Index i = 0; i <= nn; i++) A(i, i) -= x;
            s = std::abs(A(nn, nn - 1)) + std::abs(A(nn - 1, nn - 2));
            y = x = 0.75 * s;
            w = -0.4375 * s * s;
          }
          ++its;
          Index m;
          for (m = nn - 2; m >= l; m--) {
            z = A(m, m);
            r = x - z;
            s = y - z;
            p = (r * s - w) / A(m + 1, m) + A(m, m + 1);
            q = A(m + 1, m + 1) - z - r - s;
            r = A(m + 2, m + 1);
            s = std::abs(p) + std::abs(q) + std::abs(r);
            p /= s; q /= s; r /= s;
            if (m == l) break;
            const double u = std::abs(A(m, m - 1)) * (std::abs(q) + std::abs(r));
            const double v = std::abs(p) * (std::abs(A(m - 1, m - 1)) + std::abs(z) + std::abs(A(m + 1, m + 1)));
            if (u + v == v) break;
          }
          for (Index i = m + 2; i <= nn; i++) {
            A(i, i - 2) = 0.0;
            if (i != m + 2) A(i, i - 3) = 0.0;
          }
          for (Index k = m; k <= nn - 1; k++) {
            if (k != m) {
              p = A(k, k - 1);
              q = A(k + 1, k - 1);
              r = 0.0;
              if (k != nn - 1) r = A(k + 2, k - 1);
              if ((x = std::abs(p) + std::abs(q) + std::abs(r)) != 0.0) { p /= x; q /= x; r /= x; }
            }
            if ((s = sign(std::sqrt(p * p + q * q + r * r), p)) != 0.0) {
              if (k == m) {
                if (l != m) A(k, k - 1) = -A(k, k - 1);
              } else {
                A(k, k - 1) = -s * x;
              }
              p += s; x = p / s; y = q / s; z = r / s; q /= p; r /= p;
              for (Index j = k; j <= nn; j++) {
                p = A(k, j) + q * A(k + 1, j);
                if (k != nn - 1) { p += r * A(k + 2, j); A(k + 2, j) -= p * z; }
                A(k + 1, j) -= p * y;
                A(k, j) -= p * x;
              }
              const Index mmin = nn < k + 3 ? nn : k + 3;
              for (Index i = l; i <= mmin; i++) {
                p = x * A(i, k) + y * A(i, k + 1);
                if (k != nn - 1) { p += z * A(i, k + 2); A(i, k + 2) -= p * r; }
                A(i, k + 1) -= p * q;
                A(i, k) -= p;
              }
            }
          }
        }
      }
    } while (nn >= 0 && l < nn - 1);
  }
  std::vector<std::complex<double>> ev(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) ev[size_t(i)] = {wr[size_t(i)], wi[size_t(i)]};
  return ev;
}

}  // namespace shim

// ---------------------------------------------------------------------------------- eigen solvers
template <class M>
class GeneralizedSelfAdjointEigenSolver {
 public:
  GeneralizedSelfAdjointEigenSolver(const MatrixXd& A, const MatrixXd& B) { compute(A, B); }
  ComputationInfo info() const { return info_; }
  const MatrixXd& eigenvectors() const { return S_; }
  const VectorXd& eigenvalues() const { return lam_; }

 private:
  void compute(const MatrixXd& A, const MatrixXd& B) {  // B = L L^T, C = L^-1 A L^-T = Q D Q^T, S = L^-T Q
    const Index n = A.rows();
    std::vector<double> L(size_t(n * n), 0.0);
    for (Index j = 0; j < n; ++j) {
      double d = B(j, j);
      for (Index k = 0; k < j; ++k) d -= L[size_t(j + n * k)] * L[size_t(j + n * k)];
      if (!(d > 0.0)) { info_ = NumericalIssue; return; }
      L[size_t(j + n * j)] = std::sqrt(d);
      for (Index i = j + 1; i < n; ++i) {
        double s = B(i, j);
        for (Index k = 0; k < j; ++k) s -= L[size_t(i + n * k)] * L[size_t(j + n * k)];
        L[size_t(i + n * j)] = s / L[size_t(j + n * j)];
      }
    }
    std::vector<double> T(size_t(n * n)), C(size_t(n * n)), Q;
    for (Index c = 0; c < n; ++c)
      for (Index i = 0; i < n; ++i) {
        double s = A(i, c);
        for (Index k = 0; k < i; ++k) s -= L[size_t(i + n * k)] * T[size_t(k + n * c)];
        T[size_t(i + n * c)] = s / L[size_t(i + n * i)];
      }
    for (Index r = 0; r < n; ++r)
      for (Index i = 0; i < n; ++i) {
        double s = T[size_t(r + n * i)];
        for (Index k = 0; k < i; ++k) s -= L[size_t(i + n * k)] * C[size_t(r + n * k)];
        C[size_t(r + n * i)] = s / L[size_t(i + n * i)];
      }
    for (Index i = 0; i < n; ++i)
      for (Index j = i + 1; j < n; ++j) C[size_t(i + n * j)] = C[size_t(j + n * i)] = 0.5 * (C[size_t(i + n * j)] + C[size_t(j + n * i)]);
    shim::sym_jacobi(n, C, Q);
    std::vector<Index> ord(static_cast<size_t>(n));
    std::iota(ord.begin(), ord.end(), Index(0));
    std::sort(ord.begin(), ord.end(), [&](Index a, Index b) { return C[size_t(a + n * a)] < C[size_t(b + n * b)]; });
    lam_.resize(n);
    S_.resize(n, n);
    for (Index cc = 0; cc < n; ++cc) {
      const Index c = ord[size_t(cc)];
      lam_[cc] = C[size_t(c + n * c)];
      for (Index i = n - 1; i >= 0; --i) {
        double s = Q[size_t(i + n * c)];
        for (Index k = i + 1; k < n; ++k) s -= L[size_t(k + n * i)] * S_(k, cc);
        S_(i, cc) = s / L[size_t(i + n * i)];
      }
    }
    info_ = Success;
  }
  ComputationInfo info_ = NumericalIssue;
  MatrixXd S_;
  VectorXd lam_;
};

struct ComplexVector {
  std::vector<std::complex<double>> v;
  VectorXd cwiseAbs() const {
    VectorXd a(Index(v.size()));
    for (size_t i = 0; i < v.size(); ++i) a[Index(i)] = std::abs(v[i]);
    return a;
  }
  Index size() const { return Index(v.size()); }
  std::complex<double> operator[](Index i) const { return v[size_t(i)]; }
};

template <class M>
class EigenSolver {
 public:
  explicit EigenSolver(const MatrixXd& H) {
    const Index n = H.rows();
    std::vector<double> a(size_t(n * n));
    for (Index i = 0; i < n; ++i)
      for (Index j = 0; j < n; ++j) a[size_t(i * n + j)] = H(i, j);
    ev_.v = shim::eigenvalues_general(n, a);
  }
  const ComplexVector& eigenvalues() const { return ev_; }

 private:
  ComplexVector ev_;
};

template <class M>
class JacobiSVD {  // singular values of a 3x3 matrix: sqrt(eig(J^T J)), descending
 public:
  explicit JacobiSVD(const Matrix3d& J) {
    std::vector<double> A(9), Q;
    for (Index i = 0; i < 3; ++i)
      for (Index j = 0; j < 3; ++j) {
        double s = 0.0;
        for (Index k = 0; k < 3; ++k) s += J(k, i) * J(k, j);
        A[size_t(i + 3 * j)] = s;
      }
    shim::sym_jacobi(3, A, Q);
    double e[3] = {A[0], A[4], A[8]};
    std::sort(e, e + 3, [](double a, double b) { return a > b; });
    for (int i = 0; i < 3; ++i) sv_[i] = std::sqrt(std::max(0.0, e[i]));
  }
  const Vector3d& singularValues() const { return sv_; }

 private:
  Vector3d sv_;
};

template <class M>
class LDLT {  // SPD systems: L D L^T without pivoting
 public:
  LDLT() = default;
  void compute(const MatrixXd& A) {
    n_ = A.rows();
    L_ = A;
    d_.assign(size_t(n_), 0.0);
    info_ = Success;
    for (Index j = 0; j < n_; ++j) {
      double dj = L_(j, j);
      for (Index k = 0; k < j; ++k) dj -= L_(j, k) * L_(j, k) * d_[size_t(k)];
      if (dj == 0.0) { info_ = NumericalIssue; return; }
      d_[size_t(j)] = dj;
      for (Index i = j + 1; i < n_; ++i) {
        double s = L_(i, j);
        for (Index k = 0; k < j; ++k) s -= L_(i, k) * L_(j, k) * d_[size_t(k)];
        L_(i, j) = s / dj;
      }
    }
  }
  ComputationInfo info() const { return info_; }
  VectorXd solve(const VectorXd& b) const {
    VectorXd y = b;
    for (Index i = 0; i < n_; ++i)
      for (Index k = 0; k < i; ++k) y[i] -= L_(i, k) * y[k];
    for (Index i = 0; i < n_; ++i) y[i] /= d_[size_t(i)];
    for (Index i = n_ - 1; i >= 0; --i)
      for (Index k = i + 1; k < n_; ++k) y[i] -= L_(k, i) * y[k];
    return y;
  }

 private:
  Index n_ = 0;
  MatrixXd L_;
  std::vector<double> d_;
  ComputationInfo info_ = NumericalIssue;
};

// ---------------------------------------------------------------------------------- sparse
template <class S>
struct Triplet {
  Index i, j;
  S v;
  Triplet(Index i_, Index j_, S v_) : i(i_), j(j_), v(v_) {}
  Index row() const { return i; }
  Index col() const { return j; }
  S value() const { return v; }
};

template <class S, int Opt = RowMajor>
class SparseMatrix;

template <class S, int Opt>
struct SparseTransposed {
  const SparseMatrix<S, Opt>* m;
};

template <class S, int Opt>
class SparseMatrix {  // compressed rows, ascending columns
 public:
  using Scalar = S;
  Index r = 0, c = 0;
  std::vector<Index> ptr{0};
  std::vector<Index> idx;
  std::vector<S> val;

  SparseMatrix() = default;
  SparseMatrix(Index rr, Index cc) { resize(rr, cc); }
  SparseMatrix(const SparseTransposed<S, Opt>& t) {  // explicit transpose
    const SparseMatrix& m = *t.m;
    resize(m.c, m.r);
    std::vector<Index> cnt(size_t(r) + 1, 0);
    for (Index k : m.idx) cnt[size_t(k) + 1]++;
    for (Index i = 0; i < r; ++i) cnt[size_t(i) + 1] += cnt[size_t(i)];
    ptr = cnt;
    idx.assign(m.idx.size(), 0);
    val.assign(m.val.size(), S(0));
    std::vector<Index> fill(ptr.begin(), ptr.end() - 1);
    for (Index i = 0; i < m.r; ++i)
      for (Index k = m.ptr[size_t(i)]; k < m.ptr[size_t(i) + 1]; ++k) {
        const Index p = fill[size_t(m.idx[size_t(k)])]++;
        idx[size_t(p)] = i;
        val[size_t(p)] = m.val[size_t(k)];
      }
  }
  void resize(Index rr, Index cc) {
    r = rr;
    c = cc;
    ptr.assign(size_t(rr) + 1, 0);
    idx.clear();
    val.clear();
  }
  Index rows() const { return r; }
  Index cols() const { return c; }
  Index nonZeros() const { return Index(val.size()); }
  void makeCompressed() {}
  void prune(S reference, S epsilon) {  // keep |v| > |reference| * epsilon (Eigen's isMuchSmallerThan)
    std::vector<Index> np{0};
    std::vector<Index> ni;
    std::vector<S> nv;
    for (Index i = 0; i < r; ++i) {
      for (Index k = ptr[size_t(i)]; k < ptr[size_t(i) + 1]; ++k)
        if (!(std::abs(val[size_t(k)]) <= std::abs(reference) * epsilon)) {
          ni.push_back(idx[size_t(k)]);
          nv.push_back(val[size_t(k)]);
        }
      np.push_back(Index(ni.size()));
    }
    ptr.swap(np);
    idx.swap(ni);
    val.swap(nv);
  }
  S coeff(Index i, Index j) const {
    auto b = idx.begin() + ptr[size_t(i)], e = idx.begin() + ptr[size_t(i) + 1];
    auto it = std::lower_bound(b, e, j);
    return (it != e && *it == j) ? val[size_t(it - idx.begin())] : S(0);
  }
  template <class It>
  void setFromTriplets(It begin, It end) {  // duplicates summed in insertion order
    std::vector<std::vector<std::pair<Index, S>>> rows(static_cast<size_t>(r));
    for (It t = begin; t != end; ++t) rows[size_t(t->row())].push_back({t->col(), t->value()});
    ptr.assign(size_t(r) + 1, 0);
    idx.clear();
    val.clear();
    for (Index i = 0; i < r; ++i) {
      auto& row = rows[size_t(i)];
      std::stable_sort(row.begin(), row.end(), [](auto& a, auto& b) { return a.first < b.first; });
      Index last = -1;
      for (auto& kv : row) {
        if (kv.first == last) {
          val.back() += kv.second;
        } else {
          idx.push_back(kv.first);
          val.push_back(kv.second);
          last = kv.first;
        }
      }
      ptr[size_t(i) + 1] = Index(idx.size());
    }
  }
  SparseTransposed<S, Opt> transpose() const { return SparseTransposed<S, Opt>{this}; }
  class InnerIterator {
   public:
    InnerIterator(const SparseMatrix& m, Index i) : m_(m), i_(i), k_(m.ptr[size_t(i)]), end_(m.ptr[size_t(i) + 1]) {}
    Index row() const { return i_; }
    explicit operator bool() const { return k_ < end_; }
    InnerIterator& operator++() { ++k_; return *this; }
    Index col() const { return m_.idx[size_t(k_)]; }
    Index index() const { return col(); }
    S value() const { return m_.val[size_t(k_)]; }

   private:
    const SparseMatrix& m_;
    Index i_, k_, end_;
  };
};

template <class S, int Opt>
SparseMatrix<S, Opt> operator*(const SparseMatrix<S, Opt>& a, const SparseMatrix<S, Opt>& b) {
  SparseMatrix<S, Opt> out(a.r, b.c);
  std::map<Index, S> acc;
  for (Index i = 0; i < a.r; ++i) {
    acc.clear();
    for (Index k = a.ptr[size_t(i)]; k < a.ptr[size_t(i) + 1]; ++k) {
      const Index kk = a.idx[size_t(k)];
      const S av = a.val[size_t(k)];
      for (Index l = b.ptr[size_t(kk)]; l < b.ptr[size_t(kk) + 1]; ++l) acc[b.idx[size_t(l)]] += av * b.val[size_t(l)];
    }
    for (auto& kv : acc) {
      out.idx.push_back(kv.first);
      out.val.push_back(kv.second);
    }
    out.ptr[size_t(i) + 1] = Index(out.idx.size());
  }
  return out;
}
template <class S, int Opt, int R, int C>
Matrix<S, Dynamic, 1> operator*(const SparseMatrix<S, Opt>& a, const Matrix<S, R, C>& x) {
  Matrix<S, Dynamic, 1> y(a.r);
  for (Index i = 0; i < a.r; ++i) {
    S s = S(0);
    for (Index k = a.ptr[size_t(i)]; k < a.ptr[size_t(i) + 1]; ++k) s += a.val[size_t(k)] * x[a.idx[size_t(k)]];
    y[i] = s;
  }
  return y;
}
template <class S, int Opt, int R, int C>
Matrix<S, Dynamic, 1> operator*(const SparseTransposed<S, Opt>& t, const Matrix<S, R, C>& x) {
  const SparseMatrix<S, Opt>& a = *t.m;
  Matrix<S, Dynamic, 1> y(a.c);
  for (Index i = 0; i < a.r; ++i)
    for (Index k = a.ptr[size_t(i)]; k < a.ptr[size_t(i) + 1]; ++k) y[a.idx[size_t(k)]] += a.val[size_t(k)] * x[i];
  return y;
}

// dense copy of a sparse matrix: MatrixXd(sparse)
template <class S, int R, int C>
template <int Opt>
Matrix<S, R, C>::Matrix(const SparseMatrix<S, Opt>& a) : r(a.r), c(a.c) {
  d.assign(size_t(r * c), S(0));
  for (Index i = 0; i < a.r; ++i)
    for (Index k = a.ptr[size_t(i)]; k < a.ptr[size_t(i) + 1]; ++k) (*this)(i, a.idx[size_t(k)]) = a.val[size_t(k)];
}

}  // namespace Eigen
