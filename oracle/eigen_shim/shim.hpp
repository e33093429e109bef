// ORACLE TEST INFRASTRUCTURE — a minimal, eager Eigen-API subset that lets the reference's own
// translation units (/root/reference/proj/core/src/{gll,mesh,sem_space,schwarz,chebyshev,krylov,
// amg}.cpp) compile UNMODIFIED in this image, which ships no Eigen.
// Every operation is evaluated eagerly into a column-major dense matrix; no expression
// templates. Results match real Eigen up to summation-order rounding (~1e-16 relative); the
// decompositions (generalised symmetric eigen, Hessenberg QR eigenvalues, 3x3 SVD, LDLT) return
// the same mathematical objects. Never linked into the product library.
#pragma once

#include <algorithm>
#include <cassert>
#include <cmath>
#include <complex>
#include <cstddef>
#include <initializer_list>
#include <stdexcept>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
enum { Upper = 1, Lower = 2, RowMajor = 1, ColMajor = 0 };

template <class S, int R = Dynamic, int C = Dynamic>
class Matrix;
template <class S, int Opt>
class SparseMatrix;

// ---------------------------------------------------------------------------------- views
// A strided (column-major) window onto a matrix's storage.
template <class S>
struct View {
  S* p = nullptr;
  Index r = 0, c = 0, ld = 0;
  View() = default;
  View(S* p_, Index r_, Index c_, Index ld_) : p(p_), r(r_), c(c_), ld(ld_) {}
  Index rows() const { return r; }
  Index cols() const { return c; }
  Index size() const { return r * c; }
  S& operator()(Index i, Index j) const { return p[i + ld * j]; }
  S& operator[](Index i) const { return r == 1 ? p[ld * i] : p[i]; }
  S& operator()(Index i) const { return (*this)[i]; }
};

template <class S>
class Block;
template <class S>
struct BlockTri;
template <class S>
struct Transposed;
template <class S>
struct ArrayRef;

template <class S>
Matrix<S> to_matrix(const View<S>& v) {
  Matrix<S> m(v.r, v.c);
  for (Index j = 0; j < v.c; ++j)
    for (Index i = 0; i < v.r; ++i) m(i, j) = v(i, j);
  return m;
}

// ---------------------------------------------------------------------------------- Matrix
template <class S, int R, int C>
class Matrix {
 public:
  using Scalar = S;
  std::vector<S> d;
  Index r = 0, c = 0;

  Matrix() {
    if (R > 0 && C > 0) {
      r = R;
      c = C;
      d.assign(size_t(R * C), S(0));
    } else if (R > 0 && C == Dynamic) {
      r = R;
    } else if (C > 0 && R == Dynamic) {
      c = C;
    }
  }
  explicit Matrix(Index n) {  // vectors
    if (C == 1) { r = n; c = 1; } else if (R == 1) { r = 1; c = n; } else { r = n; c = n; }
    d.assign(size_t(r * c), S(0));
  }
  Matrix(Index rr, Index cc) : r(rr), c(cc) { d.assign(size_t(rr * cc), S(0)); }
  Matrix(S x, S y, S z) : r(3), c(1) { d = {x, y, z}; }  // Vector3d(x,y,z)
  template <int R2, int C2>
  Matrix(const Matrix<S, R2, C2>& o) : d(o.d), r(o.r), c(o.c) {}
  Matrix(const View<S>& v) { *this = to_matrix(v); }
  template <int Opt>
  explicit Matrix(const SparseMatrix<S, Opt>& sp);  // MatrixXd(sparse), amg.cpp:124
  Matrix(const Block<S>& b);
  Matrix(const Matrix&) = default;
  Matrix(Matrix&&) = default;
  Matrix& operator=(const Matrix&) = default;
  Matrix& operator=(Matrix&&) = default;
  template <int R2, int C2>
  Matrix& operator=(const Matrix<S, R2, C2>& o) {
    d = o.d;
    r = o.r;
    c = o.c;
    return *this;
  }
  Matrix& operator=(const Block<S>& b);

  static Matrix Zero(Index n) { Matrix m(n); return m; }
  static Matrix Zero(Index rr, Index cc) { return Matrix(rr, cc); }
  static Matrix Zero() { return Matrix(); }
  static Matrix Ones(Index n) { Matrix m(n); std::fill(m.d.begin(), m.d.end(), S(1)); return m; }
  static Matrix Constant(Index n, S v) { Matrix m(n); std::fill(m.d.begin(), m.d.end(), v); return m; }
  static Matrix Constant(Index rr, Index cc, S v) { Matrix m(rr, cc); std::fill(m.d.begin(), m.d.end(), v); return m; }
  static Matrix Identity(Index n) { Matrix m(n, n); for (Index i = 0; i < n; ++i) m(i, i) = S(1); return m; }

  Index rows() const { return r; }
  Index cols() const { return c; }
  Index size() const { return r * c; }
  S* data() { return d.data(); }
  const S* data() const { return d.data(); }
  void resize(Index n) {
    if (C == 1 || c == 1 || (R == Dynamic && C == Dynamic && c <= 1)) { r = n; c = 1; } else { r = 1; c = n; }
    d.assign(size_t(r * c), S(0));
  }
  void resize(Index rr, Index cc) { r = rr; c = cc; d.assign(size_t(rr * cc), S(0)); }
  void setZero() { std::fill(d.begin(), d.end(), S(0)); }
  Matrix& setZero(Index n) { resize(n); return *this; }

  S& operator()(Index i, Index j) { return d[size_t(i + r * j)]; }
  const S& operator()(Index i, Index j) const { return d[size_t(i + r * j)]; }
  S& operator[](Index i) { return d[size_t(i)]; }
  const S& operator[](Index i) const { return d[size_t(i)]; }
  S& operator()(Index i) { return d[size_t(i)]; }
  const S& operator()(Index i) const { return d[size_t(i)]; }

  View<S> view() const { return View<S>(const_cast<S*>(d.data()), r, c, r); }
  Block<S> col(Index j) const;
  Block<S> row(Index i) const;
  Block<S> head(Index k) const;
  Block<S> leftCols(Index k) const;
  Block<S> topLeftCorner(Index rr, Index cc) const;
  Block<S> block(Index i, Index j, Index rr, Index cc) const;
  Transposed<S> transpose() const;
  ArrayRef<S> array() const;
  Matrix& noalias() { return *this; }

  // arithmetic (eager)
  Matrix& operator+=(const Matrix& o) { for (size_t t = 0; t < d.size(); ++t) d[t] += o.d[t]; return *this; }
  Matrix& operator-=(const Matrix& o) { for (size_t t = 0; t < d.size(); ++t) d[t] -= o.d[t]; return *this; }
  Matrix& operator*=(S s) { for (auto& v : d) v *= s; return *this; }
  Matrix& operator/=(S s) { for (auto& v : d) v /= s; return *this; }
  Matrix operator-() const { Matrix m(*this); for (auto& v : m.d) v = -v; return m; }

  S dot(const Matrix& o) const { S s = S(0); for (size_t t = 0; t < d.size(); ++t) s += d[t] * o.d[t]; return s; }
  S squaredNorm() const { S s = S(0); for (auto v : d) s += v * v; return s; }
  S norm() const { return std::sqrt(squaredNorm()); }
  S sum() const { S s = S(0); for (auto v : d) s += v; return s; }
  S mean() const { return sum() / S(d.size()); }
  S maxCoeff() const { return *std::max_element(d.begin(), d.end()); }
  S minCoeff() const { return *std::min_element(d.begin(), d.end()); }
  Matrix cwiseAbs() const { Matrix m(*this); for (auto& v : m.d) v = std::abs(v); return m; }
  Matrix cwiseProduct(const Matrix& o) const { Matrix m(*this); for (size_t t = 0; t < d.size(); ++t) m.d[t] *= o.d[t]; return m; }
  S determinant() const;
  Matrix inverse() const;
  template <int Mode>
  struct TriView {
    const Matrix* m;
    template <class V>
    Matrix<S, Dynamic, 1> solve(const V& bb) const;
  };
  template <int Mode>
  TriView<Mode> triangularView() const { return TriView<Mode>{this}; }
};

using MatrixXd = Matrix<double>;
using VectorXd = Matrix<double, Dynamic, 1>;
using VectorXi = Matrix<int, Dynamic, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Matrix3d = Matrix<double, 3, 3>;
using VectorXcd = Matrix<std::complex<double>, Dynamic, 1>;

// ---------------------------------------------------------------------------------- Block
template <class S>
class Block : public View<S> {
 public:
  using View<S>::View;
  Block(const View<S>& v) : View<S>(v) {}
  using View<S>::p;
  using View<S>::r;
  using View<S>::c;
  using View<S>::ld;
  template <class Src>
  Block& assign(const Src& m) {
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) (*this)(i, j) = m(i, j);
    return *this;
  }
  template <int R, int C>
  Block& operator=(const Matrix<S, R, C>& m) { return assign(m); }
  Block& operator=(const Block& b) { Matrix<S> tmp(b); return assign(tmp); }
  template <int R, int C>
  Block& operator+=(const Matrix<S, R, C>& m) {
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) (*this)(i, j) += m(i, j);
    return *this;
  }
  template <int R, int C>
  Block& operator-=(const Matrix<S, R, C>& m) {
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) (*this)(i, j) -= m(i, j);
    return *this;
  }
  Block head(Index k) const { return Block(p, r == 1 ? 1 : k, r == 1 ? k : 1, ld); }
  Block col(Index j) const { return Block(p + ld * j, r, 1, ld); }
  Block leftCols(Index k) const { return Block(p, r, k, ld); }
  Block topLeftCorner(Index rr, Index cc) const { return Block(p, rr, cc, ld); }
  Transposed<S> transpose() const;
  Block& noalias() { return *this; }
  S norm() const { Matrix<S> m(*this); return m.norm(); }
  S dot(const Matrix<S, Dynamic, 1>& o) const { Matrix<S> m(*this); return m.dot(o); }
  Matrix<S> cwiseAbs() const { return Matrix<S>(*this).cwiseAbs(); }
  S maxCoeff() const { return Matrix<S>(*this).maxCoeff(); }
  template <int Mode>
  BlockTri<S> triangularView() const;
};

template <class S, int R, int C>
Matrix<S, R, C>::Matrix(const Block<S>& b) {
  r = b.r;
  c = b.c;
  d.resize(size_t(r * c));
  for (Index j = 0; j < c; ++j)
    for (Index i = 0; i < r; ++i) d[size_t(i + r * j)] = b(i, j);
}
template <class S, int R, int C>
Matrix<S, R, C>& Matrix<S, R, C>::operator=(const Block<S>& b) {
  Matrix tmp(b);
  *this = std::move(tmp);
  return *this;
}
template <class S, int R, int C>
Block<S> Matrix<S, R, C>::col(Index j) const { return Block<S>(const_cast<S*>(d.data()) + r * j, r, 1, r); }
template <class S, int R, int C>
Block<S> Matrix<S, R, C>::row(Index i) const { return Block<S>(const_cast<S*>(d.data()) + i, 1, c, r); }
template <class S, int R, int C>
Block<S> Matrix<S, R, C>::head(Index k) const { return Block<S>(const_cast<S*>(d.data()), k, 1, r); }
template <class S, int R, int C>
Block<S> Matrix<S, R, C>::leftCols(Index k) const { return Block<S>(const_cast<S*>(d.data()), r, k, r); }
template <class S, int R, int C>
Block<S> Matrix<S, R, C>::topLeftCorner(Index rr, Index cc) const { return Block<S>(const_cast<S*>(d.data()), rr, cc, r); }
template <class S, int R, int C>
Block<S> Matrix<S, R, C>::block(Index i, Index j, Index rr, Index cc) const {
  return Block<S>(const_cast<S*>(d.data()) + i + r * j, rr, cc, r);
}

// ---------------------------------------------------------------------------------- Map
template <class M>
class Map : public Block<typename std::remove_const<M>::type::Scalar> {
  using S = typename std::remove_const<M>::type::Scalar;

 public:
  Map(const S* p, Index rr, Index cc) : Block<S>(const_cast<S*>(p), rr, cc, rr) {}
  Map(const S* p, Index n) : Block<S>(const_cast<S*>(p), n, 1, n) {}
  using Block<S>::operator=;
  Map& noalias() { return *this; }
};

// ---------------------------------------------------------------------------------- transpose
template <class S>
struct Transposed {  // lazy transpose of a view, consumed by operator*
  using Scalar = S;
  View<S> v;
  Index rows() const { return v.c; }
  Index cols() const { return v.r; }
  S operator()(Index i, Index j) const { return v(j, i); }
};
template <class S, int R, int C>
Transposed<S> Matrix<S, R, C>::transpose() const { return Transposed<S>{view()}; }
template <class S>
Transposed<S> Block<S>::transpose() const { return Transposed<S>{*this}; }

// ---------------------------------------------------------------------------------- products
template <class A, class B>
Matrix<typename B::Scalar> gemm(const A& a, const B& b, Index m, Index k, Index n) {
  using S = typename B::Scalar;
  Matrix<S> out(m, n);
  for (Index j = 0; j < n; ++j)
    for (Index l = 0; l < k; ++l) {
      const S blj = b(l, j);
      if (blj == S(0)) continue;
      for (Index i = 0; i < m; ++i) out(i, j) += a(i, l) * blj;
    }
  return out;
}
template <class S>
struct ViewAdapter {  // uniform (i,j) access + Scalar
  using Scalar = S;
  View<S> v;
  S operator()(Index i, Index j) const { return v(i, j); }
};
template <class S, int R1, int C1, int R2, int C2>
Matrix<S, (R1 > 0 && C2 > 0) ? R1 : Dynamic, (R1 > 0 && C2 > 0) ? C2 : ((C2 == 1) ? 1 : Dynamic)> operator*(
    const Matrix<S, R1, C1>& a, const Matrix<S, R2, C2>& b) {
  auto m = gemm(a, b, a.r, a.c, b.c);
  Matrix<S, (R1 > 0 && C2 > 0) ? R1 : Dynamic, (R1 > 0 && C2 > 0) ? C2 : ((C2 == 1) ? 1 : Dynamic)> out;
  out.d = std::move(m.d);
  out.r = a.r;
  out.c = b.c;
  return out;
}
template <class S, int R2, int C2>
Matrix<S, Dynamic, (C2 == 1) ? 1 : Dynamic> operator*(const Block<S>& a, const Matrix<S, R2, C2>& b) {
  auto m = gemm(ViewAdapter<S>{a}, b, a.r, a.c, b.c);
  Matrix<S, Dynamic, (C2 == 1) ? 1 : Dynamic> out;
  out.d = std::move(m.d);
  out.r = a.r;
  out.c = b.c;
  return out;
}
template <class S, int R1, int C1>
Matrix<S> operator*(const Matrix<S, R1, C1>& a, const Block<S>& b) {
  return gemm(a, ViewAdapter<S>{b}, a.r, a.c, b.c);
}
template <class S, int R2, int C2>
Matrix<S, Dynamic, (C2 == 1) ? 1 : Dynamic> operator*(const Transposed<S>& a, const Matrix<S, R2, C2>& b) {
  // (V^T w): dot products of the columns of V with b
  Matrix<S, Dynamic, (C2 == 1) ? 1 : Dynamic> out;
  out.r = a.rows();
  out.c = b.c;
  out.d.assign(size_t(out.r * out.c), S(0));
  for (Index j = 0; j < b.c; ++j)
    for (Index i = 0; i < a.rows(); ++i) {
      S s = S(0);
      for (Index l = 0; l < a.cols(); ++l) s += a.v(l, i) * b(l, j);
      out(i, j) = s;
    }
  return out;
}
template <class S>
Matrix<S> operator*(const Transposed<S>& a, const Block<S>& b) {
  Matrix<S> out(a.rows(), b.c);
  for (Index j = 0; j < b.c; ++j)
    for (Index i = 0; i < a.rows(); ++i) {
      S s = S(0);
      for (Index l = 0; l < a.cols(); ++l) s += a.v(l, i) * b(l, j);
      out(i, j) = s;
    }
  return out;
}
template <class S, int R1, int C1>
Matrix<S, R1, R1> operator*(const Matrix<S, R1, C1>& a, const Transposed<S>& b) {
  auto m = gemm(a, b, a.r, a.c, b.cols());
  Matrix<S, R1, R1> out;
  out.d = std::move(m.d);
  out.r = a.r;
  out.c = b.cols();
  return out;
}
template <class S>
Matrix<S> operator*(const Block<S>& a, const Transposed<S>& b) {
  return gemm(ViewAdapter<S>{a}, b, a.r, a.c, b.cols());
}
template <class S>
Matrix<S> operator*(const Block<S>& a, const Block<S>& b) {
  return gemm(ViewAdapter<S>{a}, ViewAdapter<S>{b}, a.r, a.c, b.c);
}

// ---------------------------------------------------------------------------------- elementwise
template <class S, int R, int C>
Matrix<S, R, C> operator+(Matrix<S, R, C> a, const Matrix<S, R, C>& b) { a += b; return a; }
template <class S, int R, int C>
Matrix<S, R, C> operator-(Matrix<S, R, C> a, const Matrix<S, R, C>& b) { a -= b; return a; }
template <class S, int R, int C>
Matrix<S, R, C> operator*(Matrix<S, R, C> a, S s) { a *= s; return a; }
template <class S, int R, int C>
Matrix<S, R, C> operator*(S s, Matrix<S, R, C> a) { for (auto& v : a.d) v = s * v; return a; }
template <class S, int R, int C>
Matrix<S, R, C> operator/(Matrix<S, R, C> a, S s) { a /= s; return a; }
template <class S>
Matrix<S, Dynamic, 1> operator/(const Block<S>& b, S s) { Matrix<S, Dynamic, 1> v = b; v /= s; return v; }
template <class S>
Matrix<S, Dynamic, 1> operator*(S s, const Block<S>& b) { Matrix<S, Dynamic, 1> v = b; for (auto& x : v.d) x = s * x; return v; }
template <class S, int R, int C>
Matrix<S, R, C> operator-(const Matrix<S, R, C>& a, const Block<S>& b) {
  Matrix<S, R, C> m(a);
  for (Index i = 0; i < m.size(); ++i) m.d[size_t(i)] -= b[i];
  return m;
}
template <class S, int R, int C>
Matrix<S, R, C> operator-(const Block<S>& a, const Matrix<S, R, C>& b) {
  Matrix<S, R, C> m(b);
  for (Index i = 0; i < m.size(); ++i) m.d[size_t(i)] = a[i] - m.d[size_t(i)];
  return m;
}

// ---------------------------------------------------------------------------------- arrays
template <class S>
struct ArrayRef {
  S* p;
  Index n;
  ArrayRef& operator*=(const ArrayRef& o) { for (Index i = 0; i < n; ++i) p[i] *= o.p[i]; return *this; }
  ArrayRef& operator-=(S s) { for (Index i = 0; i < n; ++i) p[i] -= s; return *this; }
  ArrayRef& operator+=(S s) { for (Index i = 0; i < n; ++i) p[i] += s; return *this; }
  ArrayRef& operator*=(S s) { for (Index i = 0; i < n; ++i) p[i] *= s; return *this; }
};
template <class S, int R, int C>
ArrayRef<S> Matrix<S, R, C>::array() const { return ArrayRef<S>{const_cast<S*>(d.data()), size()}; }

// ---------------------------------------------------------------------------------- 3x3
template <class S, int R, int C>
S Matrix<S, R, C>::determinant() const {
  const Matrix& m = *this;
  return m(0, 0) * (m(1, 1) * m(2, 2) - m(2, 1) * m(1, 2)) - m(1, 0) * (m(0, 1) * m(2, 2) - m(2, 1) * m(0, 2)) +
         m(2, 0) * (m(0, 1) * m(1, 2) - m(1, 1) * m(0, 2));
}
template <class S, int R, int C>
Matrix<S, R, C> Matrix<S, R, C>::inverse() const {
  const Matrix& m = *this;
  Matrix out(3, 3);
  const S c00 = m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1), c10 = m(1, 2) * m(2, 0) - m(1, 0) * m(2, 2),
          c20 = m(1, 0) * m(2, 1) - m(1, 1) * m(2, 0);
  const S det = m(0, 0) * c00 + m(0, 1) * c10 + m(0, 2) * c20;
  const S id = S(1) / det;
  out(0, 0) = c00 * id;
  out(1, 0) = c10 * id;
  out(2, 0) = c20 * id;
  out(0, 1) = (m(0, 2) * m(2, 1) - m(0, 1) * m(2, 2)) * id;
  out(1, 1) = (m(0, 0) * m(2, 2) - m(0, 2) * m(2, 0)) * id;
  out(2, 1) = (m(0, 1) * m(2, 0) - m(0, 0) * m(2, 1)) * id;
  out(0, 2) = (m(0, 1) * m(1, 2) - m(0, 2) * m(1, 1)) * id;
  out(1, 2) = (m(0, 2) * m(1, 0) - m(0, 0) * m(1, 2)) * id;
  out(2, 2) = (m(0, 0) * m(1, 1) - m(0, 1) * m(1, 0)) * id;
  return out;
}

// upper-triangular back substitution (triangularView<Upper>().solve)
template <class S, int R, int C>
template <int Mode>
template <class V>
Matrix<S, Dynamic, 1> Matrix<S, R, C>::TriView<Mode>::solve(const V& bb) const {
  Matrix<S, Dynamic, 1> b = bb;
  const Index n = m->rows();
  Matrix<S, Dynamic, 1> y(n);
  for (Index i = n - 1; i >= 0; --i) {
    S acc = b[i];
    for (Index k = i + 1; k < n; ++k) acc -= (*m)(i, k) * y[k];
    y[i] = acc / (*m)(i, i);
  }
  return y;
}
// Block::triangularView (topLeftCorner(j,j).triangularView<Upper>())
template <class S>
struct BlockTri {
  Matrix<S> m;
  template <class V>
  Matrix<S, Dynamic, 1> solve(const V& b) const { return m.template triangularView<Upper>().solve(b); }
};
template <class S>
template <int Mode>
BlockTri<S> Block<S>::triangularView() const {
  static_assert(Mode == Upper, "shim: only upper-triangular solves are used by the reference");
  return BlockTri<S>{Matrix<S>(*this)};
}

}  // namespace Eigen

#include "shim_decomp.hpp"
