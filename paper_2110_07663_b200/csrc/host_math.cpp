#include "host_math.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>

#include "common.hpp"

namespace sb {

namespace {

// P_p and P_p' by the Bonnet recurrences (gll.cpp:12-25).
void legendre_pd(int p, double x, double& P, double& dP) {
  if (p == 0) { P = 1.0; dP = 0.0; return; }
  double a = 1.0, b = x, da = 0.0, db = 1.0;
  for (int k = 2; k <= p; ++k) {
    const double c = ((2.0 * k - 1.0) * x * b - (k - 1.0) * a) / k;
    const double dc = da + (2.0 * k - 1.0) * b;
    a = b; da = db; b = c; db = dc;
  }
  P = b; dP = db;
}

std::vector<double> bary(const std::vector<double>& x) {
  const size_t n = x.size();
  std::vector<double> w(n, 1.0);
  for (size_t j = 0; j < n; ++j)
    for (size_t k = 0; k < n; ++k)
      if (k != j) w[j] /= (x[j] - x[k]);
  return w;
}

Gll build(int p) {
  Gll g;
  g.order = p;
  g.nodes.assign(p + 1, 0.0);
  g.weights.assign(p + 1, 0.0);
  g.nodes[0] = -1.0;
  g.nodes[p] = 1.0;
  for (int j = 1; j < p; ++j) {  // Newton on P_p' (gll.cpp:47-58)
    double x = -std::cos(M_PI * j / p);
    for (int it = 0; it < 100; ++it) {
      double P, dP;
      legendre_pd(p, x, P, dP);
      const double d2 = (2.0 * x * dP - p * (p + 1.0) * P) / (1.0 - x * x);
      const double dx = dP / d2;
      x -= dx;
      if (std::abs(dx) < 4.0 * std::numeric_limits<double>::epsilon()) break;
    }
    g.nodes[j] = x;
  }
  for (int j = 1; j < p - j; ++j) {  // exact symmetry (gll.cpp:60-65)
    const double t = 0.5 * (g.nodes[p - j] - g.nodes[j]);
    g.nodes[j] = -t;
    g.nodes[p - j] = t;
  }
  if (p % 2 == 0) g.nodes[p / 2] = 0.0;
  for (int j = 0; j <= p; ++j) {
    double P, dP;
    legendre_pd(p, g.nodes[j], P, dP);
    g.weights[j] = 2.0 / (p * (p + 1.0) * P * P);
  }
  for (int j = 0; j < p + 1 - j; ++j) {
    const double t = 0.5 * (g.weights[j] + g.weights[p - j]);
    g.weights[j] = g.weights[p - j] = t;
  }
  // differentiation matrix (gll.cpp:120-134), column-major
  const int n = p + 1;
  const auto w = bary(g.nodes);
  g.diff.assign(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i) {
    double diag = 0.0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      const double v = (w[j] / w[i]) / (g.nodes[i] - g.nodes[j]);
      g.diff[i + size_t(n) * j] = v;
      diag -= v;
    }
    g.diff[i + size_t(n) * i] = diag;
  }
  return g;
}

}  // namespace

const Gll& gll(int order) {
  if (order < 1 || order > 16)
    invalid("gll: order must be in [1,16], got " + std::to_string(order));
  static std::vector<Gll> table;
  static std::once_flag once;
  std::call_once(once, [] {
    table.resize(17);
    for (int p = 1; p <= 16; ++p) table[p] = build(p);
  });
  return table[order];
}

std::vector<double> lagrange_interpolation_matrix(const std::vector<double>& from,
                                                  const std::vector<double>& to) {
  const size_t n = from.size(), m = to.size();
  const auto w = bary(from);
  std::vector<double> out(m * n, 0.0);
  for (size_t i = 0; i < m; ++i) {
    const double x = to[i];
    int hit = -1;
    for (size_t j = 0; j < n; ++j)
      if (x == from[j]) { hit = int(j); break; }
    if (hit >= 0) { out[i * n + hit] = 1.0; continue; }
    double den = 0.0;
    for (size_t j = 0; j < n; ++j) den += w[j] / (x - from[j]);
    for (size_t j = 0; j < n; ++j) out[i * n + j] = (w[j] / (x - from[j])) / den;
  }
  return out;
}

namespace {
double prof_r(double eps, double x) { return (x <= 0.5) ? (2.0 - eps) * x : 1.0 + eps * (x - 1.0); }
double prof_l(double eps, double x) { return 1.0 - prof_r(eps, 1.0 - x); }
double blend(double a, double b, double t) {
  if (t <= 0.0) return a;
  if (t >= 1.0) return b;
  return a + (b - a) * t * t * (3.0 - 2.0 * t);
}
double kprofile(double eps, double x, double s) {
  const int layer = std::min(static_cast<int>(x * 6.0), 5);
  const double lam = x * 6.0 - layer;
  const double l = prof_l(eps, s), r = prof_r(eps, s);
  switch (layer) {
    case 0: return l;
    case 1: return blend(l, r, lam);
    case 2: return blend(r, l, lam / 2.0);
    case 3: return blend(r, l, (1.0 + lam) / 2.0);
    case 4: return blend(l, r, lam);
    default: return r;
  }
}
}  // namespace

std::array<double, 3> kershaw_map(double eps, double x, double y, double z) {
  return {x - 0.5, kprofile(eps, x, y) - 0.5, kprofile(eps, x, z) - 0.5};
}

void uniform_pm1_range(uint64_t seed, int64_t offset, int64_t n, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (int64_t i = 0; i < offset; ++i) (void)dist(rng);
  for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}

void uniform_pm1(uint64_t seed, int64_t n, double* out) { uniform_pm1_range(seed, 0, n, out); }

bool gen_sym_eig(int n, const double* A, const double* B, double* lambda, double* S) {
  // B = L L^T
  std::vector<double> L(size_t(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = B[j + n * j];
    for (int k = 0; k < j; ++k) d -= L[j + n * k] * L[j + n * k];
    if (!(d > 0.0)) return false;
    L[j + n * j] = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double s = B[i + n * j];
      for (int k = 0; k < j; ++k) s -= L[i + n * k] * L[j + n * k];
      L[i + n * j] = s / L[j + n * j];
    }
  }
  // C = L^-1 A L^-T (solve column-wise)
  std::vector<double> T(size_t(n) * n), C(size_t(n) * n);
  for (int c = 0; c < n; ++c)  // T = L^-1 A
    for (int i = 0; i < n; ++i) {
      double s = A[i + n * c];
      for (int k = 0; k < i; ++k) s -= L[i + n * k] * T[k + n * c];
      T[i + n * c] = s / L[i + n * i];
    }
  for (int r = 0; r < n; ++r)  // C^T = L^-1 T^T
    for (int i = 0; i < n; ++i) {
      double s = T[r + n * i];
      for (int k = 0; k < i; ++k) s -= L[i + n * k] * C[r + n * k];
      C[r + n * i] = s / L[i + n * i];
    }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const double s = 0.5 * (C[i + n * j] + C[j + n * i]);
      C[i + n * j] = C[j + n * i] = s;
    }
  // cyclic Jacobi: C = Q diag Q^T
  std::vector<double> Q(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i) Q[i + n * i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += C[i + n * j] * C[i + n * j];
        if (i != j) off += C[i + n * j] * C[i + n * j];
      }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = C[p + n * q];
        if (apq == 0.0) continue;
        const double app = C[p + n * p], aqq = C[q + n * q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // columns p, q
          const double ckp = C[k + n * p], ckq = C[k + n * q];
          C[k + n * p] = c * ckp - s * ckq;
          C[k + n * q] = s * ckp + c * ckq;
        }
        for (int k = 0; k < n; ++k) {  // rows p, q
          const double cpk = C[p + n * k], cqk = C[q + n * k];
          C[p + n * k] = c * cpk - s * cqk;
          C[q + n * k] = s * cpk + c * cqk;
        }
        for (int k = 0; k < n; ++k) {
          const double qkp = Q[k + n * p], qkq = Q[k + n * q];
          Q[k + n * p] = c * qkp - s * qkq;
          Q[k + n * q] = s * qkp + c * qkq;
        }
      }
  }
  std::vector<int> ord(n);
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return C[a + n * a] < C[b + n * b]; });
  // S = L^-T Q (back substitution per column)
  for (int cc = 0; cc < n; ++cc) {
    const int c = ord[cc];
    lambda[cc] = C[c + n * c];
    for (int i = n - 1; i >= 0; --i) {
      double s = Q[i + n * c];
      for (int k = i + 1; k < n; ++k) s -= L[k + n * i] * S[k + n * cc];
      S[i + n * cc] = s / L[i + n * i];
    }
  }
  return true;
}

double max_abs_eig(int n, const double* Hc) {
  if (n <= 0) return 0.0;
  // row-major working copy a[i][j]
  std::vector<double> a(size_t(n) * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) a[size_t(i) * n + j] = Hc[i + size_t(n) * j];
  auto A = [&](int i, int j) -> double& { return a[size_t(i) * n + j]; };
  // reduce to Hessenberg (elimination with pivoting) in case H is general
  for (int m = 1; m < n - 1; ++m) {
    double x = 0.0;
    int i = m;
    for (int j = m; j < n; ++j)
      if (std::abs(A(j, m - 1)) > std::abs(x)) { x = A(j, m - 1); i = j; }
    if (i != m) {
      for (int j = m - 1; j < n; ++j) std::swap(A(i, j), A(m, j));
      for (int j = 0; j < n; ++j) std::swap(A(j, i), A(j, m));
    }
    if (x != 0.0)
      for (i = m + 1; i < n; ++i) {
        double y = A(i, m - 1);
        if (y != 0.0) {
          y /= x;
          A(i, m - 1) = y;
          for (int j = m; j < n; ++j) A(i, j) -= y * A(m, j);
          for (int j = 0; j < n; ++j) A(j, m) += y * A(j, i);
        }
      }
  }
  for (int i = 2; i < n; ++i)
    for (int j = 0; j < i - 1; ++j) A(i, j) = 0.0;
  std::vector<double> wr(n, 0.0), wi(n, 0.0);
  double anorm = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = std::max(i - 1, 0); j < n; ++j) anorm += std::abs(A(i, j));
  int nn = n - 1, l = 0;
  double t = 0.0, p = 0, q = 0, r = 0, s = 0, w = 0, x = 0, y = 0, z = 0;
  auto sign = [](double a_, double b_) { return b_ >= 0.0 ? std::abs(a_) : -std::abs(a_); };
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
        wr[nn] = x + t;
        wi[nn--] = 0.0;
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
            wr[nn - 1] = wr[nn] = x + z;
            if (z != 0.0) wr[nn] = x - w / z;
            wi[nn - 1] = wi[nn] = 0.0;
          } else {
            wr[nn - 1] = wr[nn] = x + p;
            wi[nn - 1] = -(wi[nn] = z);
          }
          nn -= 2;
        } else {
          if (its == 60) numeric("max_abs_eig: QR iteration did not converge");
          if (its == 10 || its == 20) {
            t += x;
            for (int i = 0; i <= nn; i++) A(i, i) -= x;
            s = std::abs(A(nn, nn - 1)) + std::abs(A(nn - 1, nn - 2));
            y = x = 0.75 * s;
            w = -0.4375 * s * s;
          }
          ++its;
          int m;
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
          for (int i = m + 2; i <= nn; i++) {
            A(i, i - 2) = 0.0;
            if (i != m + 2) A(i, i - 3) = 0.0;
          }
          for (int k = m; k <= nn - 1; k++) {
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
              for (int j = k; j <= nn; j++) {
                p = A(k, j) + q * A(k + 1, j);
                if (k != nn - 1) { p += r * A(k + 2, j); A(k + 2, j) -= p * z; }
                A(k + 1, j) -= p * y;
                A(k, j) -= p * x;
              }
              const int mmin = nn < k + 3 ? nn : k + 3;
              for (int i = l; i <= mmin; i++) {
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
  double best = 0.0;
  for (int i = 0; i < n; ++i) best = std::max(best, std::hypot(wr[i], wi[i]));
  return best;
}

}  // namespace sb
