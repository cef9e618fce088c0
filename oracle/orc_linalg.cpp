// ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp).
// Dense helpers and the square-root primitives of proj/src/linalg.cpp.
#include <cmath>
#include <limits>

#include "orc.hpp"

namespace orc {

Mat operator*(const Mat& a, const Mat& b) {
  if (a.c != b.r) throw DimensionError("oracle matmul: inner dimensions disagree");
  Mat out(a.r, b.c);
  for (int i = 0; i < a.r; ++i)
    for (int k = 0; k < a.c; ++k) {
      const double aik = a(i, k);
      if (aik == 0.0) continue;
      for (int j = 0; j < b.c; ++j) out(i, j) += aik * b(k, j);
    }
  return out;
}

Vec operator*(const Mat& a, const Vec& x) {
  if (a.c != static_cast<int>(x.size())) throw DimensionError("oracle matvec: size mismatch");
  Vec out(a.r, 0.0);
  for (int i = 0; i < a.r; ++i) {
    double acc = 0.0;
    for (int k = 0; k < a.c; ++k) acc += a(i, k) * x[k];
    out[i] = acc;
  }
  return out;
}

Mat operator+(const Mat& a, const Mat& b) {
  if (a.r != b.r || a.c != b.c) throw DimensionError("oracle add: shape mismatch");
  Mat out = a;
  for (std::size_t i = 0; i < out.v.size(); ++i) out.v[i] += b.v[i];
  return out;
}

Mat operator-(const Mat& a, const Mat& b) {
  if (a.r != b.r || a.c != b.c) throw DimensionError("oracle sub: shape mismatch");
  Mat out = a;
  for (std::size_t i = 0; i < out.v.size(); ++i) out.v[i] -= b.v[i];
  return out;
}

Mat operator*(double s, const Mat& a) {
  Mat out = a;
  for (double& x : out.v) x *= s;
  return out;
}

Vec operator+(const Vec& a, const Vec& b) {
  if (a.size() != b.size()) throw DimensionError("oracle vadd: size mismatch");
  Vec out = a;
  for (std::size_t i = 0; i < a.size(); ++i) out[i] += b[i];
  return out;
}

Vec operator-(const Vec& a, const Vec& b) {
  if (a.size() != b.size()) throw DimensionError("oracle vsub: size mismatch");
  Vec out = a;
  for (std::size_t i = 0; i < a.size(); ++i) out[i] -= b[i];
  return out;
}

Vec operator*(double s, const Vec& a) {
  Vec out = a;
  for (double& x : out) x *= s;
  return out;
}

Mat transpose(const Mat& a) {
  Mat out(a.c, a.r);
  for (int i = 0; i < a.r; ++i)
    for (int j = 0; j < a.c; ++j) out(j, i) = a(i, j);
  return out;
}

Mat block(const Mat& a, int r0, int c0, int rows, int cols) {
  Mat out(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) out(i, j) = a(r0 + i, c0 + j);
  return out;
}

void set_block(Mat& a, int r0, int c0, const Mat& b) {
  for (int i = 0; i < b.r; ++i)
    for (int j = 0; j < b.c; ++j) a(r0 + i, c0 + j) = b(i, j);
}

Mat diag_mul_left(const Vec& d, const Mat& a) {
  Mat out = a;
  for (int i = 0; i < a.r; ++i)
    for (int j = 0; j < a.c; ++j) out(i, j) *= d[i];
  return out;
}

Mat diag_mul_right(const Mat& a, const Vec& d) {
  Mat out = a;
  for (int i = 0; i < a.r; ++i)
    for (int j = 0; j < a.c; ++j) out(i, j) *= d[j];
  return out;
}

Vec cwise(const Vec& a, const Vec& b) {
  Vec out(a.size());
  for (std::size_t i = 0; i < a.size(); ++i) out[i] = a[i] * b[i];
  return out;
}

bool all_finite(const Mat& a) {
  for (double x : a.v)
    if (!std::isfinite(x)) return false;
  return true;
}

bool all_finite(const Vec& a) {
  for (double x : a)
    if (!std::isfinite(x)) return false;
  return true;
}

Mat dense_cov(const Mat& s) { return s * transpose(s); }

// Householder QR of a (rows >= cols) matrix in place, Eigen's unblocked
// convention (HouseholderQR -> householder_qr_inplace_unblocked; blocks of
// 48 columns are never reached at the sizes of this path):
//   makeHouseholder: beta = -sign(c0) * ||x||, essential = tail / (c0 - beta),
//   tau = (beta - c0) / beta; tau = 0, beta = c0 when ||tail||^2 <= DBL_MIN.
static void householder_qr_inplace(Mat& a) {
  const int rows = a.r, cols = a.c;
  const int size = std::min(rows, cols);
  const double tol = std::numeric_limits<double>::min();
  for (int k = 0; k < size; ++k) {
    const int remaining_rows = rows - k;
    double tail_sq = 0.0;
    for (int i = k + 1; i < rows; ++i) tail_sq += a(i, k) * a(i, k);
    const double c0 = a(k, k);
    double tau, beta;
    if (tail_sq <= tol) {
      tau = 0.0;
      beta = c0;
      for (int i = k + 1; i < rows; ++i) a(i, k) = 0.0;
    } else {
      beta = std::sqrt(c0 * c0 + tail_sq);
      if (c0 >= 0.0) beta = -beta;
      const double denom = c0 - beta;
      for (int i = k + 1; i < rows; ++i) a(i, k) /= denom;
      tau = (beta - c0) / beta;
    }
    a(k, k) = beta;
    if (remaining_rows == 1 || tau == 0.0) continue;
    // applyHouseholderOnTheLeft(essential = a[k+1:, k], tau) on a[k:, k+1:].
    for (int j = k + 1; j < cols; ++j) {
      double tmp = a(k, j);
      for (int i = k + 1; i < rows; ++i) tmp += a(i, k) * a(i, j);
      a(k, j) -= tau * tmp;
      for (int i = k + 1; i < rows; ++i) a(i, j) -= tau * a(i, k) * tmp;
    }
  }
}

// proj/src/linalg.cpp:9-27 — tria(M) = R^T with R from QR(M^T); zero-pad
// when M has fewer columns than rows; non-finite input is rejected.
Mat tria(const Mat& m) {
  if (!all_finite(m)) throw InvalidInputError("tria: input contains non-finite entries");
  const int n = m.r;
  Mat src = m;
  if (m.c < n) {
    src = Mat(n, n);
    set_block(src, 0, 0, m);
  }
  Mat qr = transpose(src);  // (k x n), k >= n
  householder_qr_inplace(qr);
  Mat out(n, n);  // R^T: out(i, j) = R(j, i) for j <= i
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) out(i, j) = qr(j, i);
  return out;
}

// proj/src/linalg.cpp:29-36
Mat sqrt_sum(const Mat& a, const Mat& b) {
  if (a.r != b.r) throw DimensionError("sqrt_sum: factors must have the same number of rows");
  Mat stacked(a.r, a.c + b.c);
  set_block(stacked, 0, 0, a);
  set_block(stacked, 0, a.c, b);
  return tria(stacked);
}

Vec solve_lower(const Mat& l, const Vec& b) {
  const int n = l.r;
  Vec x = b;
  for (int i = 0; i < n; ++i) {
    double acc = x[i];
    for (int k = 0; k < i; ++k) acc -= l(i, k) * x[k];
    x[i] = acc / l(i, i);
  }
  return x;
}

Mat solve_lower(const Mat& l, const Mat& b) {
  const int n = l.r;
  Mat x = b;
  for (int j = 0; j < b.c; ++j)
    for (int i = 0; i < n; ++i) {
      double acc = x(i, j);
      for (int k = 0; k < i; ++k) acc -= l(i, k) * x(k, j);
      x(i, j) = acc / l(i, i);
    }
  return x;
}

Mat solve_upper(const Mat& u, const Mat& b) {
  const int n = u.r;
  Mat x = b;
  for (int j = 0; j < b.c; ++j)
    for (int i = n - 1; i >= 0; --i) {
      double acc = x(i, j);
      for (int k = i + 1; k < n; ++k) acc -= u(i, k) * x(k, j);
      x(i, j) = acc / u(i, i);
    }
  return x;
}

// proj/src/linalg.cpp:38-52
double whitened_sq_norm(const Vec& v, const Mat& q_sqrt) {
  if (q_sqrt.r != q_sqrt.c || q_sqrt.r != static_cast<int>(v.size()))
    throw DimensionError(
        "whitened_sq_norm: factor must be square and match the vector length");
  if (!all_finite(v) || !all_finite(q_sqrt))
    throw InvalidInputError("whitened_sq_norm: non-finite input");
  for (int i = 0; i < q_sqrt.r; ++i)
    if (q_sqrt(i, i) == 0.0)
      throw SingularFactorError("whitened_sq_norm: factor has a zero diagonal entry");
  const Vec w = solve_lower(q_sqrt, v);
  double acc = 0.0;
  for (double x : w) acc += x * x;
  return acc;
}

// proj/src/linalg.cpp:54-62
void require_nonsingular_triangular(const Mat& t, const char* context) {
  if (t.r == 0) return;
  double largest = 0.0;
  for (int i = 0; i < t.r; ++i) largest = std::max(largest, std::abs(t(i, i)));
  for (int i = 0; i < t.r; ++i)
    if (std::abs(t(i, i)) <= 1e-13 * largest)
      throw SingularFactorError(std::string(context) + ": triangular factor is singular");
}

// proj/src/linalg.cpp:64-71
bool is_lower_triangular(const Mat& m) {
  for (int j = 1; j < m.c; ++j)
    for (int i = 0; i < j && i < m.r; ++i)
      if (m(i, j) != 0.0) return false;
  return true;
}

}  // namespace orc
