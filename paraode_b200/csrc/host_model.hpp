// Host-side, one-time model setup for the device solver: IWP prior blocks
// (proj/src/prior.cpp:79-117), exact Taylor initialisation
// (proj/src/prior.cpp:119-168, Taylor-mode arithmetic of
// proj/include/paraode/jet.hpp extended with division and square root for
// the Pleiades field) and the shipped problem defaults.  Everything per time
// step runs on the GPU; this file only produces O(D^2) constants.
#pragma once

#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/paraode_b200.h"
#include "context.hpp"

namespace pode {
namespace host {

inline double factorial(int n) {
  double f = 1.0;
  for (int k = 2; k <= n; ++k) f *= k;
  return f;
}

inline double binomial(int n, int k) {
  if (k < 0 || k > n) return 0.0;
  return factorial(n) / (factorial(k) * factorial(n - k));
}

// Binomial (Pascal) block replicated over dim (prior.cpp:99-107), row-major D x D.
inline std::vector<double> preconditioned_phi(int nu, int dim) {
  const int b = nu + 1, D = b * dim;
  std::vector<double> out(size_t(D) * D, 0.0);
  for (int r = 0; r < dim; ++r)
    for (int i = 0; i <= nu; ++i)
      for (int j = i; j <= nu; ++j) out[size_t(r * b + i) * D + r * b + j] = binomial(nu - i, j - i);
  return out;
}

// Cholesky factor of the Hilbert-like block 1/(2nu+1-i-j), replicated
// (prior.cpp:109-117; the block is positive definite for every nu >= 1, so
// the LLT branch of psd_sqrt is the one taken).
inline std::vector<double> preconditioned_q_sqrt(int nu, int dim) {
  const int b = nu + 1, D = b * dim;
  std::vector<double> blk(size_t(b) * b), l(size_t(b) * b, 0.0);
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < b; ++j) blk[i * b + j] = 1.0 / (2 * nu + 1 - i - j);
  for (int k = 0; k < b; ++k) {
    double x = blk[k * b + k];
    for (int j = 0; j < k; ++j) x -= l[k * b + j] * l[k * b + j];
    if (!(x > 0.0)) throw ApiError(PODE_ERR_SINGULAR_FACTOR, "preconditioned_q_sqrt: block not positive definite");
    const double piv = std::sqrt(x);
    l[k * b + k] = piv;
    for (int i = k + 1; i < b; ++i) {
      double s = blk[i * b + k];
      for (int j = 0; j < k; ++j) s -= l[i * b + j] * l[k * b + j];
      l[i * b + k] = s / piv;
    }
  }
  std::vector<double> out(size_t(D) * D, 0.0);
  for (int r = 0; r < dim; ++r)
    for (int i = 0; i < b; ++i)
      for (int j = 0; j < b; ++j) out[size_t(r * b + i) * D + r * b + j] = l[i * b + j];
  return out;
}

// ------------------------------------------------------- Taylor series ---
struct Jet {
  std::vector<double> c;
  explicit Jet(int order = 0, double v = 0.0) : c(size_t(order) + 1, 0.0) { c[0] = v; }
  int order() const { return int(c.size()) - 1; }
};
inline Jet operator+(Jet a, const Jet& b) {
  for (size_t k = 0; k < a.c.size(); ++k) a.c[k] += b.c[k];
  return a;
}
inline Jet operator-(Jet a, const Jet& b) {
  for (size_t k = 0; k < a.c.size(); ++k) a.c[k] -= b.c[k];
  return a;
}
inline Jet operator*(const Jet& a, const Jet& b) {  // truncated Cauchy product
  Jet o(a.order());
  for (size_t k = 0; k < a.c.size(); ++k) {
    double acc = 0.0;
    for (size_t i = 0; i <= k; ++i) acc += a.c[i] * b.c[k - i];
    o.c[k] = acc;
  }
  return o;
}
inline Jet operator/(const Jet& a, const Jet& b) {
  Jet q(a.order());
  for (size_t k = 0; k < a.c.size(); ++k) {
    double acc = a.c[k];
    for (size_t i = 1; i <= k; ++i) acc -= b.c[i] * q.c[k - i];
    q.c[k] = acc / b.c[0];
  }
  return q;
}
inline Jet jsqrt(const Jet& a) {
  Jet s(a.order());
  s.c[0] = std::sqrt(a.c[0]);
  for (size_t k = 1; k < a.c.size(); ++k) {
    double acc = a.c[k];
    for (size_t i = 1; i < k; ++i) acc -= s.c[i] * s.c[k - i];
    s.c[k] = acc / (2.0 * s.c[0]);
  }
  return s;
}
inline Jet operator+(Jet a, double s) {
  a.c[0] += s;
  return a;
}
inline Jet operator-(Jet a, double s) {
  a.c[0] -= s;
  return a;
}
inline Jet operator*(Jet a, double s) {
  for (double& x : a.c) x *= s;
  return a;
}
inline Jet operator*(double s, const Jet& a) { return a * s; }
inline Jet operator-(const Jet& a) { return a * -1.0; }
inline Jet operator-(double s, const Jet& a) { return (-a) + s; }

struct Problem {
  int kind = 0, dim = 0;
  double t_end = 0.0;
  std::vector<double> y0, params;
};

inline Problem resolve_problem(const pode_problem& p) {
  Problem q;
  q.kind = p.kind;
  q.dim = p.dim;
  q.t_end = p.t_end;
  if (p.dim < 1) throw ApiError(PODE_ERR_INVALID_INPUT, "problem: dim must be >= 1");
  if (p.y0 == nullptr) throw ApiError(PODE_ERR_INVALID_INPUT, "problem: y0 is NULL");
  q.y0.assign(p.y0, p.y0 + p.dim);
  if (p.n_params > 0) q.params.assign(p.params, p.params + p.n_params);
  int want_dim = 0;
  switch (p.kind) {
    case PODE_LOGISTIC: want_dim = 1; break;
    case PODE_RIGID_BODY: want_dim = 3; break;
    case PODE_VAN_DER_POL:
      want_dim = 2;
      if (q.params.empty()) q.params = {1.0};
      break;
    case PODE_FITZHUGH_NAGUMO:
      want_dim = 2;
      if (q.params.empty()) q.params = {0.2, 0.2, 3.0};
      break;
    case PODE_PLEIADES: want_dim = 28; break;
    case PODE_POLE:
      want_dim = 1;
      if (q.params.empty()) q.params = {0.75};
      break;
    case PODE_AFFINE:
      want_dim = p.dim;
      if (int(q.params.size()) != p.dim * p.dim + p.dim)
        throw ApiError(PODE_ERR_INVALID_INPUT, "affine problem: params must hold L (d*d) and c (d)");
      break;
    default:
      throw ApiError(PODE_ERR_INVALID_INPUT,
                     "problem: unknown kind (a problem without a registered device field cannot run "
                     "on the GPU; there is no CPU fallback)");
  }
  if (p.dim != want_dim) throw ApiError(PODE_ERR_DIMENSION, "problem: dimension does not match its kind");
  return q;
}

// t: the time series (prior.cpp:131-133 passes Jet::variable(0)); only
// PODE_POLE depends on it.
template <typename S>
std::vector<S> field_series(const Problem& p, const std::vector<S>& y, const S& t) {
  std::vector<S> out(size_t(p.dim), y[0]);
  switch (p.kind) {
    case PODE_POLE:
      out[0] = (y[0] * 0.0 + 1.0) / (t - p.params[0]);
      break;
    case PODE_LOGISTIC:
      out[0] = y[0] * (1.0 - y[0]);
      break;
    case PODE_RIGID_BODY:
      out[0] = -2.0 * (y[1] * y[2]);
      out[1] = 1.25 * (y[0] * y[2]);
      out[2] = -0.5 * (y[0] * y[1]);
      break;
    case PODE_VAN_DER_POL: {
      const double mu = p.params[0];
      out[0] = y[1];
      out[1] = mu * ((1.0 - y[0] * y[0]) * y[1] - y[0]);
      break;
    }
    case PODE_FITZHUGH_NAGUMO: {
      const double a = p.params[0], b = p.params[1], c = p.params[2];
      out[0] = c * ((y[0] - (y[0] * y[0] * y[0]) * (1.0 / 3.0)) + y[1]);
      out[1] = ((y[0] - a) + b * y[1]) * (-1.0 / c);
      break;
    }
    case PODE_PLEIADES: {
      constexpr int B = 7;
      for (int i = 0; i < B; ++i) {
        out[i] = y[2 * B + i];
        out[B + i] = y[3 * B + i];
      }
      for (int i = 0; i < B; ++i) {
        S ax = y[0] * 0.0, ay = y[0] * 0.0;
        for (int j = 0; j < B; ++j) {
          if (j == i) continue;
          const S dx = y[j] - y[i];
          const S dy = y[B + j] - y[B + i];
          const S r2 = dx * dx + dy * dy;
          const S r3 = r2 * jsqrt(r2);
          const double mj = double(j + 1);
          ax = ax + (mj * dx) / r3;
          ay = ay + (mj * dy) / r3;
        }
        out[2 * B + i] = ax;
        out[3 * B + i] = ay;
      }
      break;
    }
    default: {  // affine
      const int d = p.dim;
      for (int i = 0; i < d; ++i) {
        S acc = y[0] * 0.0 + p.params[size_t(d * d + i)];
        for (int j = 0; j < d; ++j) acc = acc + y[j] * p.params[size_t(i * d + j)];
        out[i] = acc;
      }
    }
  }
  return out;
}

// taylor_init (prior.cpp:119-168): mean = [y, y', .., y^(nu)] per dimension.
inline std::vector<double> taylor_init(const Problem& p, int nu) {
  if (nu < 1) throw ApiError(PODE_ERR_INVALID_INPUT, "taylor_init: need nu >= 1");
  const int d = p.dim;
  std::vector<Jet> y(static_cast<size_t>(d), Jet{nu});
  for (int i = 0; i < d; ++i) y[i] = Jet(nu, p.y0[i]);
  Jet t_series(nu, 0.0);
  if (nu >= 1) t_series.c[1] = 1.0;
  for (int k = 0; k + 1 <= nu; ++k) {
    const std::vector<Jet> fy = field_series<Jet>(p, y, t_series);
    for (int i = 0; i < d; ++i) {
      if (!std::isfinite(fy[i].c[k]))
        throw ApiError(PODE_ERR_INVALID_INPUT, "taylor_init: vector field is not finite at the initial point");
      y[i].c[k + 1] = fy[i].c[k] / (k + 1);
    }
  }
  std::vector<double> mean(size_t(d) * (nu + 1));
  double kfact = 1.0;
  for (int k = 0; k <= nu; ++k) {
    if (k > 0) kfact *= k;
    for (int i = 0; i < d; ++i) mean[i * (nu + 1) + k] = kfact * y[i].c[k];
  }
  return mean;
}

}  // namespace host
}  // namespace pode
