// ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp).
// Jets, problems, the IWP prior and EK0/EK1 linearisation:
// proj/include/paraode/jet.hpp, proj/src/problems.cpp, proj/src/prior.cpp,
// proj/src/statespace.cpp.
#include <cmath>
#include <type_traits>

#include "orc.hpp"

namespace orc {

// ------------------------------------------------------------------ jets ---
static void same_order(const Jet& a, const Jet& b) {
  if (a.c.size() != b.c.size())
    throw DimensionError("Jet: mixed truncation orders in one expression");
}
Jet operator+(const Jet& a, const Jet& b) {
  same_order(a, b);
  Jet o = a;
  for (std::size_t k = 0; k < o.c.size(); ++k) o.c[k] += b.c[k];
  return o;
}
Jet operator-(const Jet& a, const Jet& b) {
  same_order(a, b);
  Jet o = a;
  for (std::size_t k = 0; k < o.c.size(); ++k) o.c[k] -= b.c[k];
  return o;
}
// jet.hpp:65-74 — Cauchy product truncated at the common order.
Jet operator*(const Jet& a, const Jet& b) {
  same_order(a, b);
  Jet o(a.order());
  for (std::size_t k = 0; k < a.c.size(); ++k) {
    double acc = 0.0;
    for (std::size_t i = 0; i <= k; ++i) acc += a.c[i] * b.c[k - i];
    o.c[k] = acc;
  }
  return o;
}
// Extension (not in the reference): series division q = a / b,
// q_k = (a_k - sum_{i=1..k} b_i q_{k-i}) / b_0.
Jet operator/(const Jet& a, const Jet& b) {
  same_order(a, b);
  Jet q(a.order());
  for (std::size_t k = 0; k < a.c.size(); ++k) {
    double acc = a.c[k];
    for (std::size_t i = 1; i <= k; ++i) acc -= b.c[i] * q.c[k - i];
    q.c[k] = acc / b.c[0];
  }
  return q;
}
// Extension: series square root, s_k = (a_k - sum_{i=1..k-1} s_i s_{k-i}) / (2 s_0).
Jet jet_sqrt(const Jet& a) {
  Jet s(a.order());
  s.c[0] = std::sqrt(a.c[0]);
  for (std::size_t k = 1; k < a.c.size(); ++k) {
    double acc = a.c[k];
    for (std::size_t i = 1; i < k; ++i) acc -= s.c[i] * s.c[k - i];
    s.c[k] = acc / (2.0 * s.c[0]);
  }
  return s;
}
Jet operator-(const Jet& a) {
  Jet o = a;
  for (double& x : o.c) x = -x;
  return o;
}
Jet operator+(const Jet& a, double s) {
  Jet o = a;
  o.c[0] += s;
  return o;
}
Jet operator-(const Jet& a, double s) {
  Jet o = a;
  o.c[0] -= s;
  return o;
}
Jet operator*(const Jet& a, double s) {
  Jet o = a;
  for (double& x : o.c) x *= s;
  return o;
}
Jet operator+(double s, const Jet& a) { return a + s; }
Jet operator-(double s, const Jet& a) { return (-a) + s; }
Jet operator*(double s, const Jet& a) { return a * s; }

// -------------------------------------------------------------- problems ---
// One definition serves doubles and jets (problems.cpp:81-107 pattern).
namespace {

constexpr int kBodies = 7;

template <typename S>
std::vector<S> eval_field(const Problem& p, const std::vector<S>& y, const S& t) {
  std::vector<S> out(static_cast<std::size_t>(p.dim), y[0]);
  switch (p.kind) {
    case kLogistic:  // problems.cpp:83-88
      out[0] = y[0] * (1.0 - y[0]);
      break;
    case kRigidBody:  // problems.cpp:90-97
      out[0] = -2.0 * (y[1] * y[2]);
      out[1] = 1.25 * (y[0] * y[2]);
      out[2] = -0.5 * (y[0] * y[1]);
      break;
    case kVanDerPol: {  // problems.cpp:99-105
      const double mu = p.params[0];
      out[0] = y[1];
      out[1] = mu * ((1.0 - y[0] * y[0]) * y[1] - y[0]);
      break;
    }
    case kFitzHughNagumo: {  // new: y' = [c(y1 - y1^3/3 + y2), -(y1 - a + b y2)/c]
      const double a = p.params[0], b = p.params[1], c = p.params[2];
      out[0] = c * ((y[0] - (y[0] * y[0] * y[0]) * (1.0 / 3.0)) + y[1]);
      out[1] = ((y[0] - a) + b * y[1]) * (-1.0 / c);
      break;
    }
    case kPleiades: {  // new: 7 bodies, m_i = i, first-order d = 28
      for (int i = 0; i < kBodies; ++i) {
        out[i] = y[2 * kBodies + i];
        out[kBodies + i] = y[3 * kBodies + i];
      }
      for (int i = 0; i < kBodies; ++i) {
        S ax = y[0] * 0.0, ay = y[0] * 0.0;
        for (int j = 0; j < kBodies; ++j) {
          if (j == i) continue;
          const S dx = y[j] - y[i];
          const S dy = y[kBodies + j] - y[kBodies + i];
          const S r2 = dx * dx + dy * dy;
          S r3;
          if constexpr (std::is_same_v<S, double>) {
            r3 = r2 * std::sqrt(r2);
          } else {
            r3 = r2 * jet_sqrt(r2);
          }
          const double mj = static_cast<double>(j + 1);
          ax = ax + (mj * dx) / r3;
          ay = ay + (mj * dy) / r3;
        }
        out[2 * kBodies + i] = ax;
        out[3 * kBodies + i] = ay;
      }
      break;
    }
    case kAffine: {  // acceptance.cpp:34-55 (y' = L y + c)
      const int d = p.dim;
      for (int i = 0; i < d; ++i) {
        S acc = y[0] * 0.0 + p.params[static_cast<std::size_t>(d * d + i)];
        for (int j = 0; j < d; ++j) acc = acc + y[j] * p.params[static_cast<std::size_t>(i * d + j)];
        out[i] = acc;
      }
      break;
    }
    case kPole: {  // the reference's non-finite-field test (test_statespace.cpp:123-139), as a
                   // time pole so the failing node is known: y' = 1 / (t - a)
      out[0] = (y[0] * 0.0 + 1.0) / (t - p.params[0]);
      break;
    }
    default:
      throw InvalidInputError("unknown problem kind");
  }
  return out;
}

}  // namespace

Vec field(const Problem& p, const Vec& y, double t) { return eval_field<double>(p, y, t); }

std::vector<Jet> field_series(const Problem& p, const std::vector<Jet>& y, const Jet& t) {
  return eval_field<Jet>(p, y, t);
}

Mat jacobian(const Problem& p, const Vec& y, double) {
  const int d = p.dim;
  Mat j(d, d);
  switch (p.kind) {
    case kLogistic:  // problems.cpp:126-128
      j(0, 0) = 1.0 - 2.0 * y[0];
      break;
    case kRigidBody:  // problems.cpp:145-151
      j(0, 0) = 0.0, j(0, 1) = -2.0 * y[2], j(0, 2) = -2.0 * y[1];
      j(1, 0) = 1.25 * y[2], j(1, 1) = 0.0, j(1, 2) = 1.25 * y[0];
      j(2, 0) = -0.5 * y[1], j(2, 1) = -0.5 * y[0], j(2, 2) = 0.0;
      break;
    case kVanDerPol: {  // problems.cpp:167-172
      const double mu = p.params[0];
      j(0, 0) = 0.0, j(0, 1) = 1.0;
      j(1, 0) = -2.0 * mu * y[0] * y[1] - mu, j(1, 1) = mu * (1.0 - y[0] * y[0]);
      break;
    }
    case kFitzHughNagumo: {
      const double b = p.params[1], c = p.params[2];
      j(0, 0) = c * (1.0 - y[0] * y[0]), j(0, 1) = c;
      j(1, 0) = -1.0 / c, j(1, 1) = -b / c;
      break;
    }
    case kPleiades: {
      for (int i = 0; i < kBodies; ++i) {
        j(i, 2 * kBodies + i) = 1.0;
        j(kBodies + i, 3 * kBodies + i) = 1.0;
      }
      for (int i = 0; i < kBodies; ++i) {
        for (int k = 0; k < kBodies; ++k) {
          if (k == i) continue;
          const double dx = y[k] - y[i], dy = y[kBodies + k] - y[kBodies + i];
          const double r2 = dx * dx + dy * dy;
          const double r = std::sqrt(r2);
          const double r3 = r2 * r, r5 = r3 * r2;
          const double mk = static_cast<double>(k + 1);
          const double dxx = mk * (1.0 / r3 - 3.0 * dx * dx / r5);
          const double dxy = mk * (-3.0 * dx * dy / r5);
          const double dyy = mk * (1.0 / r3 - 3.0 * dy * dy / r5);
          // a_x,i depends on x_k, x_i, y_k, y_i
          j(2 * kBodies + i, k) += dxx;
          j(2 * kBodies + i, i) -= dxx;
          j(2 * kBodies + i, kBodies + k) += dxy;
          j(2 * kBodies + i, kBodies + i) -= dxy;
          j(3 * kBodies + i, k) += dxy;
          j(3 * kBodies + i, i) -= dxy;
          j(3 * kBodies + i, kBodies + k) += dyy;
          j(3 * kBodies + i, kBodies + i) -= dyy;
        }
      }
      break;
    }
    case kPole:
      j(0, 0) = 0.0;
      break;
    case kAffine:
      for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) j(r, c) = p.params[static_cast<std::size_t>(r * d + c)];
      break;
    default:
      throw InvalidInputError("unknown problem kind");
  }
  return j;
}

Problem make_problem(int kind) {
  Problem p;
  p.kind = kind;
  switch (kind) {
    case kLogistic:  // problems.cpp:116-135
      p.dim = 1, p.t_end = 10.0, p.y0 = {0.01};
      break;
    case kRigidBody:  // problems.cpp:137-157
      p.dim = 3, p.t_end = 20.0, p.y0 = {1.0, 0.0, 0.9};
      break;
    case kVanDerPol:  // problems.cpp:159-179
      p.dim = 2, p.t_end = 6.3, p.y0 = {2.0, 0.0}, p.params = {1.0};
      break;
    case kFitzHughNagumo:  // SURVEY.md §8c proposal
      p.dim = 2, p.t_end = 20.0, p.y0 = {-1.0, 1.0}, p.params = {0.2, 0.2, 3.0};
      break;
    case kPleiades: {  // Hairer–Nørsett–Wanner I
      p.dim = 4 * kBodies, p.t_end = 3.0;
      const double x0[kBodies] = {3, 3, -1, -3, 2, -2, 2};
      const double y0[kBodies] = {3, -3, 2, 0, 0, -4, 4};
      const double vx0[kBodies] = {0, 0, 0, 0, 0, 1.75, -1.5};
      const double vy0[kBodies] = {0, 0, 0, -1.25, 1, 0, 0};
      p.y0.assign(x0, x0 + kBodies);
      p.y0.insert(p.y0.end(), y0, y0 + kBodies);
      p.y0.insert(p.y0.end(), vx0, vx0 + kBodies);
      p.y0.insert(p.y0.end(), vy0, vy0 + kBodies);
      break;
    }
    case kPole:  // test_statespace.cpp:123-139 restated as a time pole at t = a
      p.dim = 1, p.t_end = 1.0, p.y0 = {0.0}, p.params = {0.75};
      break;
    default:
      throw InvalidInputError("unknown problem kind");
  }
  return p;
}

Problem make_affine(const Mat& l, const Vec& c, const Vec& y0, double t_end) {
  Problem p;
  p.kind = kAffine;
  p.dim = static_cast<int>(y0.size());
  p.t_end = t_end;
  p.y0 = y0;
  p.params = l.v;
  p.params.insert(p.params.end(), c.begin(), c.end());
  return p;
}

// proj/src/problems.cpp:212-221
std::vector<double> uniform_grid(double t_end, int steps) {
  if (steps < 1 || !(t_end > 0.0))
    throw InvalidInputError("uniform_grid: need steps >= 1 and t_end > 0");
  std::vector<double> g(static_cast<std::size_t>(steps) + 1);
  for (int n = 0; n <= steps; ++n)
    g[static_cast<std::size_t>(n)] = t_end * static_cast<double>(n) / static_cast<double>(steps);
  return g;
}

// ----------------------------------------------------------------- prior ---
namespace {

double factorial(int n) {  // prior.cpp:10-14
  double f = 1.0;
  for (int k = 2; k <= n; ++k) f *= k;
  return f;
}

double binomial(int n, int k) {  // prior.cpp:16-19
  if (k < 0 || k > n) return 0.0;
  return factorial(n) / (factorial(k) * factorial(n - k));
}

void check_prior(const IwpPrior& prior) {  // prior.cpp:21-28
  if (prior.nu < 1 || prior.dim < 1) throw InvalidInputError("IwpPrior: need nu >= 1 and dim >= 1");
  if (!(prior.sigma >= 0.0) || !std::isfinite(prior.sigma))
    throw InvalidInputError("IwpPrior: sigma must be finite and nonnegative");
}

Mat replicate_block(const Mat& b, int dim) {  // prior.cpp:30-37
  Mat full(b.r * dim, b.r * dim);
  for (int r = 0; r < dim; ++r) set_block(full, r * b.r, r * b.r, b);
  return full;
}

// Eigen::LLT (llt_inplace::unblocked): fails when a pivot is <= 0.
bool llt(const Mat& a, Mat& l) {
  const int n = a.r;
  l = Mat(n, n);
  for (int k = 0; k < n; ++k) {
    double x = a(k, k);
    for (int j = 0; j < k; ++j) x -= l(k, j) * l(k, j);
    if (!(x > 0.0)) return false;
    const double piv = std::sqrt(x);
    l(k, k) = piv;
    for (int i = k + 1; i < n; ++i) {
      double s = a(i, k);
      for (int j = 0; j < k; ++j) s -= l(i, j) * l(k, j);
      l(i, k) = s / piv;
    }
  }
  return true;
}

// Cyclic Jacobi symmetric eigensolver (stands in for
// Eigen::SelfAdjointEigenSolver in the psd_sqrt fallback).
void jacobi_eigen(Mat a, Vec& w, Mat& v) {
  const int n = a.r;
  v = Mat::identity(n);
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += a(p, q) * a(p, q);
    if (off < 1e-300) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (a(p, q) == 0.0) continue;
        const double theta = (a(q, q) - a(p, p)) / (2.0 * a(p, q));
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = v(k, p), vkq = v(k, q);
          v(k, p) = c * vkp - s * vkq;
          v(k, q) = s * vkp + c * vkq;
        }
      }
  }
  w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) w[i] = a(i, i);
}

// prior.cpp:43-51 — Cholesky, else eigenvalue-clipped square root re-triangularised.
Mat psd_sqrt(const Mat& b) {
  Mat l;
  if (llt(b, l)) return l;
  Vec w;
  Mat v;
  jacobi_eigen(b, w, v);
  for (double& x : w) x = std::sqrt(std::max(x, 0.0));
  return tria(diag_mul_right(v, w));
}

}  // namespace

// prior.cpp:55-77
TransitionModel iwp_transition(const IwpPrior& prior, double h) {
  check_prior(prior);
  if (!(h > 0.0) || !std::isfinite(h))
    throw InvalidInputError("iwp_transition: step must be finite and positive");
  const int nu = prior.nu;
  Mat phi(nu + 1, nu + 1), q(nu + 1, nu + 1);
  for (int i = 0; i <= nu; ++i) {
    for (int j = i; j <= nu; ++j) phi(i, j) = std::pow(h, j - i) / factorial(j - i);
    for (int j = 0; j <= nu; ++j) {
      const int p = 2 * nu + 1 - i - j;
      q(i, j) = std::pow(h, p) / (p * factorial(nu - i) * factorial(nu - j));
    }
  }
  TransitionModel t;
  t.phi = replicate_block(phi, prior.dim);
  t.q_sqrt = prior.sigma * replicate_block(psd_sqrt(q), prior.dim);
  t.step = h;
  return t;
}

// prior.cpp:79-97
Preconditioner preconditioner(const IwpPrior& prior, double h) {
  check_prior(prior);
  if (!(h > 0.0) || !std::isfinite(h))
    throw InvalidInputError("preconditioner: step must be finite and positive");
  const int nu = prior.nu;
  Preconditioner pc;
  pc.scale.assign(prior.state_dim(), 0.0);
  pc.scale_inv.assign(prior.state_dim(), 0.0);
  const double root_h = std::sqrt(h);
  for (int r = 0; r < prior.dim; ++r)
    for (int i = 0; i <= nu; ++i) {
      const double tau = root_h * std::pow(h, nu - i) / factorial(nu - i);
      pc.scale[r * (nu + 1) + i] = tau;
      pc.scale_inv[r * (nu + 1) + i] = 1.0 / tau;
    }
  return pc;
}

// prior.cpp:99-107
Mat preconditioned_phi(const IwpPrior& prior) {
  check_prior(prior);
  const int nu = prior.nu;
  Mat b(nu + 1, nu + 1);
  for (int i = 0; i <= nu; ++i)
    for (int j = i; j <= nu; ++j) b(i, j) = binomial(nu - i, j - i);
  return replicate_block(b, prior.dim);
}

// prior.cpp:109-117
Mat preconditioned_q_sqrt(const IwpPrior& prior) {
  check_prior(prior);
  const int nu = prior.nu;
  Mat b(nu + 1, nu + 1);
  for (int i = 0; i <= nu; ++i)
    for (int j = 0; j <= nu; ++j) b(i, j) = 1.0 / (2 * nu + 1 - i - j);
  return replicate_block(psd_sqrt(b), prior.dim);
}

// prior.cpp:119-168 (every registered problem carries a series field).
GaussianSqrt taylor_init(const Problem& p, int nu) {
  if (nu < 1) throw InvalidInputError("taylor_init: need nu >= 1");
  if (p.dim < 1 || static_cast<int>(p.y0.size()) != p.dim)
    throw InvalidInputError("taylor_init: problem dimension and y0 length disagree");
  const int d = p.dim;
  std::vector<Jet> y(static_cast<std::size_t>(d), Jet(nu));
  for (int i = 0; i < d; ++i) y[i] = Jet::constant(p.y0[i], nu);
  const Jet t_series = Jet::variable(0.0, nu);
  for (int k = 0; k + 1 <= nu; ++k) {
    std::vector<Jet> fy = field_series(p, y, t_series);
    if (static_cast<int>(fy.size()) != d)
      throw DimensionError("taylor_init: series field has the wrong output dimension");
    for (int i = 0; i < d; ++i) {
      if (!std::isfinite(fy[i].c[k]))
        throw InvalidInputError("taylor_init: vector field is not finite at the initial point");
      y[i].c[k + 1] = fy[i].c[k] / (k + 1);
    }
  }
  GaussianSqrt init;
  init.mean.assign(static_cast<std::size_t>(d * (nu + 1)), 0.0);
  double kfact = 1.0;
  for (int k = 0; k <= nu; ++k) {
    if (k > 0) kfact *= k;
    for (int i = 0; i < d; ++i) init.mean[i * (nu + 1) + k] = kfact * y[i].c[k];
  }
  init.cov_sqrt = Mat(d * (nu + 1), d * (nu + 1));
  return init;
}

// ----------------------------------------------------------- statespace ---
// statespace.cpp:8-17
Mat projection_matrix(int dim, int nu, int deriv) {
  if (dim < 1 || nu < 0 || deriv < 0 || deriv > nu)
    throw InvalidInputError("projection_matrix: need dim >= 1 and 0 <= deriv <= nu");
  Mat e(dim, dim * (nu + 1));
  for (int r = 0; r < dim; ++r) e(r, r * (nu + 1) + deriv) = 1.0;
  return e;
}

namespace {
void shape_for(const Problem& p, const Vec& eta, int& dim, int& nu) {  // statespace.cpp:42-50
  if (p.dim < 1) throw InvalidInputError("linearize: problem dimension must be >= 1");
  const int n = static_cast<int>(eta.size());
  if (n % p.dim != 0 || n < 2 * p.dim)
    throw DimensionError("linearize: state length must be dim * (nu + 1) with nu >= 1");
  dim = p.dim;
  nu = n / p.dim - 1;
}
}  // namespace

// statespace.cpp:65-88
AffineObservation linearize_ek1(const Problem& p, const Vec& eta, double t) {
  int dim, nu;
  shape_for(p, eta, dim, nu);
  Vec y(dim);
  for (int r = 0; r < dim; ++r) y[r] = eta[r * (nu + 1)];
  const Vec fy = field(p, y, t);
  if (!all_finite(fy)) throw LinearizationError("linearize: vector field evaluation is not finite", t, 0);
  const Mat jac = jacobian(p, y, t);
  if (!all_finite(jac)) throw LinearizationError("linearize: Jacobian evaluation is not finite", t, 0);
  Mat h(dim, static_cast<int>(eta.size()));
  for (int r = 0; r < dim; ++r) {
    h(r, r * (nu + 1) + 1) = 1.0;
    for (int c = 0; c < dim; ++c) h(r, c * (nu + 1)) = -jac(r, c);
  }
  AffineObservation obs;
  obs.h = h;
  obs.offset = fy - jac * y;
  obs.r_sqrt = Mat(dim, dim);
  return obs;
}

// statespace.cpp:90-103
AffineObservation linearize_ek0(const Problem& p, const Vec& eta, double t) {
  int dim, nu;
  shape_for(p, eta, dim, nu);
  Vec y(dim);
  for (int r = 0; r < dim; ++r) y[r] = eta[r * (nu + 1)];
  const Vec fy = field(p, y, t);
  if (!all_finite(fy)) throw LinearizationError("linearize: vector field evaluation is not finite", t, 0);
  Mat h(dim, static_cast<int>(eta.size()));
  for (int r = 0; r < dim; ++r) h(r, r * (nu + 1) + 1) = 1.0;
  AffineObservation obs;
  obs.h = h;
  obs.offset = fy;
  obs.r_sqrt = Mat(dim, dim);
  return obs;
}

AffineObservation linearize(const Problem& p, const Vec& eta, double t, Linearization kind) {
  return kind == Linearization::kEk1 ? linearize_ek1(p, eta, t) : linearize_ek0(p, eta, t);
}

}  // namespace orc
