// paraode.hpp — source-compatible drop-in for the reference's ParaIEKS path
// (proj/include/paraode/{statespace,sequential,parallel,prior,ieks,problems,
// work_pool,errors}.hpp): the same namespace, type names, function names,
// signatures, argument meaning and exception types, with every computation
// on the B200 through the C ABI (include/paraode_b200.h).  A caller of
// para_ieks / seq_ieks / eks_solve / para_rts / seq_rts / the element
// operators / associative_scan recompiles against this header and links
// libparaode_b200.so instead of the reference library.
//
// Differences a caller can observe (each a consequence of running on the GPU):
//   * InitialValueProblem gains `registered` (a device vector field: kind +
//     params).  The shipped problems (logistic(), rigid_body(),
//     van_der_pol(), fitzhugh_nagumo(), pleiades(), problem_by_name()) are
//     registered; a problem with only host std::function callbacks throws
//     InvalidInputError from the solvers (there is no CPU fallback).
//   * WorkPool is the device context (a CUDA stream + workspace on one GPU);
//     its width is recorded but the GPU grid replaces the host threads.
//   * associative_scan runs the path's own operators on the GPU
//     (combine_filtering / combine_smoothing); any other operator or element
//     type throws InvalidInputError.
//   * Square-root factors are lower triangular but, like the reference's
//     Householder factors, only L L^T is pinned (linalg.hpp:12-17).
// Matrix / Vector are Eigen::MatrixXd / Eigen::VectorXd when <Eigen/Dense>
// is on the include path (linalg.hpp:9-10), otherwise a minimal dense type
// with the subset of that interface this header uses.
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "paraode_b200.hpp"

#if defined(__has_include)
#if __has_include(<Eigen/Dense>) && !defined(PARAODE_NO_EIGEN)
#include <Eigen/Dense>
#define PARAODE_HAVE_EIGEN 1
#endif
#endif

namespace paraode {

#ifdef PARAODE_HAVE_EIGEN
using Matrix = Eigen::MatrixXd;
using Vector = Eigen::VectorXd;
using Index = Eigen::Index;
#else
using Index = std::ptrdiff_t;
// Row-major dense stand-ins for Eigen::MatrixXd / VectorXd.
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols) : r_(rows), c_(cols), v_(size_t(rows * cols), 0.0) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  double& operator()(Index i, Index j) { return v_[size_t(i * c_ + j)]; }
  double operator()(Index i, Index j) const { return v_[size_t(i * c_ + j)]; }
  static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
  static Matrix Identity(Index n, Index = -1) {
    Matrix m(n, n);
    for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> v_;
};
class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n) : v_(size_t(n), 0.0) {}
  Vector(std::initializer_list<double> x) : v_(x) {}
  Index size() const { return Index(v_.size()); }
  double& operator()(Index i) { return v_[size_t(i)]; }
  double operator()(Index i) const { return v_[size_t(i)]; }
  double& operator[](Index i) { return v_[size_t(i)]; }
  double operator[](Index i) const { return v_[size_t(i)]; }
  static Vector Zero(Index n) { return Vector(n); }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }

 private:
  std::vector<double> v_;
};
#endif

// ------------------------------------------------------------- errors ---
// errors.hpp:10-60 (the same classes as the shim, under the reference's names)
using SolverError = b200::SolverError;
using InvalidInputError = b200::InvalidInputError;
using DimensionError = b200::DimensionError;
using SingularFactorError = b200::SingularFactorError;
using LinearizationError = b200::LinearizationError;
using ScanError = b200::ScanError;

// ------------------------------------------------------------- types ---
struct GaussianSqrt {  // statespace.hpp:13-16
  Vector mean;
  Matrix cov_sqrt;
};
struct AffineObservation {  // statespace.hpp:36-40
  Matrix h;
  Vector offset;
  Matrix r_sqrt;
};
struct TransitionModel {  // statespace.hpp:44-48
  Matrix phi;
  Matrix q_sqrt;
  double step = 0.0;
};
enum class Linearization { kEk1, kEk0 };

// A device vector field: the registry of include/paraode_b200.h.
struct RegisteredField {
  bool valid = false;
  pode_problem_kind kind = PODE_LOGISTIC;
  std::vector<double> params;
};

struct InitialValueProblem {  // statespace.hpp:24-31 (+ registered)
  int dim = 0;
  double t_end = 0.0;
  Vector y0;
  std::function<Vector(const Vector&, double)> field;
  std::function<Matrix(const Vector&, double)> jacobian;
  RegisteredField registered;  // required on the B200
};

struct FilteringElement {  // parallel.hpp:20-26
  Matrix a;
  Vector b;
  Matrix c_sqrt;
  Vector eta;
  Matrix j_sqrt;
};
struct SmoothingElement {  // parallel.hpp:32-36
  Matrix e;
  Vector g;
  Matrix l_sqrt;
};
struct ScanStats {  // sequential.hpp:42-50
  std::size_t combine_invocations = 0;
  std::size_t sequential_depth = 0;
  void merge_max(const ScanStats& other) {
    combine_invocations = std::max(combine_invocations, other.combine_invocations);
    sequential_depth = std::max(sequential_depth, other.sequential_depth);
  }
};
struct RtsResult {  // sequential.hpp:52-56
  std::vector<GaussianSqrt> filtered;
  std::vector<GaussianSqrt> smoothed;
  ScanStats stats;
};
struct IwpPrior {  // prior.hpp:12-18
  int nu = 1;
  int dim = 1;
  double sigma = 1.0;
  int state_dim() const { return dim * (nu + 1); }
};
struct IeksConfig {  // ieks.hpp:32-38
  int max_iterations = 100;
  double traj_rtol = 1e-13;
  double obj_atol = 1e-9;
  double obj_rtol = 1e-6;
  Linearization linearization = Linearization::kEk1;
};
struct SolverReport {  // ieks.hpp:77-87
  std::vector<double> times;
  std::vector<GaussianSqrt> marginals;
  std::vector<Vector> solution_means;
  std::vector<Matrix> solution_covs;
  double sigma_hat = 0.0;
  int iterations = 0;
  std::vector<double> objective_trace;
  bool converged = false;
  ScanStats scan_stats;
};

// work_pool.hpp:21-64: the execution resource a solve runs on.  On the B200
// it owns a device context (stream + workspace on GPU `device`); width is
// kept for source compatibility.  Not reentrant, like WorkPool.
class WorkPool {
 public:
  explicit WorkPool(unsigned width = 0, int device = 0) : width_(width ? width : 1), dev_(new b200::Device(device)) {}
  WorkPool(const WorkPool&) = delete;
  WorkPool& operator=(const WorkPool&) = delete;
  unsigned width() const { return width_; }
  pode_context* handle() const { return dev_->handle(); }

 private:
  unsigned width_;
  std::unique_ptr<b200::Device> dev_;
};

namespace detail {
inline WorkPool& default_pool() {  // seq_* and the element operators
  static WorkPool pool(1);
  return pool;
}
inline void check(int rc, const pode_status& st) { b200::check(rc, st); }
inline void put(const Matrix& m, double* dst, Index rows, Index cols) {
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < cols; ++j) dst[i * cols + j] = (i < m.rows() && j < m.cols()) ? m(i, j) : 0.0;
}
inline void putv(const Vector& v, double* dst, Index n) {
  for (Index i = 0; i < n; ++i) dst[i] = i < v.size() ? v(i) : 0.0;
}
inline Matrix get(const double* src, Index rows, Index cols) {
  Matrix m(rows, cols);
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < cols; ++j) m(i, j) = src[i * cols + j];
  return m;
}
inline Vector getv(const double* src, Index n) {
  Vector v(n);
  for (Index i = 0; i < n; ++i) v(i) = src[i];
  return v;
}
// Host mirrors of arrays of elements (row-major, pode_*_elements layout).
struct FBuf {
  std::vector<double> a, b, c, eta, j;
  Index n = 0, D = 0;
  FBuf(Index count, Index dim) : a(size_t(count * dim * dim)), b(size_t(count * dim)), c(size_t(count * dim * dim)),
                                 eta(size_t(count * dim)), j(size_t(count * dim * dim)), n(count), D(dim) {}
  pode_filtering_elements view() { return {a.data(), b.data(), c.data(), eta.data(), j.data()}; }
  void set(Index i, const FilteringElement& e) {
    put(e.a, &a[size_t(i * D * D)], D, D);
    putv(e.b, &b[size_t(i * D)], D);
    put(e.c_sqrt, &c[size_t(i * D * D)], D, D);
    putv(e.eta, &eta[size_t(i * D)], D);
    put(e.j_sqrt, &j[size_t(i * D * D)], D, D);
  }
  FilteringElement at(Index i) const {
    return {get(&a[size_t(i * D * D)], D, D), getv(&b[size_t(i * D)], D), get(&c[size_t(i * D * D)], D, D),
            getv(&eta[size_t(i * D)], D), get(&j[size_t(i * D * D)], D, D)};
  }
};
struct SBuf {
  std::vector<double> e, g, l;
  Index n = 0, D = 0;
  SBuf(Index count, Index dim) : e(size_t(count * dim * dim)), g(size_t(count * dim)), l(size_t(count * dim * dim)),
                                 n(count), D(dim) {}
  pode_smoothing_elements view() { return {e.data(), g.data(), l.data()}; }
  void set(Index i, const SmoothingElement& x) {
    put(x.e, &e[size_t(i * D * D)], D, D);
    putv(x.g, &g[size_t(i * D)], D);
    put(x.l_sqrt, &l[size_t(i * D * D)], D, D);
  }
  SmoothingElement at(Index i) const {
    return {get(&e[size_t(i * D * D)], D, D), getv(&g[size_t(i * D)], D), get(&l[size_t(i * D * D)], D, D)};
  }
};
// A chain (init, N transitions, N observations) in the C ABI's layout.
struct ChainBuf {
  std::vector<double> im, ic, phi, q, h, off, r;
  std::vector<int32_t> rows;
  pode_chain ch{};
  ChainBuf(const GaussianSqrt& init, const std::vector<TransitionModel>& tr, const std::vector<AffineObservation>& ob,
           const char* who) {
    if (tr.empty() || tr.size() != ob.size())
      throw DimensionError(std::string(who) + ": need N >= 1 aligned transitions and observations");
    const Index D = init.mean.size(), N = Index(tr.size());
    Index M = 0;
    for (const auto& o : ob) M = std::max<Index>(M, o.h.rows());
    const Index Mm = std::max<Index>(M, 1);
    im.resize(size_t(D));
    ic.resize(size_t(D * D));
    phi.resize(size_t(N * D * D));
    q.resize(size_t(N * D * D));
    h.resize(size_t(N * Mm * D));
    off.resize(size_t(N * Mm));
    r.resize(size_t(N * Mm * Mm));
    rows.resize(size_t(N));
    putv(init.mean, im.data(), D);
    put(init.cov_sqrt, ic.data(), D, D);
    for (Index n = 0; n < N; ++n) {
      const auto& o = ob[size_t(n)];
      if (tr[size_t(n)].phi.rows() != D || tr[size_t(n)].q_sqrt.rows() != D || (o.h.rows() > 0 && o.h.cols() != D) ||
          o.offset.size() != o.h.rows())
        throw DimensionError(std::string(who) + ": observation dimensions disagree with the state");
      put(tr[size_t(n)].phi, &phi[size_t(n * D * D)], D, D);
      put(tr[size_t(n)].q_sqrt, &q[size_t(n * D * D)], D, D);
      rows[size_t(n)] = int32_t(o.h.rows());
      put(o.h, &h[size_t(n * Mm * D)], Mm, D);
      putv(o.offset, &off[size_t(n * Mm)], Mm);
      put(o.r_sqrt, &r[size_t(n * Mm * Mm)], Mm, Mm);
    }
    ch = pode_chain{int32_t(D), int32_t(M), int64_t(N), im.data(), ic.data(), phi.data(), q.data(), 0, 0,
                    rows.data(), h.data(), off.data(), r.data(), PODE_HOST};
  }
};
}  // namespace detail

// ------------------------------------------------- element operators ---
// parallel.hpp:43-75 (one element each: a batch of one on the GPU)
inline FilteringElement make_filtering_element(const TransitionModel& trans, const AffineObservation& obs,
                                               const GaussianSqrt* init = nullptr) {
  const Index D = trans.phi.rows();
  GaussianSqrt zero{Vector::Zero(D), Matrix::Zero(D, D)};
  detail::ChainBuf cb(init ? *init : zero, {trans}, {obs}, "make_filtering_element");
  detail::FBuf out(1, D);
  pode_status st{};
  detail::check(pode_make_filtering_elements(detail::default_pool().handle(), &cb.ch, init ? 1 : 0, out.view(), &st),
                st);
  return out.at(0);
}
inline FilteringElement combine_filtering(const FilteringElement& lhs, const FilteringElement& rhs) {
  const Index D = lhs.a.rows();
  if (rhs.a.rows() != D) throw DimensionError("combine_filtering: element dimensions disagree");
  detail::FBuf l(1, D), r(1, D), o(1, D);
  l.set(0, lhs);
  r.set(0, rhs);
  pode_status st{};
  detail::check(pode_combine_filtering(detail::default_pool().handle(), 1, int32_t(D), l.view(), r.view(), o.view(),
                                       PODE_HOST, &st),
                st);
  return o.at(0);
}
inline FilteringElement filtering_identity(Index state_dim) {  // parallel.cpp:102-110
  return {Matrix::Identity(state_dim, state_dim), Vector::Zero(state_dim), Matrix::Zero(state_dim, state_dim),
          Vector::Zero(state_dim), Matrix::Zero(state_dim, state_dim)};
}
inline SmoothingElement make_smoothing_element(const GaussianSqrt& filtered, const TransitionModel& trans) {
  const Index D = filtered.mean.size();
  AffineObservation none{Matrix::Zero(0, D), Vector::Zero(0), Matrix::Zero(0, 0)};
  detail::ChainBuf cb(filtered, {trans}, {none}, "make_smoothing_element");
  std::vector<double> fm(size_t(2 * D)), fc(size_t(2 * D * D));
  detail::putv(filtered.mean, fm.data(), D);
  detail::put(filtered.cov_sqrt, fc.data(), D, D);
  detail::putv(filtered.mean, fm.data() + D, D);
  detail::put(filtered.cov_sqrt, fc.data() + D * D, D, D);
  detail::SBuf out(2, D);
  pode_status st{};
  detail::check(pode_make_smoothing_elements(detail::default_pool().handle(), &cb.ch, fm.data(), fc.data(), out.view(),
                                             &st),
                st);
  return out.at(0);
}
inline SmoothingElement terminal_smoothing_element(const GaussianSqrt& filtered) {  // parallel.cpp:137-144
  const Index D = filtered.mean.size();
  return {Matrix::Zero(D, D), filtered.mean, filtered.cov_sqrt};
}
inline SmoothingElement combine_smoothing(const SmoothingElement& lhs, const SmoothingElement& rhs) {
  const Index D = lhs.e.rows();
  if (rhs.e.rows() != D) throw DimensionError("combine_smoothing: element dimensions disagree");
  detail::SBuf l(1, D), r(1, D), o(1, D);
  l.set(0, lhs);
  r.set(0, rhs);
  pode_status st{};
  detail::check(pode_combine_smoothing(detail::default_pool().handle(), 1, int32_t(D), l.view(), r.view(), o.view(),
                                       PODE_HOST, &st),
                st);
  return o.at(0);
}
inline SmoothingElement smoothing_identity(Index state_dim) {  // parallel.cpp:158-164
  return {Matrix::Identity(state_dim, state_dim), Vector::Zero(state_dim), Matrix::Zero(state_dim, state_dim)};
}

// --------------------------------------------------- associative_scan ---
// parallel.hpp:136-149.  The B200 scans run the path's operators: op must be
// combine_filtering (FilteringElement) or combine_smoothing
// (SmoothingElement).  stats receive the GPU tree's combines and depth.
enum class ScanDirection { kForward, kReverse };

inline std::vector<FilteringElement> associative_scan(FilteringElement (*op)(const FilteringElement&,
                                                                             const FilteringElement&),
                                                      std::vector<FilteringElement> elems, ScanDirection direction,
                                                      ScanStats& stats, WorkPool& pool) {
  if (op != &combine_filtering)
    throw InvalidInputError("associative_scan: only combine_filtering scans FilteringElements on the B200");
  if (elems.size() < 2) return elems;
  const Index n = Index(elems.size()), D = elems[0].a.rows();
  detail::FBuf io(n, D);
  for (Index i = 0; i < n; ++i) io.set(i, elems[size_t(i)]);
  pode_scan_stats s{};
  pode_status st{};
  detail::check(pode_scan_filtering(pool.handle(), n, int32_t(D), io.view(), io.view(),
                                    direction == ScanDirection::kReverse ? 1 : 0, PODE_HOST, &s, &st),
                st);
  stats.combine_invocations += std::size_t(s.combine_invocations);
  stats.sequential_depth += std::size_t(s.sequential_depth);
  for (Index i = 0; i < n; ++i) elems[size_t(i)] = io.at(i);
  return elems;
}
inline std::vector<SmoothingElement> associative_scan(SmoothingElement (*op)(const SmoothingElement&,
                                                                             const SmoothingElement&),
                                                      std::vector<SmoothingElement> elems, ScanDirection direction,
                                                      ScanStats& stats, WorkPool& pool) {
  if (op != &combine_smoothing)
    throw InvalidInputError("associative_scan: only combine_smoothing scans SmoothingElements on the B200");
  if (elems.size() < 2) return elems;
  const Index n = Index(elems.size()), D = elems[0].e.rows();
  detail::SBuf io(n, D);
  for (Index i = 0; i < n; ++i) io.set(i, elems[size_t(i)]);
  pode_scan_stats s{};
  pode_status st{};
  detail::check(pode_scan_smoothing(pool.handle(), n, int32_t(D), io.view(), io.view(),
                                    direction == ScanDirection::kReverse ? 1 : 0, PODE_HOST, &s, &st),
                st);
  stats.combine_invocations += std::size_t(s.combine_invocations);
  stats.sequential_depth += std::size_t(s.sequential_depth);
  for (Index i = 0; i < n; ++i) elems[size_t(i)] = io.at(i);
  return elems;
}
// Any other operator: no GPU implementation (and no CPU fallback).
template <typename Elem, typename Op>
std::vector<Elem> associative_scan(const Op&, std::vector<Elem>, ScanDirection, ScanStats&, WorkPool&) {
  throw InvalidInputError("associative_scan: only the ParaIEKS operators (combine_filtering, combine_smoothing) "
                          "run on the B200");
}

// ----------------------------------------------------------- smoothers ---
namespace detail {
inline RtsResult rts(const GaussianSqrt& init, const std::vector<TransitionModel>& transitions,
                     const std::vector<AffineObservation>& observations, WorkPool& pool, const char* who) {
  ChainBuf cb(init, transitions, observations, who);
  const Index D = init.mean.size(), n1 = Index(transitions.size()) + 1;
  std::vector<double> fm(size_t(n1 * D)), fc(size_t(n1 * D * D)), sm(size_t(n1 * D)), sc(size_t(n1 * D * D));
  pode_rts_out out{fm.data(), fc.data(), sm.data(), sc.data()};
  pode_scan_stats s{};
  pode_status st{};
  check(pode_rts(pool.handle(), &cb.ch, out, &s, &st), st);
  RtsResult res;
  res.filtered.resize(size_t(n1));
  res.smoothed.resize(size_t(n1));
  for (Index n = 0; n < n1; ++n) {
    res.filtered[size_t(n)] = {getv(&fm[size_t(n * D)], D), get(&fc[size_t(n * D * D)], D, D)};
    res.smoothed[size_t(n)] = {getv(&sm[size_t(n * D)], D), get(&sc[size_t(n * D * D)], D, D)};
  }
  res.stats.combine_invocations = std::size_t(s.combine_invocations);
  res.stats.sequential_depth = std::size_t(s.sequential_depth);
  return res;
}
}  // namespace detail

// parallel.hpp:155-156
inline RtsResult para_rts(const GaussianSqrt& init, const std::vector<TransitionModel>& transitions,
                          const std::vector<AffineObservation>& observations, WorkPool& pool) {
  return detail::rts(init, transitions, observations, pool, "para_rts");
}
// sequential.hpp:59-60: the same smoother on the GPU (the association order
// differs from kf_forward + rts_smooth_pass only in rounding); stats zero as
// in the reference's sequential path.
inline RtsResult seq_rts(const GaussianSqrt& init, const std::vector<TransitionModel>& transitions,
                         const std::vector<AffineObservation>& observations) {
  RtsResult r = detail::rts(init, transitions, observations, detail::default_pool(), "seq_rts");
  r.stats = ScanStats{};
  return r;
}

// --------------------------------------------------------------- ieks ---
namespace detail {
// Host output buffers of one pode_ieks_report and their conversion to SolverReport.
struct ReportBuf {
  std::vector<double> means, cov, sm, sc, trace;
  pode_ieks_report rep;
  ReportBuf(Index n1, Index D, Index d, int max_iterations)
      : means(size_t(n1 * D)), cov(size_t(n1 * D * D)), sm(size_t(n1 * d)), sc(size_t(n1 * d * d)),
        trace(size_t(std::max(max_iterations, 1))),
        rep{means.data(), cov.data(), sm.data(), sc.data(), trace.data(), int32_t(trace.size()), PODE_HOST, 0, 0,
            0.0, {0, 0}} {}
  ReportBuf(const ReportBuf&) = delete;
  ReportBuf& operator=(const ReportBuf&) = delete;
  SolverReport report(const std::vector<double>& grid, Index D, Index d) const;
};

inline SolverReport ieks(const InitialValueProblem& ivp, const IwpPrior& prior, const std::vector<double>& grid,
                         const IeksConfig& config, WorkPool& pool, bool eks, int64_t chunk) {
  if (!ivp.registered.valid)
    throw InvalidInputError("ieks: the problem has only host callbacks; the B200 path needs a registered device "
                            "field (InitialValueProblem::registered) — there is no CPU fallback");
  if (ivp.dim != prior.dim) throw DimensionError("ieks: problem and prior dimensions disagree");
  const Index D = prior.state_dim(), d = prior.dim, n1 = Index(grid.size());
  std::vector<double> y0(size_t(ivp.dim));
  putv(ivp.y0, y0.data(), ivp.dim);
  pode_problem p{int32_t(ivp.registered.kind), ivp.dim, ivp.t_end, y0.data(),
                 ivp.registered.params.empty() ? nullptr : ivp.registered.params.data(),
                 int32_t(ivp.registered.params.size())};
  pode_prior pr{prior.nu, prior.dim, prior.sigma};
  const int lin = config.linearization == Linearization::kEk0 ? 1 : 0;
  pode_ieks_config cfg{config.max_iterations, config.traj_rtol, config.obj_atol, config.obj_rtol, lin};
  ReportBuf b(n1, D, d, config.max_iterations);
  pode_status st{};
  pode_context_set_option(pool.handle(), PODE_OPT_CHUNK_LEN, chunk);
  const int rc = eks ? pode_eks(pool.handle(), &p, &pr, grid.data(), n1, lin, &b.rep, &st)
                     : pode_ieks(pool.handle(), &p, &pr, grid.data(), n1, &cfg, &b.rep, &st);
  pode_context_set_option(pool.handle(), PODE_OPT_CHUNK_LEN, 0);
  check(rc, st);
  return b.report(grid, D, d);
}

inline pode_problem registered(const InitialValueProblem& ivp, std::vector<double>& y0) {
  if (!ivp.registered.valid)
    throw InvalidInputError("ieks: the problem has only host callbacks; the B200 path needs a registered device "
                            "field (InitialValueProblem::registered) — there is no CPU fallback");
  y0.resize(size_t(ivp.dim));
  putv(ivp.y0, y0.data(), ivp.dim);
  return pode_problem{int32_t(ivp.registered.kind), ivp.dim, ivp.t_end, y0.data(),
                      ivp.registered.params.empty() ? nullptr : ivp.registered.params.data(),
                      int32_t(ivp.registered.params.size())};
}
}  // namespace detail

namespace detail {
inline SolverReport ReportBuf::report(const std::vector<double>& grid, Index D, Index d) const {
  const Index n1 = Index(grid.size());
  SolverReport out;
  out.times = grid;
  out.marginals.resize(size_t(n1));
  out.solution_means.resize(size_t(n1));
  out.solution_covs.resize(size_t(n1));
  for (Index n = 0; n < n1; ++n) {
    out.marginals[size_t(n)] = {getv(&means[size_t(n * D)], D), get(&cov[size_t(n * D * D)], D, D)};
    out.solution_means[size_t(n)] = getv(&sm[size_t(n * d)], d);
    out.solution_covs[size_t(n)] = get(&sc[size_t(n * d * d)], d, d);
  }
  out.sigma_hat = rep.sigma_hat;
  out.iterations = rep.iterations;
  out.objective_trace.assign(trace.begin(), trace.begin() + rep.iterations);
  out.converged = rep.converged != 0;
  out.scan_stats.combine_invocations = std::size_t(rep.scan_stats.combine_invocations);
  out.scan_stats.sequential_depth = std::size_t(rep.scan_stats.sequential_depth);
  return out;
}
}  // namespace detail

// ieks.hpp:95-96
inline SolverReport para_ieks(const InitialValueProblem& ivp, const IwpPrior& prior, const std::vector<double>& grid,
                              const IeksConfig& config, WorkPool& pool) {
  return detail::ieks(ivp, prior, grid, config, pool, false, 0);
}
// ieks.hpp:98-99: the Kalman recursion in time order — the fused engine with
// the whole grid as one chunk (same iterates as para_ieks up to rounding).
inline SolverReport seq_ieks(const InitialValueProblem& ivp, const IwpPrior& prior, const std::vector<double>& grid,
                             const IeksConfig& config) {
  SolverReport r = detail::ieks(ivp, prior, grid, config, detail::default_pool(), false,
                                std::max<int64_t>(2, int64_t(grid.size()) - 1));
  r.scan_stats = ScanStats{};
  return r;
}
// ieks.hpp:103-105
inline SolverReport eks_solve(const InitialValueProblem& ivp, const IwpPrior& prior, const std::vector<double>& grid,
                              Linearization linearization = Linearization::kEk1) {
  IeksConfig cfg;
  cfg.linearization = linearization;
  return detail::ieks(ivp, prior, grid, cfg, detail::default_pool(), true, 0);
}

// Batched para_ieks (no reference counterpart — the reference solves one IVP
// per call): IVPs of one registered field kind and
// dimension with one prior, grid and config, fused into one device solve
// (pode_ieks_batch).  Element i equals para_ieks(ivps[i], ...) at the
// reference's tolerances, with its own iteration count.
inline std::vector<SolverReport> para_ieks_batch(const std::vector<InitialValueProblem>& ivps, const IwpPrior& prior,
                                                 const std::vector<double>& grid, const IeksConfig& config,
                                                 WorkPool& pool) {
  const Index D = prior.state_dim(), d = prior.dim, n1 = Index(grid.size());
  std::vector<std::vector<double>> y0(ivps.size());
  std::vector<pode_problem> ps;
  std::vector<std::unique_ptr<detail::ReportBuf>> bufs;
  std::vector<pode_ieks_report> reps;
  for (size_t i = 0; i < ivps.size(); ++i) {
    if (ivps[i].dim != prior.dim) throw DimensionError("ieks: problem and prior dimensions disagree");
    ps.push_back(detail::registered(ivps[i], y0[i]));
    bufs.push_back(std::make_unique<detail::ReportBuf>(n1, D, d, config.max_iterations));
    reps.push_back(bufs.back()->rep);
  }
  if (ps.empty()) return {};
  pode_prior pr{prior.nu, prior.dim, prior.sigma};
  const int lin = config.linearization == Linearization::kEk0 ? 1 : 0;
  pode_ieks_config cfg{config.max_iterations, config.traj_rtol, config.obj_atol, config.obj_rtol, lin};
  pode_status st{};
  detail::check(pode_ieks_batch(pool.handle(), ps.data(), int32_t(ps.size()), &pr, grid.data(), n1, &cfg,
                                reps.data(), &st),
                st);
  std::vector<SolverReport> out;
  for (size_t i = 0; i < ps.size(); ++i) {
    bufs[i]->rep = reps[i];  // iterations, convergence, sigma-hat
    out.push_back(bufs[i]->report(grid, D, d));
  }
  return out;
}

// ----------------------------------------------------------- problems ---
// problems.hpp:45-66 (+ FitzHugh-Nagumo and Pleiades):
// registered device fields with host field callbacks for source compatibility.
struct NamedProblem {
  std::string name;
  InitialValueProblem ivp;
  std::function<Vector(double)> reference;  // not provided (the GPU RK4 table is pode_rk4_table)
};
namespace detail {
inline NamedProblem named(const std::string& name, pode_problem_kind kind, int dim, double t_end,
                          std::vector<double> y0, std::vector<double> params,
                          std::function<Vector(const Vector&, double)> field) {
  NamedProblem p;
  p.name = name;
  p.ivp.dim = dim;
  p.ivp.t_end = t_end;
  p.ivp.y0 = Vector(dim);
  for (int i = 0; i < dim; ++i) p.ivp.y0(i) = y0[size_t(i)];
  p.ivp.field = std::move(field);
  p.ivp.registered = RegisteredField{true, kind, std::move(params)};
  return p;
}
}  // namespace detail
inline NamedProblem logistic() {
  return detail::named("logistic", PODE_LOGISTIC, 1, 10.0, {0.01}, {}, [](const Vector& y, double) {
    Vector f(1);
    f(0) = y(0) * (1.0 - y(0));
    return f;
  });
}
inline NamedProblem rigid_body() {
  return detail::named("rigidbody", PODE_RIGID_BODY, 3, 20.0, {1.0, 0.0, 0.9}, {}, [](const Vector& y, double) {
    Vector f(3);
    f(0) = -2.0 * (y(1) * y(2));
    f(1) = 1.25 * (y(0) * y(2));
    f(2) = -0.5 * (y(0) * y(1));
    return f;
  });
}
inline NamedProblem van_der_pol(double mu = 1.0) {
  return detail::named("vanderpol", PODE_VAN_DER_POL, 2, 6.3, {2.0, 0.0}, {mu}, [mu](const Vector& y, double) {
    Vector f(2);
    f(0) = y(1);
    f(1) = mu * ((1.0 - y(0) * y(0)) * y(1) - y(0));
    return f;
  });
}
inline NamedProblem fitzhugh_nagumo(double a = 0.2, double b = 0.2, double c = 3.0) {
  return detail::named("fhn", PODE_FITZHUGH_NAGUMO, 2, 20.0, {-1.0, 1.0}, {a, b, c},
                       [a, b, c](const Vector& y, double) {
                         Vector f(2);
                         f(0) = c * ((y(0) - (y(0) * y(0) * y(0)) * (1.0 / 3.0)) + y(1));
                         f(1) = ((y(0) - a) + b * y(1)) * (-1.0 / c);
                         return f;
                       });
}
inline NamedProblem pleiades() {
  return detail::named("pleiades", PODE_PLEIADES, 28, 3.0,
                       {3, 3, -1, -3, 2, -2, 2, 3, -3, 2, 0, 0, -4, 4, 0, 0, 0, 0, 0, 1.75, -1.5, 0, 0, 0, -1.25, 1, 0, 0},
                       {}, nullptr);
}
inline std::vector<NamedProblem> shipped_problems() { return {logistic(), rigid_body(), van_der_pol()}; }
inline NamedProblem problem_by_name(const std::string& name) {  // problems.cpp:190-195 (+ fhn, pleiades)
  if (name == "logistic") return logistic();
  if (name == "rigidbody") return rigid_body();
  if (name == "vanderpol") return van_der_pol();
  if (name == "fhn") return fitzhugh_nagumo();
  if (name == "pleiades") return pleiades();
  throw InvalidInputError("unknown problem '" + name + "'");
}
inline std::vector<double> uniform_grid(double t_end, int steps) {  // problems.cpp:212-221
  if (!(t_end > 0.0) || steps < 1) throw InvalidInputError("uniform_grid: need t_end > 0 and steps >= 1");
  std::vector<double> g(size_t(steps) + 1);
  for (int n = 0; n <= steps; ++n) g[size_t(n)] = t_end * double(n) / double(steps);
  return g;
}

}  // namespace paraode
