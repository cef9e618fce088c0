// paraode_b200.hpp — header-only C++ mirror of the reference's solver API
// (proj/include/paraode/{parallel,ieks,errors}.hpp) on top of the C ABI
// (include/paraode_b200.h).  Same function names, argument meaning and
// exception types; every call runs on the B200, there is no CPU fallback.
//
// The functions are templates over the caller's dense types, so they accept
// the reference's Eigen::MatrixXd / Eigen::VectorXd directly (any Matrix
// with rows(), cols(), operator()(i, j) and a (rows, cols) constructor, and
// any Vector with size(), operator()(i) / operator[](i) and a (n)
// constructor).  See INTEGRATION.md.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../paraode_b200.h"

namespace paraode {
namespace b200 {

// ------------------------------------------------------------- errors ---
// proj/include/paraode/errors.hpp:10-60
class SolverError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class InvalidInputError : public SolverError {
 public:
  using SolverError::SolverError;
};
class DimensionError : public SolverError {
 public:
  using SolverError::SolverError;
};
class SingularFactorError : public SolverError {
 public:
  using SolverError::SolverError;
};
class LinearizationError : public SolverError {
 public:
  LinearizationError(const std::string& w, double t, std::size_t i) : SolverError(w), time_(t), index_(i) {}
  double time() const { return time_; }
  std::size_t index() const { return index_; }

 private:
  double time_;
  std::size_t index_;
};
class ScanError : public SolverError {
 public:
  using SolverError::SolverError;
};
// No usable B200 (the C ABI's PODE_ERR_CUDA / PODE_ERR_UNSUPPORTED).
class DeviceError : public SolverError {
 public:
  using SolverError::SolverError;
};

inline void check(int rc, const pode_status& st) {
  if (rc == PODE_OK) return;
  const std::string msg(st.msg);
  switch (rc) {
    case PODE_ERR_INVALID_INPUT: throw InvalidInputError(msg);
    case PODE_ERR_DIMENSION: throw DimensionError(msg);
    case PODE_ERR_SINGULAR_FACTOR: throw SingularFactorError(msg);
    case PODE_ERR_LINEARIZATION:
      throw LinearizationError(msg, st.time, static_cast<std::size_t>(st.index < 0 ? 0 : st.index));
    case PODE_ERR_SCAN: throw ScanError(msg);
    default: throw DeviceError(msg);
  }
}

// ------------------------------------------------------------- device ---
// Takes the place of the reference's WorkPool (work_pool.hpp:21-64): the
// execution resource a solve runs on.  Not reentrant, like WorkPool.
class Device {
 public:
  explicit Device(int index = 0) {
    pode_status st{};
    check(pode_context_create(index, &ctx_, &st), st);
  }
  ~Device() { pode_context_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  pode_context* handle() const { return ctx_; }

 private:
  pode_context* ctx_ = nullptr;
};

namespace detail {
template <class M>
void put(const M& m, double* dst, int rows, int cols) {
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) dst[i * cols + j] = (i < int(m.rows()) && j < int(m.cols())) ? m(i, j) : 0.0;
}
template <class V>
void putv(const V& v, double* dst, int n) {
  for (int i = 0; i < n; ++i) dst[i] = i < int(v.size()) ? v[i] : 0.0;
}
template <class M>
M get(const double* src, int rows, int cols) {
  M m(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) m(i, j) = src[i * cols + j];
  return m;
}
template <class V>
V getv(const double* src, int n) {
  V v(n);
  for (int i = 0; i < n; ++i) v[i] = src[i];
  return v;
}
}  // namespace detail

// -------------------------------------------------------------- types ---
template <class Matrix, class Vector>
struct GaussianSqrt {  // statespace.hpp:13-16
  Vector mean;
  Matrix cov_sqrt;
};

struct ScanStats {  // sequential.hpp:42-50
  std::size_t combine_invocations = 0;
  std::size_t sequential_depth = 0;
};

template <class Matrix, class Vector>
struct RtsResult {  // sequential.hpp:52-56
  std::vector<GaussianSqrt<Matrix, Vector>> filtered, smoothed;
  ScanStats stats;
};

// para_rts (parallel.hpp:155-156).  Transition needs .phi and .q_sqrt;
// Observation needs .h, .offset and .r_sqrt (statespace.hpp:36-48).
template <class Matrix, class Vector, class Gaussian, class Transition, class Observation>
RtsResult<Matrix, Vector> para_rts(const Gaussian& init, const std::vector<Transition>& transitions,
                                   const std::vector<Observation>& observations, Device& dev) {
  if (transitions.empty() || transitions.size() != observations.size())
    throw DimensionError("para_rts: need N >= 1 aligned transitions and observations");
  const int D = int(init.mean.size());
  const int64_t N = int64_t(transitions.size());
  int M = 0;
  for (const auto& o : observations) M = std::max(M, int(o.h.rows()));
  const int Mm = std::max(M, 1);
  std::vector<double> im(D), ic(size_t(D) * D), phi(size_t(N) * D * D), q(size_t(N) * D * D);
  std::vector<int32_t> rows(N);
  std::vector<double> h(size_t(N) * Mm * D), off(size_t(N) * Mm), r(size_t(N) * Mm * Mm);
  detail::putv(init.mean, im.data(), D);
  detail::put(init.cov_sqrt, ic.data(), D, D);
  for (int64_t n = 0; n < N; ++n) {
    detail::put(transitions[n].phi, phi.data() + n * D * D, D, D);
    detail::put(transitions[n].q_sqrt, q.data() + n * D * D, D, D);
    const auto& o = observations[n];
    const int m = int(o.h.rows());
    if (int(o.h.cols()) != D || int(o.offset.size()) != m || int(o.r_sqrt.rows()) != m)
      throw DimensionError("para_rts: observation dimensions disagree with the state");
    if (int(o.r_sqrt.cols()) > m)
      throw DimensionError("para_rts: r_sqrt with more columns than rows is not supported");
    rows[n] = m;
    detail::put(o.h, h.data() + n * Mm * D, Mm, D);
    detail::putv(o.offset, off.data() + n * Mm, Mm);
    detail::put(o.r_sqrt, r.data() + n * Mm * Mm, Mm, Mm);
  }
  pode_chain ch{D, M, N, im.data(), ic.data(), phi.data(), q.data(), 0, 0, rows.data(), h.data(), off.data(),
                r.data(), PODE_HOST};
  const int64_t n1 = N + 1;
  std::vector<double> fm(size_t(n1) * D), fc(size_t(n1) * D * D), sm(size_t(n1) * D), sc(size_t(n1) * D * D);
  pode_rts_out out{fm.data(), fc.data(), sm.data(), sc.data()};
  pode_scan_stats stats{};
  pode_status st{};
  check(pode_rts(dev.handle(), &ch, out, &stats, &st), st);
  RtsResult<Matrix, Vector> res;
  res.filtered.resize(size_t(n1));
  res.smoothed.resize(size_t(n1));
  for (int64_t n = 0; n < n1; ++n) {
    res.filtered[n] = {detail::getv<Vector>(fm.data() + n * D, D), detail::get<Matrix>(fc.data() + n * D * D, D, D)};
    res.smoothed[n] = {detail::getv<Vector>(sm.data() + n * D, D), detail::get<Matrix>(sc.data() + n * D * D, D, D)};
  }
  res.stats.combine_invocations = std::size_t(stats.combine_invocations);
  res.stats.sequential_depth = std::size_t(stats.sequential_depth);
  return res;
}

// --------------------------------------------------------------- ieks ---
struct IwpPrior {  // prior.hpp:12-18
  int nu = 1;
  int dim = 1;
  double sigma = 1.0;
  int state_dim() const { return dim * (nu + 1); }
};

enum class Linearization { kEk1, kEk0 };

struct IeksConfig {  // ieks.hpp:32-38
  int max_iterations = 100;
  double traj_rtol = 1e-13;
  double obj_atol = 1e-9;
  double obj_rtol = 1e-6;
  Linearization linearization = Linearization::kEk1;
};

// A registered device vector field (replaces InitialValueProblem's host
// callbacks, statespace.hpp:24-31).
struct Problem {
  pode_problem_kind kind = PODE_LOGISTIC;
  int dim = 1;
  double t_end = 10.0;
  std::vector<double> y0{0.01};
  std::vector<double> params;
};

template <class Matrix, class Vector>
struct SolverReport {  // ieks.hpp:77-87
  std::vector<double> times;
  std::vector<GaussianSqrt<Matrix, Vector>> marginals;
  std::vector<Vector> solution_means;
  std::vector<Matrix> solution_covs;
  double sigma_hat = 0.0;
  int iterations = 0;
  std::vector<double> objective_trace;
  bool converged = false;
  ScanStats scan_stats;
};

namespace detail {
template <class Matrix, class Vector>
SolverReport<Matrix, Vector> report(const std::vector<double>& grid, int D, int d, const std::vector<double>& means,
                                    const std::vector<double>& cov, const std::vector<double>& sm,
                                    const std::vector<double>& sc, const std::vector<double>& trace,
                                    const pode_ieks_report& rep);
}  // namespace detail

// para_ieks (ieks.hpp:95-96).
template <class Matrix, class Vector>
SolverReport<Matrix, Vector> para_ieks(const Problem& problem, const IwpPrior& prior,
                                       const std::vector<double>& grid, const IeksConfig& config, Device& dev) {
  const int D = prior.state_dim(), d = prior.dim;
  const int64_t n1 = int64_t(grid.size());
  pode_problem p{int32_t(problem.kind), problem.dim, problem.t_end, problem.y0.data(),
                 problem.params.empty() ? nullptr : problem.params.data(), int32_t(problem.params.size())};
  pode_prior pr{prior.nu, prior.dim, prior.sigma};
  pode_ieks_config cfg{config.max_iterations, config.traj_rtol, config.obj_atol, config.obj_rtol,
                       config.linearization == Linearization::kEk0 ? 1 : 0};
  std::vector<double> means(size_t(n1) * D), cov(size_t(n1) * D * D), sm(size_t(n1) * d), sc(size_t(n1) * d * d);
  std::vector<double> trace(size_t(std::max(config.max_iterations, 1)));
  pode_ieks_report rep{means.data(), cov.data(), sm.data(), sc.data(), trace.data(), int32_t(trace.size()),
                       PODE_HOST, 0, 0, 0.0, {0, 0}};
  pode_status st{};
  check(pode_ieks(dev.handle(), &p, &pr, grid.data(), n1, &cfg, &rep, &st), st);
  return detail::report<Matrix, Vector>(grid, D, d, means, cov, sm, sc, trace, rep);
}

namespace detail {
template <class Matrix, class Vector>
SolverReport<Matrix, Vector> report(const std::vector<double>& grid, int D, int d, const std::vector<double>& means,
                                    const std::vector<double>& cov, const std::vector<double>& sm,
                                    const std::vector<double>& sc, const std::vector<double>& trace,
                                    const pode_ieks_report& rep) {
  const int64_t n1 = int64_t(grid.size());
  SolverReport<Matrix, Vector> out;
  out.times = grid;
  out.marginals.resize(size_t(n1));
  out.solution_means.resize(size_t(n1));
  out.solution_covs.resize(size_t(n1));
  for (int64_t n = 0; n < n1; ++n) {
    out.marginals[n] = {detail::getv<Vector>(means.data() + n * D, D),
                        detail::get<Matrix>(cov.data() + n * D * D, D, D)};
    out.solution_means[n] = detail::getv<Vector>(sm.data() + n * d, d);
    out.solution_covs[n] = detail::get<Matrix>(sc.data() + n * d * d, d, d);
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

// eks_solve (ieks.hpp:103-105): one pass linearised at the predicted means.
template <class Matrix, class Vector>
SolverReport<Matrix, Vector> eks_solve(const Problem& problem, const IwpPrior& prior, const std::vector<double>& grid,
                                       Linearization linearization, Device& dev) {
  const int D = prior.state_dim(), d = prior.dim;
  const int64_t n1 = int64_t(grid.size());
  pode_problem p{int32_t(problem.kind), problem.dim, problem.t_end, problem.y0.data(),
                 problem.params.empty() ? nullptr : problem.params.data(), int32_t(problem.params.size())};
  pode_prior pr{prior.nu, prior.dim, prior.sigma};
  std::vector<double> means(size_t(n1) * D), cov(size_t(n1) * D * D), sm(size_t(n1) * d), sc(size_t(n1) * d * d);
  std::vector<double> trace(1);
  pode_ieks_report rep{means.data(), cov.data(), sm.data(), sc.data(), trace.data(), 1, PODE_HOST, 0, 0, 0.0, {0, 0}};
  pode_status st{};
  check(pode_eks(dev.handle(), &p, &pr, grid.data(), n1, linearization == Linearization::kEk0 ? 1 : 0, &rep, &st),
        st);
  return detail::report<Matrix, Vector>(grid, D, d, means, cov, sm, sc, trace, rep);
}

// para_ieks over time-axis shard `rank` of `ranks` (one process per GPU;
// DESIGN.md §6).  `allgather(send, count, recv)` gathers `count` doubles of
// every rank into recv[rank * count + i] (MPI_Allgather, NCCL, ...) and
// returns 0 on success.  The report holds this shard's nodes (times,
// marginals, solution moments from pode_shard_range's first node on); the
// scalars are those of the whole solve.
template <class Matrix, class Vector>
SolverReport<Matrix, Vector> para_ieks_sharded(const Problem& problem, const IwpPrior& prior,
                                               const std::vector<double>& grid, const IeksConfig& config,
                                               int rank, int ranks, pode_allgather_fn allgather, void* user,
                                               Device& dev) {
  const int D = prior.state_dim(), d = prior.dim;
  const int64_t n1 = int64_t(grid.size());
  int64_t first = 0, cnt = 0;
  pode_shard_range(n1, rank, ranks, &first, &cnt);
  pode_problem p{int32_t(problem.kind), problem.dim, problem.t_end, problem.y0.data(),
                 problem.params.empty() ? nullptr : problem.params.data(), int32_t(problem.params.size())};
  pode_prior pr{prior.nu, prior.dim, prior.sigma};
  pode_ieks_config cfg{config.max_iterations, config.traj_rtol, config.obj_atol, config.obj_rtol,
                       config.linearization == Linearization::kEk0 ? 1 : 0};
  std::vector<double> means(size_t(cnt) * D), cov(size_t(cnt) * D * D), sm(size_t(cnt) * d), sc(size_t(cnt) * d * d);
  std::vector<double> trace(size_t(std::max(config.max_iterations, 1)));
  pode_ieks_report rep{means.data(), cov.data(), sm.data(), sc.data(), trace.data(), int32_t(trace.size()),
                       PODE_HOST, 0, 0, 0.0, {0, 0}};
  pode_shard_comm comm{rank, ranks, allgather, user};
  pode_status st{};
  check(pode_ieks_sharded(dev.handle(), &p, &pr, grid.data(), n1, &cfg, &comm, &rep, &st), st);
  SolverReport<Matrix, Vector> out;
  out.times.assign(grid.begin() + first, grid.begin() + first + cnt);
  out.marginals.resize(size_t(cnt));
  out.solution_means.resize(size_t(cnt));
  out.solution_covs.resize(size_t(cnt));
  for (int64_t n = 0; n < cnt; ++n) {
    out.marginals[n] = {detail::getv<Vector>(means.data() + n * D, D),
                        detail::get<Matrix>(cov.data() + n * D * D, D, D)};
    out.solution_means[n] = detail::getv<Vector>(sm.data() + n * d, d);
    out.solution_covs[n] = detail::get<Matrix>(sc.data() + n * d * d, d, d);
  }
  out.sigma_hat = rep.sigma_hat;
  out.iterations = rep.iterations;
  out.objective_trace.assign(trace.begin(), trace.begin() + rep.iterations);
  out.converged = rep.converged != 0;
  out.scan_stats.combine_invocations = std::size_t(rep.scan_stats.combine_invocations);
  out.scan_stats.sequential_depth = std::size_t(rep.scan_stats.sequential_depth);
  return out;
}

}  // namespace b200
}  // namespace paraode
