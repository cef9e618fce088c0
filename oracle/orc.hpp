// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain C++ restatement of the reference CPU algorithm (paraode, C++20 +
// Eigen; /root/reference/proj) for the ParaIEKS hot path.  The reference
// itself cannot be compiled in this image (Eigen 3.3+ is absent, its vendored
// CLI11/json/doctest are gitignored), so this file restates
// it function by function, each citing the reference file:line it follows.
//
// Pinning: the restatement is checked against every known-answer test the
// reference's own test-suite holds for this path (tests/test_oracle_*.py,
// tests/golden/), reproducing the reference's std::mt19937 fixtures
// bit-for-bit (same libstdc++ distributions, same draw order), and against an
// independent numpy dense-covariance restatement of proj/tests/oracles.cpp.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this code — and only as the checker or the
// CPU baseline, never as the product path.
// ============================================================================
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- errors ---
// proj/include/paraode/errors.hpp:10-60
struct SolverError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidInputError : SolverError {
  using SolverError::SolverError;
};
struct DimensionError : SolverError {
  using SolverError::SolverError;
};
struct SingularFactorError : SolverError {
  using SolverError::SolverError;
};
struct LinearizationError : SolverError {
  LinearizationError(const std::string& w, double t, std::size_t i)
      : SolverError(w), time(t), index(i) {}
  double time;
  std::size_t index;
};
struct ScanError : SolverError {
  using SolverError::SolverError;
};

// ---------------------------------------------------------- dense types ---
// Row-major dynamic dense matrix (the reference uses Eigen::MatrixXd,
// proj/include/paraode/linalg.hpp:9-10; layout is irrelevant to the
// arithmetic restated here).
struct Mat {
  int r = 0, c = 0;
  std::vector<double> v;
  Mat() = default;
  Mat(int rows, int cols) : r(rows), c(cols), v(static_cast<std::size_t>(rows) * cols, 0.0) {}
  double& operator()(int i, int j) { return v[static_cast<std::size_t>(i) * c + j]; }
  double operator()(int i, int j) const { return v[static_cast<std::size_t>(i) * c + j]; }
  static Mat zero(int rows, int cols) { return Mat(rows, cols); }
  static Mat identity(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};
using Vec = std::vector<double>;

Mat operator*(const Mat& a, const Mat& b);
Vec operator*(const Mat& a, const Vec& x);
Mat operator+(const Mat& a, const Mat& b);
Mat operator-(const Mat& a, const Mat& b);
Mat operator*(double s, const Mat& a);
Vec operator+(const Vec& a, const Vec& b);
Vec operator-(const Vec& a, const Vec& b);
Vec operator*(double s, const Vec& a);
Mat transpose(const Mat& a);
Mat block(const Mat& a, int r0, int c0, int rows, int cols);
void set_block(Mat& a, int r0, int c0, const Mat& b);
Mat diag_mul_left(const Vec& d, const Mat& a);   // diag(d) * a
Mat diag_mul_right(const Mat& a, const Vec& d);  // a * diag(d)
Vec cwise(const Vec& a, const Vec& b);
bool all_finite(const Mat& a);
bool all_finite(const Vec& a);
Mat dense_cov(const Mat& s);  // s s^T

// --------------------------------------------------------------- linalg ---
// proj/src/linalg.cpp:9-71
Mat tria(const Mat& m);
Mat sqrt_sum(const Mat& a, const Mat& b);
double whitened_sq_norm(const Vec& v, const Mat& q_sqrt);
bool is_lower_triangular(const Mat& m);
void require_nonsingular_triangular(const Mat& t, const char* context);
// Solves L X = B (L lower, forward substitution) and U X = B (U upper).
Mat solve_lower(const Mat& l, const Mat& b);
Vec solve_lower(const Mat& l, const Vec& b);
Mat solve_upper(const Mat& u, const Mat& b);

// ------------------------------------------------------------------ jet ---
// proj/include/paraode/jet.hpp:17-102, extended with division and sqrt
// (needed by the Pleiades field, which the reference does not ship).
struct Jet {
  std::vector<double> c;
  Jet() = default;
  explicit Jet(int order) : c(static_cast<std::size_t>(order) + 1, 0.0) {}
  static Jet constant(double v, int order) {
    Jet j(order);
    j.c[0] = v;
    return j;
  }
  static Jet variable(double v, int order) {
    Jet j(order);
    j.c[0] = v;
    if (order >= 1) j.c[1] = 1.0;
    return j;
  }
  int order() const { return static_cast<int>(c.size()) - 1; }
};
Jet operator+(const Jet& a, const Jet& b);
Jet operator-(const Jet& a, const Jet& b);
Jet operator*(const Jet& a, const Jet& b);
Jet operator/(const Jet& a, const Jet& b);
Jet operator-(const Jet& a);
Jet operator+(const Jet& a, double s);
Jet operator-(const Jet& a, double s);
Jet operator*(const Jet& a, double s);
Jet operator+(double s, const Jet& a);
Jet operator-(double s, const Jet& a);
Jet operator*(double s, const Jet& a);
Jet jet_sqrt(const Jet& a);

// ---------------------------------------------------------- state space ---
// proj/include/paraode/statespace.hpp:13-78
struct GaussianSqrt {
  Vec mean;
  Mat cov_sqrt;
};
struct AffineObservation {
  Mat h;
  Vec offset;
  Mat r_sqrt;
};
struct TransitionModel {
  Mat phi;
  Mat q_sqrt;
  double step = 0.0;
};

// Problem registry: the reference's InitialValueProblem carries host
// std::function callbacks (statespace.hpp:24-31); here problems are named
// kinds with parameters, the same registry the device side uses.
enum ProblemKind : int {
  kLogistic = 1,
  kRigidBody = 2,
  kVanDerPol = 3,
  kFitzHughNagumo = 4,
  kPleiades = 5,
  kAffine = 6,
  kPole = 7,  // test kind: y' = 1 / (t - a), the reference's non-finite-field case
};
struct Problem {
  int kind = 0;
  int dim = 0;
  double t_end = 0.0;
  Vec y0;
  Vec params;  // affine: L (dim*dim row-major) then c (dim); vdp: mu; fhn: a, b, c
};
Vec field(const Problem& p, const Vec& y, double t);
Mat jacobian(const Problem& p, const Vec& y, double t);
std::vector<Jet> field_series(const Problem& p, const std::vector<Jet>& y, const Jet& t);
Problem make_problem(int kind);  // shipped defaults (problems.cpp:116-179 + FHN/Pleiades)
Problem make_affine(const Mat& l, const Vec& c, const Vec& y0, double t_end);

Mat projection_matrix(int dim, int nu, int deriv);
AffineObservation linearize_ek1(const Problem& p, const Vec& eta, double t);
AffineObservation linearize_ek0(const Problem& p, const Vec& eta, double t);
enum class Linearization { kEk1 = 0, kEk0 = 1 };
AffineObservation linearize(const Problem& p, const Vec& eta, double t, Linearization kind);

// ---------------------------------------------------------------- prior ---
// proj/include/paraode/prior.hpp:12-50
struct IwpPrior {
  int nu = 1;
  int dim = 1;
  double sigma = 1.0;
  int state_dim() const { return dim * (nu + 1); }
};
TransitionModel iwp_transition(const IwpPrior& prior, double h);
struct Preconditioner {
  Vec scale, scale_inv;
};
Preconditioner preconditioner(const IwpPrior& prior, double h);
Mat preconditioned_phi(const IwpPrior& prior);
Mat preconditioned_q_sqrt(const IwpPrior& prior);
GaussianSqrt taylor_init(const Problem& p, int nu);

// ----------------------------------------------------------- sequential ---
// proj/include/paraode/sequential.hpp:11-60
GaussianSqrt kf_predict(const GaussianSqrt& s, const TransitionModel& t);
GaussianSqrt kf_update(const GaussianSqrt& pred, const AffineObservation& obs);
std::vector<GaussianSqrt> kf_forward(const GaussianSqrt& init,
                                     const std::vector<TransitionModel>& tr,
                                     const std::vector<AffineObservation>& obs);
std::vector<GaussianSqrt> rts_smooth_pass(const std::vector<GaussianSqrt>& filtered,
                                          const std::vector<TransitionModel>& tr);
struct ScanStats {
  std::size_t combine_invocations = 0;
  std::size_t sequential_depth = 0;
  void merge_max(const ScanStats& o) {
    if (o.combine_invocations > combine_invocations) combine_invocations = o.combine_invocations;
    if (o.sequential_depth > sequential_depth) sequential_depth = o.sequential_depth;
  }
};
struct RtsResult {
  std::vector<GaussianSqrt> filtered, smoothed;
  ScanStats stats;
};
RtsResult seq_rts(const GaussianSqrt& init, const std::vector<TransitionModel>& tr,
                  const std::vector<AffineObservation>& obs);

// ------------------------------------------------------------- parallel ---
// proj/include/paraode/parallel.hpp:20-156
struct FilteringElement {
  Mat a;
  Vec b;
  Mat c_sqrt;
  Vec eta;
  Mat j_sqrt;
};
struct SmoothingElement {
  Mat e;
  Vec g;
  Mat l_sqrt;
};
FilteringElement make_filtering_element(const TransitionModel& t, const AffineObservation& o,
                                        const GaussianSqrt* init = nullptr);
FilteringElement combine_filtering(const FilteringElement& lhs, const FilteringElement& rhs);
FilteringElement filtering_identity(int d);
SmoothingElement make_smoothing_element(const GaussianSqrt& filtered, const TransitionModel& t);
SmoothingElement terminal_smoothing_element(const GaussianSqrt& filtered);
SmoothingElement combine_smoothing(const SmoothingElement& lhs, const SmoothingElement& rhs);
SmoothingElement smoothing_identity(int d);

// Restatement of proj/src/work_pool.cpp:7-85 (fixed-width std::thread pool,
// dynamic index assignment, caller participates, first error rethrown).
class WorkPool {
 public:
  explicit WorkPool(unsigned width = 0);
  ~WorkPool();
  WorkPool(const WorkPool&) = delete;
  WorkPool& operator=(const WorkPool&) = delete;
  unsigned width() const { return width_; }
  void parallel_for(std::size_t count, const std::function<void(std::size_t)>& body);

 private:
  struct Impl;
  Impl* impl_ = nullptr;
  unsigned width_ = 1;
};
void parallel_map(WorkPool* pool, std::size_t count, const std::function<void(std::size_t)>& body);

// proj/include/paraode/parallel.hpp:86-127 — the exact reduce / recurse /
// fix-up tree (combination tree is a function of the element count alone).
template <typename Elem, typename Op>
void scan_in_place(std::vector<Elem>& x, const Op& op, std::size_t block, std::size_t total,
                   ScanStats& stats, WorkPool* pool) {
  const std::size_t n = x.size();
  if (n < 2) return;
  auto combine = [&](const Elem& lhs, const Elem& rhs, std::size_t lo, std::size_t hi) -> Elem {
    try {
      return op(lhs, rhs);
    } catch (const std::exception& e) {
      throw ScanError("associative_scan: combine failed on elements [" + std::to_string(lo) +
                      ", " + std::to_string(hi) + "]: " + e.what());
    }
  };
  const std::size_t pairs = n / 2;
  std::vector<Elem> reduced(pairs);
  parallel_map(pool, pairs, [&](std::size_t i) {
    const std::size_t lo = 2 * i * block;
    const std::size_t hi = std::min((2 * i + 2) * block, total) - 1;
    reduced[i] = combine(x[2 * i], x[2 * i + 1], lo, hi);
  });
  stats.combine_invocations += pairs;
  stats.sequential_depth += 1;
  scan_in_place(reduced, op, 2 * block, total, stats, pool);
  const std::size_t fixups = (n + 1) / 2 - 1;
  parallel_map(pool, n, [&](std::size_t p) {
    if (p == 0) return;
    if (p % 2 == 1) {
      x[p] = reduced[p / 2];
    } else {
      const std::size_t hi = std::min((p + 1) * block, total) - 1;
      x[p] = combine(reduced[p / 2 - 1], x[p], 0, hi);
    }
  });
  stats.combine_invocations += fixups;
  if (fixups > 0) stats.sequential_depth += 1;
}

enum class ScanDirection { kForward, kReverse };

// proj/include/paraode/parallel.hpp:136-149
template <typename Elem, typename Op>
std::vector<Elem> associative_scan(const Op& op, std::vector<Elem> elems, ScanDirection dir,
                                   ScanStats& stats, WorkPool* pool) {
  if (elems.size() < 2) return elems;
  if (dir == ScanDirection::kForward) {
    scan_in_place(elems, op, 1, elems.size(), stats, pool);
    return elems;
  }
  std::reverse(elems.begin(), elems.end());
  auto flipped = [&op](const Elem& lhs, const Elem& rhs) { return op(rhs, lhs); };
  scan_in_place(elems, flipped, 1, elems.size(), stats, pool);
  std::reverse(elems.begin(), elems.end());
  return elems;
}

RtsResult para_rts(const GaussianSqrt& init, const std::vector<TransitionModel>& tr,
                   const std::vector<AffineObservation>& obs, WorkPool* pool);

// ----------------------------------------------------------------- ieks ---
// proj/include/paraode/ieks.hpp:16-105
struct DiscretizedPrior {
  IwpPrior prior;
  std::vector<double> times;
  std::vector<Vec> node_scale, node_scale_inv;
  std::vector<TransitionModel> transitions;
  Mat q_unit_sqrt;
  std::size_t steps() const { return transitions.size(); }
};
DiscretizedPrior discretize(const IwpPrior& prior, const std::vector<double>& grid);
struct IeksConfig {
  int max_iterations = 100;
  double traj_rtol = 1e-13;
  double obj_atol = 1e-9;
  double obj_rtol = 1e-6;
  Linearization linearization = Linearization::kEk1;
};
double objective_value(const std::vector<Vec>& states, const std::vector<TransitionModel>& tr);
bool stopping_check(const std::vector<Vec>& prev, const std::vector<Vec>& next, double prev_obj,
                    double new_obj, const IeksConfig& cfg);
struct InnovationStats {
  double whitened_sq_sum = 0.0;
  std::size_t count = 0;
};
InnovationStats innovation_stats(const GaussianSqrt& init, const std::vector<TransitionModel>& tr,
                                 const std::vector<AffineObservation>& obs,
                                 const std::vector<GaussianSqrt>& filtered, WorkPool* pool);
double calibrate_sigma(const InnovationStats& s);
struct SolverReport {
  std::vector<double> times;
  std::vector<GaussianSqrt> marginals;
  std::vector<Vec> solution_means;
  std::vector<Mat> solution_covs;
  double sigma_hat = 0.0;
  int iterations = 0;
  std::vector<double> objective_trace;
  bool converged = false;
  ScanStats scan_stats;
};
// pool == nullptr → seq_ieks (ieks.cpp:219-222); else para_ieks (:214-217).
SolverReport ieks_drive(const Problem& p, const IwpPrior& prior, const std::vector<double>& grid,
                        const IeksConfig& cfg, WorkPool* pool);
SolverReport eks_solve(const Problem& p, const IwpPrior& prior, const std::vector<double>& grid,
                       Linearization lin);

std::vector<double> uniform_grid(double t_end, int steps);

}  // namespace orc
