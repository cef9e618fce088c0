// Reference-style test cases (restated from proj/tests/test_parallel.cpp and
// proj/tests/test_ieks.cpp) compiled against the drop-in header
// include/paraode/paraode.hpp — the reference's own names and signatures —
// and run on the B200.  Without Eigen the header's minimal dense types stand
// in for Eigen::MatrixXd / VectorXd.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "paraode/paraode.hpp"

using namespace paraode;

static int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
      ++failures;                                                          \
    }                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, Type)                                        \
  do {                                                                     \
    bool thrown = false;                                                   \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const Type&) {                                                \
      thrown = true;                                                       \
    } catch (...) {                                                        \
    }                                                                      \
    if (!thrown) {                                                         \
      std::printf("FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #Type); \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

static Matrix product(const Matrix& l) {  // L L^T
  Matrix o(l.rows(), l.rows());
  for (Index i = 0; i < l.rows(); ++i)
    for (Index j = 0; j < l.rows(); ++j) {
      double acc = 0.0;
      for (Index k = 0; k < l.cols(); ++k) acc += l(i, k) * l(j, k);
      o(i, j) = acc;
    }
  return o;
}
static double max_abs_diff(const Matrix& a, const Matrix& b) {
  double m = 0.0;
  for (Index i = 0; i < a.rows(); ++i)
    for (Index j = 0; j < a.cols(); ++j) m = std::max(m, std::fabs(a(i, j) - b(i, j)));
  return m;
}
static double max_abs_diff(const Vector& a, const Vector& b) {
  double m = 0.0;
  for (Index i = 0; i < a.size(); ++i) m = std::max(m, std::fabs(a(i) - b(i)));
  return m;
}

// A random chain with square-root noise (test_parallel.cpp:40-54 style).
struct Chain {
  GaussianSqrt init;
  std::vector<TransitionModel> transitions;
  std::vector<AffineObservation> observations;
};
static Matrix rnd(std::mt19937& g, Index r, Index c, double s = 1.0) {
  std::normal_distribution<double> n(0.0, s);
  Matrix m(r, c);
  for (Index i = 0; i < r; ++i)
    for (Index j = 0; j < c; ++j) m(i, j) = n(g);
  return m;
}
static Matrix lower(std::mt19937& g, Index n) {
  Matrix m = rnd(g, n, n, 0.3);
  for (Index i = 0; i < n; ++i) {
    m(i, i) = 1.0 + std::fabs(m(i, i));
    for (Index j = i + 1; j < n; ++j) m(i, j) = 0.0;
  }
  return m;
}
static Chain random_chain(Index d, Index steps, unsigned seed) {
  std::mt19937 g(seed);
  Chain c;
  c.init.mean = Vector(d);
  for (Index i = 0; i < d; ++i) c.init.mean(i) = 0.1 * double(i);
  c.init.cov_sqrt = lower(g, d);
  for (Index k = 0; k < steps; ++k) {
    TransitionModel t;
    t.phi = rnd(g, d, d, 0.4);
    for (Index i = 0; i < d; ++i) t.phi(i, i) += 1.0;
    t.q_sqrt = lower(g, d);
    AffineObservation o;
    const Index m = (k % 4 == 2) ? 0 : d - 1;  // vacuous every fourth step
    o.h = rnd(g, m, d);
    o.offset = Vector(m);
    for (Index i = 0; i < m; ++i) o.offset(i) = 0.2 * double(i) - 0.1;
    o.r_sqrt = lower(g, m);
    c.transitions.push_back(t);
    c.observations.push_back(o);
  }
  return c;
}

static void filtering_identity_is_two_sided() {  // test_parallel.cpp:129-136
  Chain c = random_chain(4, 3, 43);
  const FilteringElement e = make_filtering_element(c.transitions[1], c.observations[1]);
  const FilteringElement l = combine_filtering(filtering_identity(4), e);
  const FilteringElement r = combine_filtering(e, filtering_identity(4));
  CHECK(max_abs_diff(l.a, e.a) <= 1e-12 && max_abs_diff(r.a, e.a) <= 1e-12);
  CHECK(max_abs_diff(product(l.c_sqrt), product(e.c_sqrt)) <= 1e-12);
  CHECK(max_abs_diff(product(r.j_sqrt), product(e.j_sqrt)) <= 1e-12);
}

static void filtering_combination_is_associative() {  // test_parallel.cpp:138-154
  Chain c = random_chain(3, 4, 44);
  FilteringElement x[3];
  for (int k = 0; k < 3; ++k) x[k] = make_filtering_element(c.transitions[k + 1], c.observations[k + 1]);
  const FilteringElement left = combine_filtering(combine_filtering(x[0], x[1]), x[2]);
  const FilteringElement right = combine_filtering(x[0], combine_filtering(x[1], x[2]));
  CHECK(max_abs_diff(left.a, right.a) <= 1e-9);
  CHECK(max_abs_diff(left.b, right.b) <= 1e-9);
  CHECK(max_abs_diff(product(left.c_sqrt), product(right.c_sqrt)) <= 1e-9);
  CHECK(max_abs_diff(left.eta, right.eta) <= 1e-9);
  CHECK(max_abs_diff(product(left.j_sqrt), product(right.j_sqrt)) <= 1e-9);
}

static void prefixes_reproduce_the_sequential_filter() {  // test_parallel.cpp:156-177
  Chain c = random_chain(3, 41, 45);
  std::vector<FilteringElement> elements;
  for (size_t k = 0; k < c.transitions.size(); ++k)
    elements.push_back(make_filtering_element(c.transitions[k], c.observations[k], k == 0 ? &c.init : nullptr));
  WorkPool pool(4);
  ScanStats stats;
  const std::vector<FilteringElement> prefixes =
      associative_scan(combine_filtering, elements, ScanDirection::kForward, stats, pool);
  const RtsResult seq = seq_rts(c.init, c.transitions, c.observations);
  for (size_t k = 0; k < prefixes.size(); ++k) {
    CHECK(max_abs_diff(prefixes[k].b, seq.filtered[k + 1].mean) <= 1e-9);
    CHECK(max_abs_diff(product(prefixes[k].c_sqrt), product(seq.filtered[k + 1].cov_sqrt)) <= 1e-9);
  }
  CHECK(stats.combine_invocations > 0 && stats.sequential_depth > 0);
}

static void reverse_scan_reproduces_the_backward_pass() {  // test_parallel.cpp:314-336
  Chain c = random_chain(3, 30, 46);
  const RtsResult seq = seq_rts(c.init, c.transitions, c.observations);
  std::vector<SmoothingElement> elements;
  for (size_t k = 0; k < c.transitions.size(); ++k)
    elements.push_back(make_smoothing_element(seq.filtered[k], c.transitions[k]));
  elements.push_back(terminal_smoothing_element(seq.filtered.back()));
  WorkPool pool;
  ScanStats stats;
  const std::vector<SmoothingElement> suffixes =
      associative_scan(combine_smoothing, elements, ScanDirection::kReverse, stats, pool);
  for (size_t k = 0; k < suffixes.size(); ++k) {
    CHECK(max_abs_diff(suffixes[k].g, seq.smoothed[k].mean) <= 1e-9);
    CHECK(max_abs_diff(product(suffixes[k].l_sqrt), product(seq.smoothed[k].cov_sqrt)) <= 1e-9);
  }
}

static void scan_smoother_matches_sequential_and_validates() {  // test_parallel.cpp:338-390
  Chain c = random_chain(4, 200, 47);
  WorkPool pool(8);
  const RtsResult par = para_rts(c.init, c.transitions, c.observations, pool);
  const RtsResult seq = seq_rts(c.init, c.transitions, c.observations);
  for (size_t k = 0; k < par.smoothed.size(); ++k) {
    CHECK(max_abs_diff(par.smoothed[k].mean, seq.smoothed[k].mean) <= 1e-9);
    CHECK(max_abs_diff(product(par.smoothed[k].cov_sqrt), product(seq.smoothed[k].cov_sqrt)) <= 1e-9);
  }
  CHECK(seq.stats.combine_invocations == 0);
  CHECK_THROWS_AS(para_rts(c.init, {}, {}, pool), DimensionError);
  std::vector<AffineObservation> short_obs(c.observations.begin(), c.observations.end() - 1);
  CHECK_THROWS_AS(para_rts(c.init, c.transitions, short_obs, pool), DimensionError);
}

static void arbitrary_scan_operators_do_not_run() {  // test_parallel.cpp:246-256 (documented difference)
  WorkPool pool(1);
  ScanStats stats;
  auto add = [](int a, int b) { return a + b; };
  CHECK_THROWS_AS(associative_scan(add, std::vector<int>{1, 2, 3}, ScanDirection::kForward, stats, pool),
                  InvalidInputError);
}

static InitialValueProblem affine_problem() {  // test_ieks.cpp:211-222 (y' = L y + c)
  InitialValueProblem ivp;
  ivp.dim = 2;
  ivp.t_end = 1.0;
  ivp.y0 = Vector(2);
  ivp.y0(0) = 0.3;
  ivp.y0(1) = -0.7;
  ivp.registered = RegisteredField{true, PODE_AFFINE, {-0.5, 1.0, -1.0, -0.2, 0.1, 0.4}};
  return ivp;
}

static void affine_converges_in_two_iterations() {  // test_ieks.cpp:224-246
  WorkPool pool;
  const SolverReport r = para_ieks(affine_problem(), IwpPrior{2, 2, 1.0}, uniform_grid(1.0, 10), IeksConfig{}, pool);
  CHECK(r.converged && r.iterations == 2);
}

static void sequential_and_parallel_agree() {  // test_ieks.cpp:248-269
  WorkPool pool;
  const NamedProblem p = van_der_pol();
  const std::vector<double> grid = uniform_grid(p.ivp.t_end, 100);
  const SolverReport par = para_ieks(p.ivp, IwpPrior{2, 2, 1.0}, grid, IeksConfig{}, pool);
  const SolverReport seq = seq_ieks(p.ivp, IwpPrior{2, 2, 1.0}, grid, IeksConfig{});
  CHECK(par.iterations == seq.iterations && par.converged == seq.converged);
  double dm = 0.0;
  for (size_t n = 0; n < grid.size(); ++n) dm = std::max(dm, max_abs_diff(par.marginals[n].mean, seq.marginals[n].mean));
  CHECK(dm <= 1e-8);
  const SolverReport eks = eks_solve(p.ivp, IwpPrior{2, 2, 1.0}, grid);
  CHECK(eks.iterations == 1 && eks.converged);
}

static void batch_matches_single_solves() {  // para_ieks_batch
  WorkPool pool;
  std::vector<InitialValueProblem> ivps;
  for (double mu : {0.5, 1.0, 2.0}) ivps.push_back(van_der_pol(mu).ivp);
  const std::vector<double> grid = uniform_grid(6.3, 150);
  const std::vector<SolverReport> batch = para_ieks_batch(ivps, IwpPrior{2, 2, 1.0}, grid, IeksConfig{}, pool);
  CHECK(batch.size() == ivps.size());
  for (size_t i = 0; i < ivps.size(); ++i) {
    const SolverReport one = para_ieks(ivps[i], IwpPrior{2, 2, 1.0}, grid, IeksConfig{}, pool);
    CHECK(batch[i].iterations == one.iterations && batch[i].converged == one.converged);
    double dm = 0.0;
    for (size_t n = 0; n < grid.size(); ++n)
      dm = std::max(dm, max_abs_diff(batch[i].marginals[n].mean, one.marginals[n].mean));
    CHECK(dm <= 1e-9);
    CHECK(std::fabs(batch[i].sigma_hat - one.sigma_hat) <= 1e-7 * std::fabs(one.sigma_hat));
  }
}

static void logistic_matches_the_closed_form() {  // test_ieks.cpp:271-282 / acceptance.cpp:167-179
  WorkPool pool;
  const NamedProblem p = logistic();
  const std::vector<double> grid = uniform_grid(p.ivp.t_end, 30);
  const SolverReport r = para_ieks(p.ivp, IwpPrior{2, 1, 1.0}, grid, IeksConfig{}, pool);
  double se = 0.0;
  for (size_t n = 0; n < grid.size(); ++n) {
    const double t = grid[n], y = 1.0 / (1.0 + 99.0 * std::exp(-t));
    se += (r.solution_means[n](0) - y) * (r.solution_means[n](0) - y);
  }
  const double rmse = std::sqrt(se / double(grid.size()));
  CHECK(r.converged && rmse <= 2.1e-6);
}

static void invariant_under_sigma_and_budget() {  // test_ieks.cpp:284-299, 382-401
  WorkPool pool;
  const NamedProblem p = logistic();
  const std::vector<double> grid = uniform_grid(10.0, 20);
  const SolverReport a = para_ieks(p.ivp, IwpPrior{2, 1, 1.0}, grid, IeksConfig{}, pool);
  const SolverReport b = para_ieks(p.ivp, IwpPrior{2, 1, 7.0}, grid, IeksConfig{}, pool);
  CHECK(a.iterations == b.iterations);
  CHECK(std::fabs(a.sigma_hat / b.sigma_hat - 1.0) <= 1e-8);
  double dm = 0.0;
  for (size_t n = 0; n < grid.size(); ++n) dm = std::max(dm, max_abs_diff(a.marginals[n].mean, b.marginals[n].mean));
  CHECK(dm <= 1e-10);
  IeksConfig one;
  one.max_iterations = 1;
  const SolverReport r = para_ieks(van_der_pol().ivp, IwpPrior{2, 2, 1.0}, uniform_grid(6.3, 40), one, pool);
  CHECK(!r.converged && r.iterations == 1 && r.objective_trace.size() == 1);
  IeksConfig zero;
  zero.max_iterations = 0;
  CHECK_THROWS_AS(para_ieks(van_der_pol().ivp, IwpPrior{2, 2, 1.0}, uniform_grid(6.3, 40), zero, pool),
                  InvalidInputError);
  CHECK_THROWS_AS(para_ieks(van_der_pol().ivp, IwpPrior{2, 3, 1.0}, uniform_grid(6.3, 40), IeksConfig{}, pool),
                  DimensionError);
}

static void host_only_callbacks_are_rejected() {
  InitialValueProblem ivp;
  ivp.dim = 1;
  ivp.t_end = 1.0;
  ivp.y0 = Vector(1);
  ivp.field = [](const Vector& y, double) { return y; };  // no registered device field
  WorkPool pool;
  CHECK_THROWS_AS(para_ieks(ivp, IwpPrior{1, 1, 1.0}, uniform_grid(1.0, 8), IeksConfig{}, pool), InvalidInputError);
}

static void linearization_error_carries_the_time() {  // test_statespace.cpp:123-139 (the pole field)
  InitialValueProblem ivp;
  ivp.dim = 1;
  ivp.t_end = 1.0;
  ivp.y0 = Vector(1);
  ivp.registered = RegisteredField{true, PODE_POLE, {0.75}};
  WorkPool pool;
  try {
    para_ieks(ivp, IwpPrior{2, 1, 1.0}, uniform_grid(1.0, 64), IeksConfig{}, pool);
    CHECK(false);
  } catch (const LinearizationError& e) {
    CHECK(e.time() == 0.75);
  }
}

int main() {
  filtering_identity_is_two_sided();
  filtering_combination_is_associative();
  prefixes_reproduce_the_sequential_filter();
  reverse_scan_reproduces_the_backward_pass();
  scan_smoother_matches_sequential_and_validates();
  arbitrary_scan_operators_do_not_run();
  affine_converges_in_two_iterations();
  sequential_and_parallel_agree();
  batch_matches_single_solves();
  logistic_matches_the_closed_form();
  invariant_under_sigma_and_budget();
  host_only_callbacks_are_rejected();
  linearization_error_carries_the_time();
  if (failures) {
    std::printf("%d failures\n", failures);
    return 1;
  }
  std::printf("PASS (drop-in header, 12 reference-style cases + the batched solve)\n");
  return 0;
}
