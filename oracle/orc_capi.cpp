// ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp).
// Flat C ABI over the restatement so the Python tests (ctypes) and bench.py's
// CPU baseline can drive it with the same row-major buffers the product ABI
// (include/paraode_b200.h) uses.  Also exports the reference's test-fixture
// generators (proj/tests/oracles.cpp:168-229) on std::mt19937, so fixtures are
// bit-identical to the reference's own tests when built with libstdc++.
#include <chrono>
#include <cstring>
#include <random>

#include "orc.hpp"

using namespace orc;

namespace {

enum { kOk = 0, kInvalid = 1, kDim = 2, kSingular = 3, kLinearization = 4, kScan = 5, kOther = 9 };

struct Status {
  int32_t code;
  int32_t iteration;
  int64_t index;
  double time;
  char msg[256];
};

int fail(Status* st, int code, const char* what) {
  if (st) {
    st->code = code;
    std::strncpy(st->msg, what, sizeof(st->msg) - 1);
    st->msg[sizeof(st->msg) - 1] = 0;
  }
  return code;
}

template <typename F>
int guarded(Status* st, F&& f) {
  if (st) std::memset(st, 0, sizeof(Status));
  try {
    f();
    return kOk;
  } catch (const LinearizationError& e) {
    if (st) {
      st->time = e.time;
      st->index = static_cast<int64_t>(e.index);
    }
    return fail(st, kLinearization, e.what());
  } catch (const ScanError& e) {
    return fail(st, kScan, e.what());
  } catch (const SingularFactorError& e) {
    return fail(st, kSingular, e.what());
  } catch (const DimensionError& e) {
    return fail(st, kDim, e.what());
  } catch (const InvalidInputError& e) {
    return fail(st, kInvalid, e.what());
  } catch (const std::exception& e) {
    return fail(st, kOther, e.what());
  }
}

Mat load(const double* p, int r, int c) {
  Mat m(r, c);
  if (r > 0 && c > 0) std::memcpy(m.v.data(), p, sizeof(double) * r * c);
  return m;
}
Vec loadv(const double* p, int n) { return Vec(p, p + n); }
void store(double* p, const Mat& m) {
  if (p && !m.v.empty()) std::memcpy(p, m.v.data(), sizeof(double) * m.v.size());
}
void storev(double* p, const Vec& v) {
  if (p && !v.empty()) std::memcpy(p, v.data(), sizeof(double) * v.size());
}

}  // namespace

extern "C" {

// Element arrays: separate row-major buffers per field, element i at
// offset i*D*D (matrices) or i*D (vectors) — same as pode_filtering_elements.
struct OrcFE {
  double* a;
  double* b;
  double* c_sqrt;
  double* eta;
  double* j_sqrt;
};
struct OrcSE {
  double* e;
  double* g;
  double* l_sqrt;
};

// Linear-Gaussian chain (pode_chain): N steps, state dim D, up to M
// observation rows per step (obs_rows[n] of them used; 0 = vacuous).
struct OrcChain {
  int32_t state_dim;
  int32_t obs_rows_max;
  int64_t steps;
  const double* init_mean;
  const double* init_cov_sqrt;
  const double* phi;     // N*D*D, or D*D when phi_shared
  const double* q_sqrt;  // N*D*D, or D*D when q_shared
  int32_t phi_shared;
  int32_t q_shared;
  const int32_t* obs_rows;
  const double* h;       // N*M*D
  const double* offset;  // N*M
  const double* r_sqrt;  // N*M*M
};

struct OrcRtsOut {
  double* filtered_mean;
  double* filtered_cov_sqrt;
  double* smoothed_mean;
  double* smoothed_cov_sqrt;
};

struct OrcScanStats {
  int64_t combine_invocations;
  int64_t sequential_depth;
};

static FilteringElement load_fe(const OrcFE& x, int64_t i, int d) {
  FilteringElement e;
  e.a = load(x.a + i * d * d, d, d);
  e.b = loadv(x.b + i * d, d);
  e.c_sqrt = load(x.c_sqrt + i * d * d, d, d);
  e.eta = loadv(x.eta + i * d, d);
  e.j_sqrt = load(x.j_sqrt + i * d * d, d, d);
  return e;
}
static void store_fe(const OrcFE& x, int64_t i, int d, const FilteringElement& e) {
  store(x.a + i * d * d, e.a);
  storev(x.b + i * d, e.b);
  store(x.c_sqrt + i * d * d, e.c_sqrt);
  storev(x.eta + i * d, e.eta);
  store(x.j_sqrt + i * d * d, e.j_sqrt);
}
static SmoothingElement load_se(const OrcSE& x, int64_t i, int d) {
  SmoothingElement e;
  e.e = load(x.e + i * d * d, d, d);
  e.g = loadv(x.g + i * d, d);
  e.l_sqrt = load(x.l_sqrt + i * d * d, d, d);
  return e;
}
static void store_se(const OrcSE& x, int64_t i, int d, const SmoothingElement& e) {
  store(x.e + i * d * d, e.e);
  storev(x.g + i * d, e.g);
  store(x.l_sqrt + i * d * d, e.l_sqrt);
}

static TransitionModel chain_transition(const OrcChain& c, int64_t n) {
  const int d = c.state_dim;
  TransitionModel t;
  t.phi = load(c.phi + (c.phi_shared ? 0 : n * d * d), d, d);
  t.q_sqrt = load(c.q_sqrt + (c.q_shared ? 0 : n * d * d), d, d);
  return t;
}
static AffineObservation chain_observation(const OrcChain& c, int64_t n) {
  const int d = c.state_dim, M = c.obs_rows_max, m = c.obs_rows[n];
  AffineObservation o;
  o.h = load(c.h + n * M * d, m, d);
  o.offset = loadv(c.offset + n * M, m);
  o.r_sqrt = Mat(m, m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) o.r_sqrt(i, j) = c.r_sqrt[n * M * M + i * M + j];
  return o;
}
static void load_chain(const OrcChain& c, GaussianSqrt& init, std::vector<TransitionModel>& tr,
                       std::vector<AffineObservation>& obs) {
  const int d = c.state_dim;
  init.mean = loadv(c.init_mean, d);
  init.cov_sqrt = load(c.init_cov_sqrt, d, d);
  tr.resize(static_cast<std::size_t>(c.steps));
  obs.resize(static_cast<std::size_t>(c.steps));
  for (int64_t n = 0; n < c.steps; ++n) {
    tr[n] = chain_transition(c, n);
    obs[n] = chain_observation(c, n);
  }
}

// ------------------------------------------------------------- linalg ---
int orc_tria(const double* m, int32_t rows, int32_t cols, double* out, Status* st) {
  return guarded(st, [&] { store(out, tria(load(m, rows, cols))); });
}

// -------------------------------------------------------- element ops ---
int orc_make_filtering_elements(const OrcChain* chain, OrcFE out, int32_t absorb_init, Status* st) {
  return guarded(st, [&] {
    GaussianSqrt init;
    std::vector<TransitionModel> tr;
    std::vector<AffineObservation> obs;
    load_chain(*chain, init, tr, obs);
    for (int64_t i = 0; i < chain->steps; ++i)
      store_fe(out, i, chain->state_dim,
               make_filtering_element(tr[i], obs[i], (absorb_init && i == 0) ? &init : nullptr));
  });
}

int orc_combine_filtering(int64_t count, int32_t d, OrcFE lhs, OrcFE rhs, OrcFE out, Status* st) {
  return guarded(st, [&] {
    for (int64_t i = 0; i < count; ++i)
      store_fe(out, i, d, combine_filtering(load_fe(lhs, i, d), load_fe(rhs, i, d)));
  });
}

// filtered: (N+1) nodes of (mean, cov_sqrt); transitions from the chain.
int orc_make_smoothing_elements(const OrcChain* chain, const double* f_mean, const double* f_cov,
                                OrcSE out, Status* st) {
  return guarded(st, [&] {
    const int d = chain->state_dim;
    for (int64_t i = 0; i <= chain->steps; ++i) {
      GaussianSqrt f{loadv(f_mean + i * d, d), load(f_cov + i * d * d, d, d)};
      store_se(out, i, d,
               i == chain->steps ? terminal_smoothing_element(f)
                                 : make_smoothing_element(f, chain_transition(*chain, i)));
    }
  });
}

int orc_combine_smoothing(int64_t count, int32_t d, OrcSE lhs, OrcSE rhs, OrcSE out, Status* st) {
  return guarded(st, [&] {
    for (int64_t i = 0; i < count; ++i)
      store_se(out, i, d, combine_smoothing(load_se(lhs, i, d), load_se(rhs, i, d)));
  });
}

// associative_scan over element arrays (parallel.hpp:136-149), serial pool.
int orc_scan_filtering(int64_t count, int32_t d, OrcFE in, OrcFE out, int32_t reverse,
                       OrcScanStats* stats, Status* st) {
  return guarded(st, [&] {
    std::vector<FilteringElement> x(static_cast<std::size_t>(count));
    for (int64_t i = 0; i < count; ++i) x[i] = load_fe(in, i, d);
    ScanStats s;
    x = associative_scan(combine_filtering, std::move(x),
                         reverse ? ScanDirection::kReverse : ScanDirection::kForward, s, nullptr);
    for (int64_t i = 0; i < count; ++i) store_fe(out, i, d, x[i]);
    if (stats) *stats = {static_cast<int64_t>(s.combine_invocations), static_cast<int64_t>(s.sequential_depth)};
  });
}

int orc_scan_smoothing(int64_t count, int32_t d, OrcSE in, OrcSE out, int32_t reverse,
                       OrcScanStats* stats, Status* st) {
  return guarded(st, [&] {
    std::vector<SmoothingElement> x(static_cast<std::size_t>(count));
    for (int64_t i = 0; i < count; ++i) x[i] = load_se(in, i, d);
    ScanStats s;
    x = associative_scan(combine_smoothing, std::move(x),
                         reverse ? ScanDirection::kReverse : ScanDirection::kForward, s, nullptr);
    for (int64_t i = 0; i < count; ++i) store_se(out, i, d, x[i]);
    if (stats) *stats = {static_cast<int64_t>(s.combine_invocations), static_cast<int64_t>(s.sequential_depth)};
  });
}

// Integer-add scan through the same tree: work/depth KATs of
// test_parallel.cpp:179-212 and acceptance.cpp:235-262.
int orc_scan_int_add(int64_t count, const int64_t* in, int64_t* out, int32_t reverse,
                     OrcScanStats* stats, Status* st) {
  return guarded(st, [&] {
    std::vector<int64_t> x(in, in + count);
    ScanStats s;
    x = associative_scan([](int64_t a, int64_t b) { return a + b; }, std::move(x),
                         reverse ? ScanDirection::kReverse : ScanDirection::kForward, s, nullptr);
    std::memcpy(out, x.data(), sizeof(int64_t) * count);
    if (stats) *stats = {static_cast<int64_t>(s.combine_invocations), static_cast<int64_t>(s.sequential_depth)};
  });
}

// ----------------------------------------------------------- smoothers ---
// mode 0: seq_rts; mode 1: para_rts on a serial pool; mode k>1: WorkPool(k).
int orc_rts(const OrcChain* chain, OrcRtsOut out, int32_t mode, OrcScanStats* stats, Status* st) {
  return guarded(st, [&] {
    GaussianSqrt init;
    std::vector<TransitionModel> tr;
    std::vector<AffineObservation> obs;
    load_chain(*chain, init, tr, obs);
    RtsResult r;
    if (mode == 0) {
      r = seq_rts(init, tr, obs);
    } else if (mode == 1) {
      r = para_rts(init, tr, obs, nullptr);
    } else {
      WorkPool pool(static_cast<unsigned>(mode));
      r = para_rts(init, tr, obs, &pool);
    }
    const int d = chain->state_dim;
    for (std::size_t n = 0; n < r.filtered.size(); ++n) {
      storev(out.filtered_mean ? out.filtered_mean + n * d : nullptr, r.filtered[n].mean);
      store(out.filtered_cov_sqrt ? out.filtered_cov_sqrt + n * d * d : nullptr, r.filtered[n].cov_sqrt);
      storev(out.smoothed_mean ? out.smoothed_mean + n * d : nullptr, r.smoothed[n].mean);
      store(out.smoothed_cov_sqrt ? out.smoothed_cov_sqrt + n * d * d : nullptr, r.smoothed[n].cov_sqrt);
    }
    if (stats) *stats = {static_cast<int64_t>(r.stats.combine_invocations), static_cast<int64_t>(r.stats.sequential_depth)};
  });
}

// -------------------------------------------------------------- solver ---
struct OrcProblem {
  int32_t kind;
  int32_t dim;
  double t_end;
  const double* y0;
  const double* params;
  int32_t n_params;
};
struct OrcPrior {
  int32_t nu;
  int32_t dim;
  double sigma;
};
struct OrcIeksConfig {
  int32_t max_iterations;
  double traj_rtol;
  double obj_atol;
  double obj_rtol;
  int32_t linearization;
};
struct OrcIeksReport {
  double* means;           // (N+1)*D
  double* cov_sqrt;        // (N+1)*D*D  (nullable)
  double* solution_means;  // (N+1)*d    (nullable)
  double* solution_covs;   // (N+1)*d*d  (nullable)
  double* objective_trace; // trace_capacity
  int32_t trace_capacity;
  int32_t iterations;
  int32_t converged;
  double sigma_hat;
  OrcScanStats scan_stats;
  double seconds;          // wall time of the solve (steady_clock)
};

static Problem to_problem(const OrcProblem& p) {
  Problem q;
  q.kind = p.kind;
  q.dim = p.dim;
  q.t_end = p.t_end;
  q.y0 = loadv(p.y0, p.dim);
  if (p.n_params > 0) q.params = loadv(p.params, p.n_params);
  if (p.kind != kAffine && q.params.empty()) q.params = make_problem(p.kind).params;
  return q;
}

// mode: 0 = seq_ieks; 1 = para_ieks on a serial pool; k > 1 = WorkPool(k); -1 = eks_solve.
int orc_ieks(const OrcProblem* problem, const OrcPrior* prior, const double* grid, int64_t n_nodes,
             const OrcIeksConfig* cfg, int32_t mode, OrcIeksReport* rep, Status* st) {
  return guarded(st, [&] {
    const Problem p = to_problem(*problem);
    const IwpPrior pr{prior->nu, prior->dim, prior->sigma};
    const std::vector<double> g(grid, grid + n_nodes);
    IeksConfig c;
    c.max_iterations = cfg->max_iterations;
    c.traj_rtol = cfg->traj_rtol;
    c.obj_atol = cfg->obj_atol;
    c.obj_rtol = cfg->obj_rtol;
    c.linearization = cfg->linearization ? Linearization::kEk0 : Linearization::kEk1;
    const auto t0 = std::chrono::steady_clock::now();
    SolverReport r;
    if (mode < 0) {
      r = eks_solve(p, pr, g, c.linearization);
    } else if (mode == 0) {
      r = ieks_drive(p, pr, g, c, nullptr);
    } else {
      WorkPool pool(mode == 1 ? 1u : static_cast<unsigned>(mode));
      r = ieks_drive(p, pr, g, c, &pool);
    }
    rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const int D = pr.state_dim(), d = pr.dim;
    for (std::size_t n = 0; n < r.marginals.size(); ++n) {
      storev(rep->means + n * D, r.marginals[n].mean);
      if (rep->cov_sqrt) store(rep->cov_sqrt + n * D * D, r.marginals[n].cov_sqrt);
      if (rep->solution_means) storev(rep->solution_means + n * d, r.solution_means[n]);
      if (rep->solution_covs) store(rep->solution_covs + n * d * d, r.solution_covs[n]);
    }
    for (std::size_t k = 0; k < r.objective_trace.size() && static_cast<int>(k) < rep->trace_capacity; ++k)
      rep->objective_trace[k] = r.objective_trace[k];
    rep->iterations = r.iterations;
    rep->converged = r.converged ? 1 : 0;
    rep->sigma_hat = r.sigma_hat;
    rep->scan_stats = {static_cast<int64_t>(r.scan_stats.combine_invocations),
                       static_cast<int64_t>(r.scan_stats.sequential_depth)};
  });
}

// ------------------------------------------------- model building blocks ---
int orc_taylor_init(const OrcProblem* problem, int32_t nu, double* mean, Status* st) {
  return guarded(st, [&] { storev(mean, taylor_init(to_problem(*problem), nu).mean); });
}

int orc_iwp_transition(const OrcPrior* prior, double h, double* phi, double* q_sqrt, Status* st) {
  return guarded(st, [&] {
    const TransitionModel t = iwp_transition(IwpPrior{prior->nu, prior->dim, prior->sigma}, h);
    store(phi, t.phi);
    store(q_sqrt, t.q_sqrt);
  });
}

int orc_preconditioner(const OrcPrior* prior, double h, double* scale, double* scale_inv, Status* st) {
  return guarded(st, [&] {
    const Preconditioner pc = preconditioner(IwpPrior{prior->nu, prior->dim, prior->sigma}, h);
    storev(scale, pc.scale);
    storev(scale_inv, pc.scale_inv);
  });
}

int orc_preconditioned_pair(const OrcPrior* prior, double* phi_bar, double* q_bar_sqrt, Status* st) {
  return guarded(st, [&] {
    const IwpPrior p{prior->nu, prior->dim, prior->sigma};
    store(phi_bar, preconditioned_phi(p));
    store(q_bar_sqrt, preconditioned_q_sqrt(p));
  });
}

// EK1/EK0 linearisation at a full state eta (statespace.cpp:65-103).
int orc_linearize(const OrcProblem* problem, int32_t nu, const double* eta, double t, int32_t ek0,
                  double* h, double* offset, Status* st) {
  return guarded(st, [&] {
    const Problem p = to_problem(*problem);
    const AffineObservation o =
        linearize(p, loadv(eta, p.dim * (nu + 1)), t, ek0 ? Linearization::kEk0 : Linearization::kEk1);
    store(h, o.h);
    storev(offset, o.offset);
  });
}

int orc_field(const OrcProblem* problem, const double* y, double t, double* f, double* jac, Status* st) {
  return guarded(st, [&] {
    const Problem p = to_problem(*problem);
    const Vec yy = loadv(y, p.dim);
    storev(f, field(p, yy, t));
    if (jac) store(jac, jacobian(p, yy, t));
  });
}

// Discretised (rescaled) prior on a grid: node scales (N+1)*D, transitions
// N*D*D phi and the unit-diffusion q factor D*D (ieks.cpp:8-47).
int orc_discretize(const OrcPrior* prior, const double* grid, int64_t n_nodes, double* node_scale,
                   double* phi, double* q_unit_sqrt, Status* st) {
  return guarded(st, [&] {
    const DiscretizedPrior dp =
        discretize(IwpPrior{prior->nu, prior->dim, prior->sigma}, std::vector<double>(grid, grid + n_nodes));
    const int D = dp.prior.state_dim();
    for (std::size_t n = 0; n < dp.node_scale.size(); ++n) storev(node_scale + n * D, dp.node_scale[n]);
    for (std::size_t n = 0; n < dp.transitions.size(); ++n) store(phi + n * D * D, dp.transitions[n].phi);
    store(q_unit_sqrt, dp.q_unit_sqrt);
  });
}

int orc_objective(int64_t n_nodes, int32_t d, const double* states, const double* phi,
                  int32_t phi_shared, const double* q_sqrt, double* value, Status* st) {
  return guarded(st, [&] {
    std::vector<Vec> s(static_cast<std::size_t>(n_nodes));
    for (int64_t n = 0; n < n_nodes; ++n) s[n] = loadv(states + n * d, d);
    std::vector<TransitionModel> tr(static_cast<std::size_t>(n_nodes - 1));
    for (int64_t n = 0; n + 1 < n_nodes; ++n) {
      tr[n].phi = load(phi + (phi_shared ? 0 : n * d * d), d, d);
      tr[n].q_sqrt = load(q_sqrt, d, d);
    }
    *value = objective_value(s, tr);
  });
}

int orc_innovation_stats(const OrcChain* chain, const double* f_mean, const double* f_cov,
                         double* sq_sum, int64_t* count, Status* st) {
  return guarded(st, [&] {
    GaussianSqrt init;
    std::vector<TransitionModel> tr;
    std::vector<AffineObservation> obs;
    load_chain(*chain, init, tr, obs);
    const int d = chain->state_dim;
    std::vector<GaussianSqrt> f(static_cast<std::size_t>(chain->steps + 1));
    for (int64_t n = 0; n <= chain->steps; ++n) f[n] = {loadv(f_mean + n * d, d), load(f_cov + n * d * d, d, d)};
    const InnovationStats s = innovation_stats(init, tr, obs, f, nullptr);
    *sq_sum = s.whitened_sq_sum;
    *count = static_cast<int64_t>(s.count);
  });
}

// ----------------------------------------------- reference fixture RNG ---
// proj/tests/oracles.cpp:168-229, draw-for-draw.
void* orc_rng_new(uint32_t seed) { return new std::mt19937(seed); }
void orc_rng_free(void* h) { delete static_cast<std::mt19937*>(h); }

static void rng_matrix(std::mt19937& rng, int rows, int cols, double* out) {
  std::normal_distribution<double> normal(0.0, 1.0);
  for (int i = 0; i < rows; ++i)
    for (int c = 0; c < cols; ++c) out[i * cols + c] = normal(rng);
}
static void rng_vector(std::mt19937& rng, int n, double* out) {
  std::normal_distribution<double> normal(0.0, 1.0);
  for (int i = 0; i < n; ++i) out[i] = normal(rng);
}
static void rng_spd_sqrt(std::mt19937& rng, int n, double* out) {
  std::uniform_real_distribution<double> diag(0.3, 1.5);
  for (int i = 0; i < n * n; ++i) out[i] = 0.0;
  std::normal_distribution<double> normal(0.0, 0.3);
  for (int i = 0; i < n; ++i) {
    for (int c = 0; c < i; ++c) out[i * n + c] = normal(rng);
    out[i * n + i] = diag(rng);
  }
}

void orc_rng_matrix(void* h, int32_t rows, int32_t cols, double* out) {
  rng_matrix(*static_cast<std::mt19937*>(h), rows, cols, out);
}
void orc_rng_vector(void* h, int32_t n, double* out) { rng_vector(*static_cast<std::mt19937*>(h), n, out); }
void orc_rng_spd_sqrt(void* h, int32_t n, double* out) { rng_spd_sqrt(*static_cast<std::mt19937*>(h), n, out); }

// oracles.cpp:194-203
void orc_rng_filtering_element(void* h, int32_t n, double* a, double* b, double* c, double* eta, double* j) {
  auto& rng = *static_cast<std::mt19937*>(h);
  rng_matrix(rng, n, n, a);
  for (int i = 0; i < n * n; ++i) a[i] *= 0.7;
  rng_vector(rng, n, b);
  rng_spd_sqrt(rng, n, c);
  rng_vector(rng, n, eta);
  rng_matrix(rng, n, n, j);
  for (int i = 0; i < n * n; ++i) j[i] *= 0.7;
}

// oracles.cpp:205-211
void orc_rng_smoothing_element(void* h, int32_t n, double* e, double* g, double* l) {
  auto& rng = *static_cast<std::mt19937*>(h);
  rng_matrix(rng, n, n, e);
  for (int i = 0; i < n * n; ++i) e[i] *= 0.7;
  rng_vector(rng, n, g);
  rng_spd_sqrt(rng, n, l);
}

// oracles.cpp:213-219 (phi = I + 0.3 * randn, q = random_spd_sqrt)
void orc_rng_transition(void* h, int32_t n, double* phi, double* q) {
  auto& rng = *static_cast<std::mt19937*>(h);
  rng_matrix(rng, n, n, phi);
  for (int i = 0; i < n * n; ++i) phi[i] *= 0.3;
  for (int i = 0; i < n; ++i) phi[i * n + i] += 1.0;
  rng_spd_sqrt(rng, n, q);
}

// oracles.cpp:221-227 (r_sqrt = 0 when noiseless, else 0.5 * random_spd_sqrt)
void orc_rng_observation(void* h, int32_t rows, int32_t n, int32_t noiseless, double* hm,
                         double* offset, double* r) {
  auto& rng = *static_cast<std::mt19937*>(h);
  rng_matrix(rng, rows, n, hm);
  rng_vector(rng, rows, offset);
  if (noiseless) {
    for (int i = 0; i < rows * rows; ++i) r[i] = 0.0;
  } else {
    rng_spd_sqrt(rng, rows, r);
    for (int i = 0; i < rows * rows; ++i) r[i] *= 0.5;
  }
}

}  // extern "C"
