// ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp).
// Square-root Kalman filter / RTS smoother (proj/src/sequential.cpp), scan
// elements and operators (proj/src/parallel.cpp) and the CPU work pool
// (proj/src/work_pool.cpp).
#include <atomic>
#include <condition_variable>
#include <exception>
#include <mutex>
#include <thread>

#include "orc.hpp"

namespace orc {

// ------------------------------------------------------------ sequential ---
namespace {
void check_aligned(const GaussianSqrt& init, const std::vector<TransitionModel>& tr,
                   const std::vector<AffineObservation>& obs) {  // sequential.cpp:7-26
  if (tr.empty() || tr.size() != obs.size())
    throw DimensionError("smoother: need N >= 1 aligned transitions and observations");
  const int d = static_cast<int>(init.mean.size());
  if (init.cov_sqrt.r != d || init.cov_sqrt.c != d)
    throw DimensionError("smoother: initial covariance factor must be square and match the mean");
  for (const auto& t : tr)
    if (t.phi.r != d || t.phi.c != d || t.q_sqrt.r != d)
      throw DimensionError("smoother: transition dimensions disagree with the state");
  for (const auto& o : obs)
    if (o.h.c != d || o.h.r != static_cast<int>(o.offset.size()))
      throw DimensionError("smoother: observation dimensions disagree with the state");
}
}  // namespace

// sequential.cpp:30-39
GaussianSqrt kf_predict(const GaussianSqrt& s, const TransitionModel& t) {
  const int d = static_cast<int>(s.mean.size());
  if (t.phi.r != d || t.phi.c != d || t.q_sqrt.r != d)
    throw DimensionError("kf_predict: transition dimensions disagree with the state");
  GaussianSqrt p;
  p.mean = t.phi * s.mean;
  p.cov_sqrt = sqrt_sum(t.phi * s.cov_sqrt, t.q_sqrt);
  return p;
}

// sequential.cpp:41-67
GaussianSqrt kf_update(const GaussianSqrt& pred, const AffineObservation& obs) {
  const int d = static_cast<int>(pred.mean.size());
  const int m = obs.h.r;
  if (obs.h.c != d || static_cast<int>(obs.offset.size()) != m || obs.r_sqrt.r != m)
    throw DimensionError("kf_update: observation dimensions disagree with the state");
  if (m == 0) return pred;
  Mat stacked(m + d, d + obs.r_sqrt.c);
  set_block(stacked, 0, 0, obs.h * pred.cov_sqrt);
  set_block(stacked, 0, d, obs.r_sqrt);
  set_block(stacked, m, 0, pred.cov_sqrt);
  const Mat psi = tria(stacked);
  const Mat s_sqrt = block(psi, 0, 0, m, m);
  require_nonsingular_triangular(s_sqrt, "kf_update: innovation covariance");
  // K = psi_21 psi_11^-1 via psi_11^T K^T = psi_21^T.
  const Mat gain = transpose(solve_upper(transpose(s_sqrt), transpose(block(psi, m, 0, d, m))));
  GaussianSqrt out;
  out.mean = pred.mean - gain * (obs.h * pred.mean - obs.offset);
  out.cov_sqrt = block(psi, m, m, d, d);
  return out;
}

// sequential.cpp:69-79
std::vector<GaussianSqrt> kf_forward(const GaussianSqrt& init,
                                     const std::vector<TransitionModel>& tr,
                                     const std::vector<AffineObservation>& obs) {
  check_aligned(init, tr, obs);
  std::vector<GaussianSqrt> marg(tr.size() + 1);
  marg[0] = init;
  for (std::size_t n = 0; n < tr.size(); ++n) marg[n + 1] = kf_update(kf_predict(marg[n], tr[n]), obs[n]);
  return marg;
}

namespace {
struct SmootherGain {
  Mat gain, residual_sqrt;
};
// sequential.cpp:89-107
SmootherGain smoother_gain(const GaussianSqrt& f, const TransitionModel& t) {
  const int d = static_cast<int>(f.mean.size());
  Mat stacked(2 * d, 2 * d);
  set_block(stacked, 0, 0, t.phi * f.cov_sqrt);
  set_block(stacked, 0, d, t.q_sqrt);
  set_block(stacked, d, 0, f.cov_sqrt);
  const Mat pi = tria(stacked);
  const Mat pred_sqrt = block(pi, 0, 0, d, d);
  require_nonsingular_triangular(pred_sqrt, "rts_smooth_pass: predicted covariance");
  SmootherGain out;
  out.gain = transpose(solve_upper(transpose(pred_sqrt), transpose(block(pi, d, 0, d, d))));
  out.residual_sqrt = block(pi, d, d, d, d);
  return out;
}
}  // namespace

// sequential.cpp:109-124
std::vector<GaussianSqrt> rts_smooth_pass(const std::vector<GaussianSqrt>& filtered,
                                          const std::vector<TransitionModel>& tr) {
  if (filtered.size() != tr.size() + 1 || tr.empty())
    throw DimensionError("rts_smooth_pass: need N+1 filtered marginals for N >= 1 transitions");
  std::vector<GaussianSqrt> sm(filtered.size());
  sm.back() = filtered.back();
  for (std::size_t n = tr.size(); n-- > 0;) {
    const SmootherGain sg = smoother_gain(filtered[n], tr[n]);
    sm[n].mean = filtered[n].mean + sg.gain * (sm[n + 1].mean - tr[n].phi * filtered[n].mean);
    sm[n].cov_sqrt = sqrt_sum(sg.gain * sm[n + 1].cov_sqrt, sg.residual_sqrt);
  }
  return sm;
}

// sequential.cpp:126-132
RtsResult seq_rts(const GaussianSqrt& init, const std::vector<TransitionModel>& tr,
                  const std::vector<AffineObservation>& obs) {
  RtsResult out;
  out.filtered = kf_forward(init, tr, obs);
  out.smoothed = rts_smooth_pass(out.filtered, tr);
  return out;
}

// -------------------------------------------------------------- parallel ---
// parallel.cpp:5-65
FilteringElement make_filtering_element(const TransitionModel& t, const AffineObservation& o,
                                        const GaussianSqrt* init) {
  const int d = t.phi.r;
  if (t.phi.c != d || t.q_sqrt.r != d || o.h.c != d)
    throw DimensionError("make_filtering_element: model dimensions disagree");
  if (init != nullptr) {
    const GaussianSqrt post = kf_update(kf_predict(*init, t), o);
    FilteringElement el;
    el.a = Mat(d, d);
    el.b = post.mean;
    el.c_sqrt = post.cov_sqrt;
    el.eta.assign(d, 0.0);
    el.j_sqrt = Mat(d, d);
    return el;
  }
  const int m = o.h.r;
  if (m == 0) {
    FilteringElement el;
    el.a = t.phi;
    el.b.assign(d, 0.0);
    el.c_sqrt = t.q_sqrt;
    el.eta.assign(d, 0.0);
    el.j_sqrt = Mat(d, d);
    return el;
  }
  Mat stacked(m + d, d + o.r_sqrt.c);
  set_block(stacked, 0, 0, o.h * t.q_sqrt);
  set_block(stacked, 0, d, o.r_sqrt);
  set_block(stacked, m, 0, t.q_sqrt);
  const Mat psi = tria(stacked);
  const Mat s_sqrt = block(psi, 0, 0, m, m);
  require_nonsingular_triangular(s_sqrt, "make_filtering_element: innovation covariance");
  const Mat gain = transpose(solve_upper(transpose(s_sqrt), transpose(block(psi, m, 0, d, m))));
  FilteringElement el;
  el.a = t.phi - gain * (o.h * t.phi);
  el.b = gain * o.offset;
  el.c_sqrt = block(psi, m, m, d, d);
  const Mat scaled_h = solve_lower(s_sqrt, o.h * t.phi);  // S^-1/2 H phi (m x d)
  el.j_sqrt = Mat(d, d);
  set_block(el.j_sqrt, 0, 0, transpose(scaled_h));
  el.eta = transpose(scaled_h) * solve_lower(s_sqrt, o.offset);
  return el;
}

// parallel.cpp:67-100
FilteringElement combine_filtering(const FilteringElement& lhs, const FilteringElement& rhs) {
  const int d = lhs.a.r;
  if (rhs.a.r != d || lhs.c_sqrt.r != d || rhs.j_sqrt.r != d || lhs.c_sqrt.c != d ||
      rhs.j_sqrt.c != d || lhs.j_sqrt.c != d || rhs.c_sqrt.c != d)
    throw DimensionError("combine_filtering: element factors must be square");
  Mat stacked(2 * d, 2 * d);
  set_block(stacked, 0, 0, transpose(lhs.c_sqrt) * rhs.j_sqrt);
  set_block(stacked, 0, d, Mat::identity(d));
  set_block(stacked, d, 0, rhs.j_sqrt);
  const Mat xi = tria(stacked);
  const Mat xi11 = block(xi, 0, 0, d, d);
  require_nonsingular_triangular(xi11, "combine_filtering: combination factor");
  const Mat xi21 = block(xi, d, 0, d, d);
  const Mat xi22 = block(xi, d, d, d, d);
  // W = C_i Xi_11^-T  (solve Xi_11 W^T = C_i^T)
  const Mat w = transpose(solve_lower(xi11, transpose(lhs.c_sqrt)));
  const Mat g = Mat::identity(d) - w * transpose(xi21);
  FilteringElement out;
  out.a = rhs.a * g * lhs.a;
  out.b = rhs.a * g * (lhs.b + lhs.c_sqrt * (transpose(lhs.c_sqrt) * rhs.eta)) + rhs.b;
  out.c_sqrt = sqrt_sum(rhs.a * w, rhs.c_sqrt);
  out.eta = transpose(lhs.a) * transpose(g) *
                (rhs.eta - rhs.j_sqrt * (transpose(rhs.j_sqrt) * lhs.b)) +
            lhs.eta;
  out.j_sqrt = sqrt_sum(transpose(lhs.a) * xi22, lhs.j_sqrt);
  return out;
}

// parallel.cpp:102-110
FilteringElement filtering_identity(int d) {
  FilteringElement el;
  el.a = Mat::identity(d);
  el.b.assign(d, 0.0);
  el.c_sqrt = Mat(d, d);
  el.eta.assign(d, 0.0);
  el.j_sqrt = Mat(d, d);
  return el;
}

// parallel.cpp:112-135
SmoothingElement make_smoothing_element(const GaussianSqrt& f, const TransitionModel& t) {
  const int d = static_cast<int>(f.mean.size());
  if (t.phi.r != d || t.phi.c != d || t.q_sqrt.r != d)
    throw DimensionError("make_smoothing_element: model dimensions disagree");
  Mat stacked(2 * d, 2 * d);
  set_block(stacked, 0, 0, t.phi * f.cov_sqrt);
  set_block(stacked, 0, d, t.q_sqrt);
  set_block(stacked, d, 0, f.cov_sqrt);
  const Mat pi = tria(stacked);
  const Mat pred_sqrt = block(pi, 0, 0, d, d);
  require_nonsingular_triangular(pred_sqrt, "make_smoothing_element: predicted covariance");
  SmoothingElement el;
  el.e = transpose(solve_upper(transpose(pred_sqrt), transpose(block(pi, d, 0, d, d))));
  el.g = f.mean - el.e * (t.phi * f.mean);
  el.l_sqrt = block(pi, d, d, d, d);
  return el;
}

// parallel.cpp:137-144
SmoothingElement terminal_smoothing_element(const GaussianSqrt& f) {
  const int d = static_cast<int>(f.mean.size());
  SmoothingElement el;
  el.e = Mat(d, d);
  el.g = f.mean;
  el.l_sqrt = f.cov_sqrt;
  return el;
}

// parallel.cpp:146-156
SmoothingElement combine_smoothing(const SmoothingElement& lhs, const SmoothingElement& rhs) {
  const int d = lhs.e.r;
  if (rhs.e.r != d) throw DimensionError("combine_smoothing: element dimensions disagree");
  SmoothingElement out;
  out.e = lhs.e * rhs.e;
  out.g = lhs.e * rhs.g + lhs.g;
  out.l_sqrt = sqrt_sum(lhs.e * rhs.l_sqrt, lhs.l_sqrt);
  return out;
}

// parallel.cpp:158-164
SmoothingElement smoothing_identity(int d) {
  SmoothingElement el;
  el.e = Mat::identity(d);
  el.g.assign(d, 0.0);
  el.l_sqrt = Mat(d, d);
  return el;
}

// parallel.cpp:166-209
RtsResult para_rts(const GaussianSqrt& init, const std::vector<TransitionModel>& tr,
                   const std::vector<AffineObservation>& obs, WorkPool* pool) {
  if (tr.empty() || tr.size() != obs.size())
    throw DimensionError("para_rts: need N >= 1 aligned transitions and observations");
  const std::size_t n = tr.size();
  std::vector<FilteringElement> fe(n);
  parallel_map(pool, n, [&](std::size_t i) {
    fe[i] = make_filtering_element(tr[i], obs[i], i == 0 ? &init : nullptr);
  });
  ScanStats fwd;
  const std::vector<FilteringElement> prefixes =
      associative_scan(combine_filtering, std::move(fe), ScanDirection::kForward, fwd, pool);
  RtsResult out;
  out.filtered.resize(n + 1);
  out.filtered[0] = init;
  parallel_map(pool, n, [&](std::size_t i) {
    out.filtered[i + 1] = GaussianSqrt{prefixes[i].b, prefixes[i].c_sqrt};
  });
  std::vector<SmoothingElement> se(n + 1);
  parallel_map(pool, n + 1, [&](std::size_t i) {
    se[i] = (i == n) ? terminal_smoothing_element(out.filtered[n])
                     : make_smoothing_element(out.filtered[i], tr[i]);
  });
  ScanStats rev;
  const std::vector<SmoothingElement> suffixes =
      associative_scan(combine_smoothing, std::move(se), ScanDirection::kReverse, rev, pool);
  out.smoothed.resize(n + 1);
  parallel_map(pool, n + 1, [&](std::size_t i) {
    out.smoothed[i] = GaussianSqrt{suffixes[i].g, suffixes[i].l_sqrt};
  });
  out.stats = fwd;
  out.stats.merge_max(rev);
  return out;
}

// ------------------------------------------------------------- work pool ---
// proj/src/work_pool.cpp:7-85
struct WorkPool::Impl {
  std::vector<std::thread> threads;
  std::mutex mutex;
  std::condition_variable work_cv, done_cv;
  const std::function<void(std::size_t)>* body = nullptr;
  std::size_t count = 0;
  std::atomic<std::size_t> next{0};
  unsigned active = 0;
  std::uint64_t epoch = 0;
  bool stopping = false;
  std::exception_ptr first_error;

  void run_items() {
    for (;;) {
      const std::size_t i = next.fetch_add(1);
      if (i >= count) return;
      {
        std::lock_guard<std::mutex> lock(mutex);
        if (first_error) continue;
      }
      try {
        (*body)(i);
      } catch (...) {
        std::lock_guard<std::mutex> lock(mutex);
        if (!first_error) first_error = std::current_exception();
      }
    }
  }

  void worker_loop() {
    std::uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lock(mutex);
        work_cv.wait(lock, [&] { return stopping || epoch != seen; });
        if (stopping) return;
        seen = epoch;
      }
      run_items();
      {
        std::lock_guard<std::mutex> lock(mutex);
        if (--active == 0) done_cv.notify_all();
      }
    }
  }
};

WorkPool::WorkPool(unsigned width) {
  if (width == 0) width = std::max(1u, std::thread::hardware_concurrency());
  width_ = width;
  impl_ = new Impl();
  for (unsigned t = 1; t < width_; ++t) impl_->threads.emplace_back([this] { impl_->worker_loop(); });
}

WorkPool::~WorkPool() {
  {
    std::lock_guard<std::mutex> lock(impl_->mutex);
    impl_->stopping = true;
  }
  impl_->work_cv.notify_all();
  for (auto& t : impl_->threads) t.join();
  delete impl_;
}

void WorkPool::parallel_for(std::size_t count, const std::function<void(std::size_t)>& body) {
  if (count == 0) return;
  if (width_ == 1) {
    for (std::size_t i = 0; i < count; ++i) body(i);
    return;
  }
  {
    std::lock_guard<std::mutex> lock(impl_->mutex);
    impl_->body = &body;
    impl_->count = count;
    impl_->next.store(0);
    impl_->first_error = nullptr;
    impl_->active = width_ - 1;
    ++impl_->epoch;
  }
  impl_->work_cv.notify_all();
  impl_->run_items();
  std::exception_ptr err;
  {
    std::unique_lock<std::mutex> lock(impl_->mutex);
    impl_->done_cv.wait(lock, [&] { return impl_->active == 0; });
    err = impl_->first_error;
    impl_->body = nullptr;
  }
  if (err) std::rethrow_exception(err);
}

void parallel_map(WorkPool* pool, std::size_t count, const std::function<void(std::size_t)>& body) {
  if (pool != nullptr) {
    pool->parallel_for(count, body);
  } else {
    for (std::size_t i = 0; i < count; ++i) body(i);
  }
}

}  // namespace orc
