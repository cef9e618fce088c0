// The IEKS Gauss-Newton loop on the device (replaces ieks_drive,
// proj/src/ieks.cpp:114-210): per-step linearisation, the scan-based
// smoother, the objective / stopping reductions and the final calibration
// and projection.  Only the three convergence scalars cross to the host per
// iteration.
#pragma once

#include <cmath>
#include <vector>

#include "engine.cuh"
#include "host_model.hpp"
#include "field.cuh"

namespace pode {

constexpr int kRedThreads = 256;

// Node scales T(h_n) (prior.cpp:79-97) with the incoming step; node 0 uses
// step 0 (ieks.cpp:28-33).
static __global__ void k_node_scales(const double* grid, int64_t n1, int nu, int dim, double* scale,
                              double* scale_inv) {
  const int64_t n = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (n >= n1) return;
  const double h = (n == 0) ? grid[1] - grid[0] : grid[n] - grid[n - 1];
  const double root_h = sqrt(h);
  const int b = nu + 1, D = b * dim;
  double fact = 1.0;
  double taus[8];
  for (int i = nu; i >= 0; --i) {  // factorial(nu - i) built up as i decreases
    const int k = nu - i;
    if (k > 0) fact *= k;
    taus[i] = root_h * pow(h, double(k)) / fact;
  }
  for (int r = 0; r < dim; ++r)
    for (int i = 0; i <= nu; ++i) {
      scale[n * D + r * b + i] = taus[i];
      scale_inv[n * D + r * b + i] = 1.0 / taus[i];
    }
}

// Rescaled transitions phi_n = phi_bar diag(T_n ⊙ T_{n+1}^-1) (ieks.cpp:37-45).
static __global__ void k_transitions(const double* phibar, const double* scale, const double* scale_inv, int64_t N,
                              int D, double* phi) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= N * D) return;
  const int64_t n = t / D;
  const int r = int(t - n * D);
  for (int c = 0; c < D; ++c)
    phi[(n * D + r) * D + c] = phibar[r * D + c] * (scale[n * D + c] * scale_inv[(n + 1) * D + c]);
}

static __global__ void k_fill_rows(const double* row, int64_t n, int D, double* out) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= n * D) return;
  out[t] = row[t % D];
}

// EK1 / EK0 linearisation at eta[i+1], rescaled into node-(i+1) coordinates
// (statespace.cpp:65-103, ieks.cpp:160-164).  obs rows = d, R = 0.
template <int DMAX>
static __global__ void k_linearize(DevProblem prob, int nu, const double* eta, const double* grid,
                            const double* scale, int64_t N, int ek0, double* h, double* off,
                            DevError* err) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= N) return;
  const int d = prob.dim, b = nu + 1, D = d * b;
  const double* e = eta + (i + 1) * D;
  const double* s = scale + (i + 1) * D;
  double y[DMAX], f[DMAX], jac[DMAX * DMAX];
  for (int r = 0; r < d; ++r) y[r] = e[r * b];
  eval_field<DMAX>(prob, y, f, jac, grid[i + 1]);
  bool finite = true;
  for (int r = 0; r < d; ++r) finite &= isfinite(f[r]);
  if (!ek0)
    for (int r = 0; r < d; ++r)
      for (int c = 0; c < d; ++c) finite &= isfinite(jac[r * DMAX + c]);
  if (!finite) raise_error(err, i + 1, kErrLinearization);
  for (int r = 0; r < d; ++r) {
    double* hr = h + (i * d + r) * D;
    for (int c = 0; c < D; ++c) hr[c] = 0.0;
    hr[r * b + 1] = 1.0 * s[r * b + 1];
    if (ek0) {
      off[i * d + r] = f[r];
    } else {
      double jy = 0.0;
      for (int c = 0; c < d; ++c) {
        hr[c * b] = -jac[r * DMAX + c] * s[c * b];
        jy += jac[r * DMAX + c] * y[c];
      }
      off[i * d + r] = f[r] - jy;
    }
  }
}

// new_eta = T ⊙ m_s, plus per-node / per-step terms of the objective
// (ieks.cpp:49-60, 136-144) and the stopping maxima (ieks.cpp:62-77);
// one block-level partial per block, summed in a fixed order.
// smean == nullptr evaluates the objective of eta_old itself (the constant
// start, ieks.cpp:147-148).
static __global__ void k_eta_objective(const double* smean, const double* scale, const double* scale_inv,
                                const double* eta_old, const double* phi, const double* qunit,
                                const double* qinv_diag, int64_t n1, int D, double* eta_new, double* part) {
  __shared__ double s_obj[kRedThreads], s_dmax[kRedThreads], s_emax[kRedThreads];
  const int64_t n = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  auto state = [&](int64_t node, int k) {
    return smean ? scale[node * D + k] * smean[node * D + k] : eta_old[node * D + k];
  };
  double obj = 0.0, dmax = 0.0, emax = 0.0;
  if (n < n1) {
    for (int k = 0; k < D; ++k) {
      const double v = state(n, k);
      if (smean) eta_new[n * D + k] = v;
      dmax = fmax(dmax, fabs(v - eta_old[n * D + k]));
      emax = fmax(emax, fabs(v));
    }
  }
  if (n < n1 - 1) {
    // increment of step n in rescaled coordinates, whitened by Q_unit^1/2
    double inc[32], w[32];
    for (int k = 0; k < D; ++k) {
      double acc = 0.0;
      for (int c = 0; c < D; ++c) acc += phi[(n * D + k) * D + c] * (scale_inv[n * D + c] * state(n, c));
      inc[k] = scale_inv[(n + 1) * D + k] * state(n + 1, k) - acc;
    }
    double acc2 = 0.0;
    for (int k = 0; k < D; ++k) {
      double a = inc[k];
      for (int c = 0; c < k; ++c) a -= qunit[k * D + c] * w[c];
      w[k] = a * qinv_diag[k];
      acc2 += w[k] * w[k];
    }
    obj = acc2;
  }
  s_obj[threadIdx.x] = obj;
  s_dmax[threadIdx.x] = dmax;
  s_emax[threadIdx.x] = emax;
  __syncthreads();
  for (int s = kRedThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      s_obj[threadIdx.x] += s_obj[threadIdx.x + s];
      s_dmax[threadIdx.x] = fmax(s_dmax[threadIdx.x], s_dmax[threadIdx.x + s]);
      s_emax[threadIdx.x] = fmax(s_emax[threadIdx.x], s_emax[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x * 3 + 0] = s_obj[0];
    part[blockIdx.x * 3 + 1] = s_dmax[0];
    part[blockIdx.x * 3 + 2] = s_emax[0];
  }
}

// Fixed-order finish of block partials (sum_0, max_1, max_2), valid in
// thread 0 of a kRedThreads block.
__device__ __forceinline__ void finish3_block(const double* part, int64_t nparts, double (&out)[3]) {
  __shared__ double s0[kRedThreads], s1[kRedThreads], s2[kRedThreads];
  double a = 0.0, b = 0.0, c = 0.0;
  for (int64_t k = threadIdx.x; k < nparts; k += blockDim.x) {
    a += part[k * 3 + 0];
    b = fmax(b, part[k * 3 + 1]);
    c = fmax(c, part[k * 3 + 2]);
  }
  s0[threadIdx.x] = a;
  s1[threadIdx.x] = b;
  s2[threadIdx.x] = c;
  __syncthreads();
  for (int s = kRedThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      s0[threadIdx.x] += s0[threadIdx.x + s];
      s1[threadIdx.x] = fmax(s1[threadIdx.x], s1[threadIdx.x + s]);
      s2[threadIdx.x] = fmax(s2[threadIdx.x], s2[threadIdx.x + s]);
    }
    __syncthreads();
  }
  out[0] = s0[0];
  out[1] = s1[0];
  out[2] = s2[0];
}

static __global__ void k_finish3(const double* part, int64_t nparts, double* out) {
  double r[3];
  finish3_block(part, nparts, r);
  if (threadIdx.x == 0) {
    out[0] = r[0];
    out[1] = r[1];
    out[2] = r[2];
  }
}

// Whitened innovation of step i from filtered[i] (innovation_stats,
// ieks.cpp:79-104): pred = kf_predict(filtered[i]); S = tria([H P^1/2, R^1/2]);
// value = ||S^-1 (H m - offset)||^2.
template <int D>
__global__ void __launch_bounds__(kThreads) k_innovation(DevChain ch, const double* fm, const double* fc,
                                                         double* values, DevError* err) {
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t i = group_index<D>(g);
  const bool ok = g.real() && i < ch.N;
  Gauss<D> f;
  f.m = ld_ent<D>(fm, i, g.r, ok);
  f.c = ld_row<D>(fc, i, g.r, ok);
  const Rw<D> phi = chain_phi<D>(ch, i, g.r, ok);
  const Rw<D> q = chain_q<D>(ch, i, g.r, ok);
  const Obs<D, D> o = load_obs<D>(ch, i, g.r, ok);
  const Gauss<D> p = kf_predict(g, f, phi, q);
  constexpr int K = 2 * D;
  Rw<K> top, none = zeros<K>();
  const Rw<D> hp = mm(g, o.h, p.c);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    top[j] = hp[j];
    top[D + j] = o.r[j];
  }
  lq<D, D, 0, K>(g, top, none);
  const bool sing = singular_diag(g, pick(top, g.r), o.m);
  const double z = matvec(g, o.h, p.m) - o.off;
  Rw<D> srow;
#pragma unroll
  for (int j = 0; j < D; ++j) srow[j] = top[j];
  publish_factor<D, D>(g, srow);
  const Rw<D> zv = gather_vec(g, z);
  const Rw<D> w = solve_vec_lower_all(g, zv);
  double v = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) v = fma(w[k], w[k], v);
  if (ok && g.r == 0) {
    values[i] = v;
    if (sing) raise_error(err, i, kErrSingular);
  }
}

// Fixed-order sum of values[0..n).
static __global__ void k_sum_blocks(const double* values, int64_t n, double* part) {
  __shared__ double s[kRedThreads];
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  s[threadIdx.x] = i < n ? values[i] : 0.0;
  __syncthreads();
  for (int k = kRedThreads / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) s[threadIdx.x] += s[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x * 3 + 0] = s[0];
    part[blockIdx.x * 3 + 1] = 0.0;
    part[blockIdx.x * 3 + 2] = 0.0;
  }
}

// Calibrated outputs in original coordinates (ieks.cpp:196-208).
static __global__ void k_outputs(const double* eta, const double* scov, const double* scale, double sigma_rel,
                          int64_t n1, int D, int nu, int dim, double* means, double* cov, double* sol_m,
                          double* sol_c) {
  const int64_t n = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (n >= n1) return;
  const int b = nu + 1;
  if (means)
    for (int k = 0; k < D; ++k) means[n * D + k] = eta[n * D + k];
  if (cov)
    for (int r = 0; r < D; ++r)
      for (int c = 0; c < D; ++c) cov[(n * D + r) * D + c] = scale[n * D + r] * scov[(n * D + r) * D + c] * sigma_rel;
  if (sol_m)
    for (int r = 0; r < dim; ++r) sol_m[n * dim + r] = eta[n * D + r * b];
  if (sol_c)
    for (int r = 0; r < dim; ++r)
      for (int c = 0; c < dim; ++c) {
        double acc = 0.0;
        for (int k = 0; k < D; ++k)
          acc += (scale[n * D + r * b] * scov[(n * D + r * b) * D + k] * sigma_rel) *
                 (scale[n * D + c * b] * scov[(n * D + c * b) * D + k] * sigma_rel);
        sol_c[(n * dim + r) * dim + c] = acc;
      }
}

struct IeksResult {
  int iterations = 0;
  bool converged = false;
  double sigma_hat = 0.0;
  std::vector<double> trace;
  ScanTally stats;
};

inline unsigned grid1(int64_t n, int threads = kRedThreads) {
  return static_cast<unsigned>((n + threads - 1) / threads);
}

// Everything a solve needs on the device besides the iteration itself.
template <int D>
struct IeksSetup {
  int nu = 0, dim = 0;
  int64_t N = 0, n1 = 0;
  double* grid = nullptr;
  double* scale = nullptr;
  double* scale_inv = nullptr;
  double* phibar = nullptr;
  double* qunit = nullptr;
  double* q = nullptr;
  double* qinv = nullptr;
  double* mu0 = nullptr;
  double* init_m = nullptr;  // T_0^-1 mu0, then D*D zeros
  std::vector<double> h_qunit, h_q, h_qinv, h_m0;
  DevProblem prob{};
};

// eks_solve's forward pass (ieks.cpp:237-250): group 0 of one warp walks the
// N steps in order, linearising step n at its own predicted mean
// eta = T_{n+1} ⊙ m^- (k_linearize's formulas, statespace.cpp:65-103); the
// step's observation model lands in the chain (H, offset), the filtered
// marginals in fm / fc (rescaled coordinates).  Inherently sequential: the
// linearisation point of step n depends on the filter up to step n.
template <int D>
__global__ void __launch_bounds__(32) k_eks_forward(DevChain ch, DevProblem prob, int nu, const double* grid,
                                                    const double* scale,
                                                    int ek0, double* fm, double* fc, DevError* err) {
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const bool ok = g.real() && g.gw == 0;
  const int d = prob.dim, b = nu + 1;
  double* const h = const_cast<double*>(ch.h);
  double* const off = const_cast<double*>(ch.off);
  Gauss<D> f;
  f.m = ok ? ch.init_mean[g.r] : 0.0;
  f.c = ld_row<D>(ch.init_cov, 0, g.r, ok);
  st_ent<D>(fm, 0, g.r, ok, f.m);
  st_row<D>(fc, 0, g.r, ok, f.c);
  // phi_n is loaded one step ahead; the step's observation rows are built
  // in registers (lane r < d owns row r; R = 0, padded rows carry the unit
  // dummy of load_obs) and only written out for the smoother / innovations
  Rw<D> phi_next = chain_phi<D>(ch, 0, g.r, ok);
#pragma unroll 1
  for (int64_t n = 0; n < ch.N; ++n) {
    const Rw<D> phi = phi_next;
    phi_next = chain_phi<D>(ch, n + 1 < ch.N ? n + 1 : n, g.r, ok);
    const Rw<D> q = chain_q<D>(ch, n, g.r, ok);
    Gauss<D> p = kf_predict(g, f, phi, q);
    const double* s = scale + (n + 1) * D;
    const Rw<D> eta = gather_vec(g, ok ? s[g.r] * p.m : 0.0);
    Obs<D, D> o;
    o.m = ok ? d : 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      o.h[j] = 0.0;
      o.r[j] = ((!ok || g.r >= d) && j == g.r) ? 1.0 : 0.0;
    }
    o.off = 0.0;
    if (ok && g.r < d) {
      double y[D], fv[D], jac[D * D];
      for (int r = 0; r < d; ++r) y[r] = eta[r * b];
      eval_field<D>(prob, y, fv, jac, grid[n + 1]);
      const int r = g.r;
      bool finite = isfinite(fv[r]);
      if (!ek0)
        for (int c = 0; c < d; ++c) finite &= isfinite(jac[r * D + c]);
      if (!finite) raise_error(err, n + 1, kErrLinearization);
      double ov;
      if (ek0) {
        ov = fv[r];
      } else {
        double jy = 0.0;
        for (int c = 0; c < d; ++c) jy += jac[r * D + c] * y[c];
        ov = fv[r] - jy;
      }
#pragma unroll
      for (int j = 0; j < D; ++j) {  // H = E_1 - F_y E_0, rescaled (k_linearize)
        double v = 0.0;
        if (j == r * b + 1)
          v = 1.0 * s[j];
        else if (!ek0 && j % b == 0)
          v = -jac[r * D + j / b] * s[j];
        o.h[j] = v;
        h[(n * d + r) * D + j] = v;
      }
      o.off = ov;
      off[n * d + r] = ov;
    }
    const bool good = kf_update<D, D>(g, p, o);
    if (ok && g.r == 0 && !good) raise_error(err, n + 1, kErrSingular);
    f = p;
    st_ent<D>(fm, n + 1, g.r, ok, f.m);
    st_row<D>(fc, n + 1, g.r, ok, f.c);
  }
}

template <int D>
struct IeksEngine {
  // node_scales = false (fused engine): T_n is recomputed in the kernels, so
  // only T_0 is needed, on the host — no scale arrays, no stream sync.
  static void setup(pode_context* ctx, const host::Problem& p, const pode_prior& prior, const double* grid_h,
                    int64_t n1, IeksSetup<D>& s, bool node_scales = true) {
    s.nu = prior.nu;
    s.dim = prior.dim;
    s.n1 = n1;
    s.N = n1 - 1;
    cudaStream_t st = ctx->stream;
    Workspace& ws = ctx->ws;
    s.grid = ws.arr<double>("ieks_grid", n1);
    cuda_check(cudaMemcpyAsync(s.grid, grid_h, sizeof(double) * n1, cudaMemcpyHostToDevice, st), "grid");
    if (node_scales) {
      s.scale = ws.arr<double>("ieks_scale", n1 * D);
      s.scale_inv = ws.arr<double>("ieks_scale_inv", n1 * D);
      k_node_scales<<<grid1(n1), kRedThreads, 0, st>>>(s.grid, n1, s.nu, s.dim, s.scale, s.scale_inv);
      note_launch(ctx, "node_scales");
    }
    const std::vector<double> phibar = host::preconditioned_phi(s.nu, s.dim);
    s.h_qunit = host::preconditioned_q_sqrt(s.nu, s.dim);
    s.h_q = s.h_qunit;
    for (auto& x : s.h_q) x *= prior.sigma;
    s.h_qinv.resize(D);
    for (int k = 0; k < D; ++k) s.h_qinv[k] = 1.0 / s.h_qunit[k * D + k];
    double* c = ws.arr<double>("ieks_consts", 3 * D * D + 2 * D + D + D * D);
    s.phibar = c;
    s.qunit = c + D * D;
    s.q = c + 2 * D * D;
    s.qinv = c + 3 * D * D;
    s.mu0 = s.qinv + D;
    s.init_m = s.mu0 + D;
    const std::vector<double> mu0 = host::taylor_init(p, s.nu);
    std::vector<double> hc(3 * D * D + 2 * D);
    std::copy(phibar.begin(), phibar.end(), hc.begin());
    std::copy(s.h_qunit.begin(), s.h_qunit.end(), hc.begin() + D * D);
    std::copy(s.h_q.begin(), s.h_q.end(), hc.begin() + 2 * D * D);
    std::copy(s.h_qinv.begin(), s.h_qinv.end(), hc.begin() + 3 * D * D);
    std::copy(mu0.begin(), mu0.end(), hc.begin() + 3 * D * D + D);
    cuda_check(cudaMemcpyAsync(c, hc.data(), sizeof(double) * hc.size(), cudaMemcpyHostToDevice, st), "consts");
    std::vector<double> si0(D);
    if (node_scales) {
      cuda_check(cudaMemcpyAsync(si0.data(), s.scale_inv, sizeof(double) * D, cudaMemcpyDeviceToHost, st), "si0");
      cuda_check(cudaStreamSynchronize(st), "sync");
    } else {  // T_0^-1 from the first step (k_node_scales' formula, ieks.cpp:28-33)
      const double h = grid_h[1] - grid_h[0], root_h = std::sqrt(h);
      double fact = 1.0;
      for (int i = s.nu; i >= 0; --i) {
        const int k = s.nu - i;
        if (k > 0) fact *= k;
        const double tau = root_h * std::pow(h, double(k)) / fact;
        for (int r = 0; r < s.dim; ++r) si0[r * (s.nu + 1) + i] = 1.0 / tau;
      }
    }
    s.h_m0.assign(D + D * D, 0.0);
    for (int k = 0; k < D; ++k) s.h_m0[k] = si0[k] * mu0[k];
    cuda_check(cudaMemcpyAsync(s.init_m, s.h_m0.data(), sizeof(double) * s.h_m0.size(), cudaMemcpyHostToDevice, st),
               "init");
    s.prob.kind = p.kind;
    s.prob.dim = s.dim;
    if (p.params.size() > size_t(kMaxParams)) throw ApiError(PODE_ERR_UNSUPPORTED, "too many problem params");
    for (size_t k = 0; k < p.params.size(); ++k) s.prob.params[k] = p.params[k];
  }

  // Observation buffers of a DevChain with rescaled transitions (d rows, R = 0).
  static DevChain chain(pode_context* ctx, const IeksSetup<D>& s, bool materialise_phi) {
    Workspace& ws = ctx->ws;
    cudaStream_t st = ctx->stream;
    const int64_t N = s.N;
    const int dim = s.dim;
    double* phi = ws.arr<double>("ieks_phi", N * D * D);
    if (materialise_phi) {
      k_transitions<<<grid1(N * D), kRedThreads, 0, st>>>(s.phibar, s.scale, s.scale_inv, N, D, phi);
      note_launch(ctx, "transitions");
    }
    double* oh = ws.arr<double>("ieks_h", N * dim * D);
    double* ooff = ws.arr<double>("ieks_off", N * dim);
    double* orr = ws.arr<double>("ieks_r", N * dim * dim);
    int32_t* orows = ws.arr<int32_t>("ieks_rows", N);
    cuda_check(cudaMemsetAsync(orr, 0, sizeof(double) * N * dim * dim, st), "r");
    std::vector<int32_t> rows(N, dim);
    cuda_check(cudaMemcpyAsync(orows, rows.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice, st), "rows");
    cuda_check(cudaStreamSynchronize(st), "sync");
    return DevChain{D, dim, N, s.init_m, s.init_m + D, phi, s.q, 0, 1, orows, oh, ooff, orr};
  }

  static void linearize(pode_context* ctx, const IeksSetup<D>& s, const DevChain& ch, const double* eta, int ek0,
                        int it) {
    DevError* err = reinterpret_cast<DevError*>(ctx->d_err);
    reset_error(ctx);
    k_linearize<D><<<grid1(s.N), kRedThreads, 0, ctx->stream>>>(s.prob, s.nu, eta, s.grid, s.scale, s.N, ek0,
                                                                const_cast<double*>(ch.h),
                                                                const_cast<double*>(ch.off), err);
    note_launch(ctx, "linearize");
    check_linearization(ctx, s, it);
  }

  // node_offset: global index of local node 0 (time-axis shards).
  // `what` (default "ieks iteration <it>") prefixes the message.
  static void check_linearization(pode_context* ctx, const IeksSetup<D>& s, int it, int64_t node_offset = 0,
                                  const char* what = nullptr) {
    const unsigned long long key = fetch_error(ctx);
    if (key == ~0ull) return;
    const int code = int(key & 0xff);
    const int64_t idx = int64_t(key >> 8) + node_offset;
    const std::string pre = what ? std::string(what) : "ieks iteration " + std::to_string(it);
    if (code == kErrLinearization) {
      double t = 0.0;
      cuda_check(cudaMemcpy(&t, s.grid + idx, sizeof(double), cudaMemcpyDeviceToHost), "t");
      throw ApiError(PODE_ERR_LINEARIZATION, pre + ": linearize: vector field evaluation is not finite", idx, t, it);
    }
    throw ApiError(PODE_ERR_SINGULAR_FACTOR, pre + (what ? ": filter" : ": smoother") + ": triangular factor is singular",
                   idx, 0.0, it);
  }

  // eks_solve (ieks.cpp:224-291): the sequential forward pass linearised at
  // the predicted means (k_eks_forward), the smoother of those filtered
  // marginals as the reverse ⊗_s scan, calibration, the objective of the
  // smoothed means and the outputs.  One "iteration", converged.
  static IeksResult run_eks(pode_context* ctx, const host::Problem& p, const pode_prior& prior, const double* grid_h,
                            int64_t n1, const pode_ieks_config& cfg, double* means, double* cov, double* sol_m,
                            double* sol_c) {
    IeksSetup<D> s;
    setup(ctx, p, prior, grid_h, n1, s);
    cudaStream_t st = ctx->stream;
    Workspace& ws = ctx->ws;
    DevError* err = reinterpret_cast<DevError*>(ctx->d_err);
    const int64_t N = s.N;
    const DevChain ch = chain(ctx, s, true);
    double* fm = ws.arr<double>("ieks_fm", n1 * D);
    double* fc = ws.arr<double>("ieks_fc", n1 * D * D);
    double* sm = ws.arr<double>("ieks_sm", n1 * D);
    double* sc = ws.arr<double>("ieks_sc", n1 * D * D);
    const int fwd_smem = int(sizeof(double) * Grp<D>::kSlots * Scratch<D>::kDoubles);
    cuda_check(cudaFuncSetAttribute(k_eks_forward<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, fwd_smem),
               "eks smem");
    reset_error(ctx);
    k_eks_forward<D><<<1, 32, fwd_smem, st>>>(ch, s.prob, s.nu, s.grid, s.scale, cfg.linearization, fm, fc, err);
    note_launch(ctx, "eks_forward");
    check_linearization(ctx, s, 1, 0, "eks_solve");
    // rts_smooth_pass of the sequential filter (sequential.cpp:105-132) as the reverse scan
    SEd se = Engine<D>::template alloc<SOps<D>>(ctx, "rts_se", N + 1);
    Engine<D>::make_smoothing(ctx, ch, fm, fc, se);
    const ScanTally t = Engine<D>::scan_smoothing(ctx, N + 1, se, se, true);
    cuda_check(cudaMemcpyAsync(sm, se.g, sizeof(double) * D * n1, cudaMemcpyDeviceToDevice, st), "smoothed");
    cuda_check(cudaMemcpyAsync(sc, se.l, sizeof(double) * D * D * n1, cudaMemcpyDeviceToDevice, st), "smoothed");
    IeksResult res;
    res.stats.combines = t.combines;
    res.stats.depth = t.depth;
    // innovation statistics and calibration (ieks.cpp:79-109)
    double* vals = ws.arr<double>("ieks_innov", N);
    cuda_check(cudaFuncSetAttribute(k_innovation<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(smem_bytes<D>())),
               "innovation smem");
    k_innovation<D><<<blocks_for<D>(N), kThreads, smem_bytes<D>(), st>>>(ch, fm, fc, vals, err);
    note_launch(ctx, "innovation");
    const int64_t np2 = grid1(N);
    double* part2 = ws.arr<double>("ieks_part2", np2 * 3 + 3);
    k_sum_blocks<<<np2, kRedThreads, 0, st>>>(vals, N, part2);
    note_launch(ctx, "sum_blocks");
    k_finish3<<<1, kRedThreads, 0, st>>>(part2, np2, part2 + np2 * 3);
    note_launch(ctx, "finish3");
    cuda_check(cudaMemcpyAsync(ctx->h_scalars, part2 + np2 * 3, sizeof(double), cudaMemcpyDeviceToHost, st),
               "innov");
    check_linearization(ctx, s, 1, 0, "eks_solve");  // syncs
    const double sigma_rel = std::sqrt(ctx->h_scalars[0] / double(N * s.dim));
    res.sigma_hat = sigma_rel * prior.sigma;
    // original-coordinate means and the objective of the smoothed trajectory (ieks.cpp:279-289)
    double* eta_old = ws.arr<double>("ieks_eta_a", n1 * D);
    double* eta_out = ws.arr<double>("ieks_eta_b", n1 * D);
    k_fill_rows<<<grid1(n1 * D), kRedThreads, 0, st>>>(s.mu0, n1, D, eta_old);
    note_launch(ctx, "fill");
    const int64_t nparts = grid1(n1);
    double* part = ws.arr<double>("ieks_part", nparts * 3 + 3);
    k_eta_objective<<<grid1(n1), kRedThreads, 0, st>>>(sm, s.scale, s.scale_inv, eta_old, ch.phi, s.qunit, s.qinv,
                                                       n1, D, eta_out, part);
    note_launch(ctx, "eta_objective");
    k_finish3<<<1, kRedThreads, 0, st>>>(part, nparts, part + nparts * 3);
    note_launch(ctx, "finish3");
    cuda_check(cudaMemcpyAsync(ctx->h_scalars, part + nparts * 3, sizeof(double) * 3, cudaMemcpyDeviceToHost, st),
               "objective");
    k_outputs<<<grid1(n1), kRedThreads, 0, st>>>(eta_out, sc, s.scale, sigma_rel, n1, D, s.nu, s.dim, means, cov,
                                                 sol_m, sol_c);
    note_launch(ctx, "outputs");
    cuda_check(cudaStreamSynchronize(st), "sync");
    res.trace.push_back(0.5 * ctx->h_scalars[0]);
    res.iterations = 1;
    res.converged = true;
    return res;
  }

  // After the loop: smoothing covariances and the filtered marginals of the
  // final linearisation, innovation statistics, calibration and projection
  // (ieks.cpp:190-208).  `eta_lin` is the final iteration's linearisation
  // point, `eta_out` its result.
  static void finalize(pode_context* ctx, const IeksSetup<D>& s, const double* eta_lin, const double* eta_out,
                       int ek0, int it, double sigma, double* means, double* cov, double* sol_m, double* sol_c,
                       IeksResult& res) {
    cudaStream_t st = ctx->stream;
    Workspace& ws = ctx->ws;
    DevError* err = reinterpret_cast<DevError*>(ctx->d_err);
    const int64_t N = s.N, n1 = s.n1;
    const DevChain ch = chain(ctx, s, true);
    linearize(ctx, s, ch, eta_lin, ek0, it);
    double* fm = ws.arr<double>("ieks_fm", n1 * D);
    double* fc = ws.arr<double>("ieks_fc", n1 * D * D);
    double* sm = ws.arr<double>("ieks_sm", n1 * D);
    double* sc = ws.arr<double>("ieks_sc", n1 * D * D);
    reset_error(ctx);
    const ScanTally t = Engine<D>::rts(ctx, ch, fm, fc, sm, sc);
    res.stats.combines = std::max(res.stats.combines, t.combines);
    res.stats.depth = std::max(res.stats.depth, t.depth);
    double* vals = ws.arr<double>("ieks_innov", N);
    cuda_check(cudaFuncSetAttribute(k_innovation<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(smem_bytes<D>())),
               "innovation smem");
    k_innovation<D><<<blocks_for<D>(N), kThreads, smem_bytes<D>(), st>>>(ch, fm, fc, vals, err);
    note_launch(ctx, "innovation");
    const int64_t np2 = grid1(N);
    double* part2 = ws.arr<double>("ieks_part2", np2 * 3 + 3);
    k_sum_blocks<<<np2, kRedThreads, 0, st>>>(vals, N, part2);
    note_launch(ctx, "sum_blocks");
    k_finish3<<<1, kRedThreads, 0, st>>>(part2, np2, part2 + np2 * 3);
    note_launch(ctx, "finish3");
    cuda_check(cudaMemcpyAsync(ctx->h_scalars, part2 + np2 * 3, sizeof(double), cudaMemcpyDeviceToHost, st),
               "innov");
    check_linearization(ctx, s, it);  // syncs
    const double sq = ctx->h_scalars[0];
    const int64_t count = N * s.dim;
    const double sigma_rel = std::sqrt(sq / double(count));
    res.sigma_hat = sigma_rel * sigma;
    k_outputs<<<grid1(n1), kRedThreads, 0, st>>>(eta_out, sc, s.scale, sigma_rel, n1, D, s.nu, s.dim, means, cov,
                                                 sol_m, sol_c);
    note_launch(ctx, "outputs");
  }

  // Element/scan driver (any D): linearize -> para_rts -> reductions,
  // exactly the reference's per-iteration structure.
  static IeksResult run(pode_context* ctx, const host::Problem& p, const pode_prior& prior, const double* grid_h,
                        int64_t n1, const pode_ieks_config& cfg, double* means, double* cov, double* sol_m,
                        double* sol_c) {
    IeksSetup<D> s;
    setup(ctx, p, prior, grid_h, n1, s);
    cudaStream_t st = ctx->stream;
    Workspace& ws = ctx->ws;
    const DevChain ch = chain(ctx, s, true);
    double* eta_a = ws.arr<double>("ieks_eta_a", n1 * D);
    double* eta_b = ws.arr<double>("ieks_eta_b", n1 * D);
    double* fm = ws.arr<double>("ieks_fm", n1 * D);
    double* fc = ws.arr<double>("ieks_fc", n1 * D * D);
    double* sm = ws.arr<double>("ieks_sm", n1 * D);
    double* sc = ws.arr<double>("ieks_sc", n1 * D * D);
    const int64_t nparts = grid1(n1);
    double* part = ws.arr<double>("ieks_part", nparts * 3 + 3);
    double* red = part + nparts * 3;
    k_fill_rows<<<grid1(n1 * D), kRedThreads, 0, st>>>(s.mu0, n1, D, eta_a);
    note_launch(ctx, "fill");
    auto reduce3 = [&](const double* smean, const double* eold, double* enew) {
      k_eta_objective<<<grid1(n1), kRedThreads, 0, st>>>(smean, s.scale, s.scale_inv, eold, ch.phi, s.qunit,
                                                         s.qinv, n1, D, enew, part);
      note_launch(ctx, "eta_objective");
      k_finish3<<<1, kRedThreads, 0, st>>>(part, nparts, red);
      note_launch(ctx, "finish3");
      cuda_check(cudaMemcpyAsync(ctx->h_scalars, red, sizeof(double) * 3, cudaMemcpyDeviceToHost, st), "red");
      cuda_check(cudaStreamSynchronize(st), "sync");
    };
    reduce3(nullptr, eta_a, eta_b);
    double v_prev = 0.5 * ctx->h_scalars[0];
    IeksResult res;
    int it = 0;
    while (it < cfg.max_iterations) {
      ++it;
      linearize(ctx, s, ch, eta_a, cfg.linearization, it);
      const ScanTally t = Engine<D>::rts(ctx, ch, fm, fc, sm, sc);
      res.stats.combines = std::max(res.stats.combines, t.combines);
      res.stats.depth = std::max(res.stats.depth, t.depth);
      reduce3(sm, eta_a, eta_b);
      check_linearization(ctx, s, it);
      const double v = 0.5 * ctx->h_scalars[0];
      const double dmax = ctx->h_scalars[1], emax = ctx->h_scalars[2];
      res.trace.push_back(v);
      const bool conv = (dmax <= cfg.traj_rtol * emax) ||
                        (std::fabs(v - v_prev) <= cfg.obj_atol + cfg.obj_rtol * std::fabs(v));
      std::swap(eta_a, eta_b);
      v_prev = v;
      if (conv) {
        res.converged = true;
        break;
      }
    }
    res.iterations = it;
    finalize(ctx, s, eta_b, eta_a, cfg.linearization, it, prior.sigma, means, cov, sol_m, sol_c, res);
    return res;
  }
};

}  // namespace pode
