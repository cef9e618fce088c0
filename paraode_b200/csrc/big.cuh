// Large-state fused IEKS engine (D > 16; Pleiades, d = 28, IWP(3): D = 112).
//
// One CTA per time chunk (~one per SM), the chunk's matrices in its own
// global-memory workspace (L2-resident) and every product on the FP64
// tensor pipe (big_la.cuh).  The algebra is that of the fused iteration
// (fast.cuh / lane.cuh) in covariance form — P = C C^T, Lambda = J J^T — so
// that each time step is a handful of dense contractions plus two Cholesky
// factorisations of SPD matrices (the predicted covariance P-, whose
// factor is the Pi_11 of make_smoothing_element, and the innovation
// covariance S, the Psi_11 of kf_update): the same Gaussians the
// reference's Householder trias produce (parallel.cpp:38-64, 112-135;
// sequential.cpp:30-67), whose factors it leaves unpinned (linalg.hpp:12-17;
// compare L L^T only).
//
// Per Gauss-Newton iteration:
//   A  (parallel)   fold each chunk into its aggregate (A, b, P, eta, Lambda)
//                   conditioned on the chunk's first state (EK1 linearisation
//                   on the fly, statespace.cpp:65-88 rescaled as ieks.cpp:160-164)
//   B  (one CTA)    the chunk-boundary filtered marginals, carried chunk to
//                   chunk: x_s | carry ~ N((I + P Lambda)^-1 (m + P eta),
//                   (I + P Lambda)^-1 P), then (A m_s + b, A P_s A^T + P_a) —
//                   the Gaussian-carry ⊗_f (parallel.cpp:67-100); with ~#SM
//                   chunks this chain is a few % of the iteration
//   C  (parallel)   filter through each chunk; smoothing elements
//                   E_k = P+ phi^T (P-)^-1, g_k = m+ - E_k phi m+
//                   (parallel.cpp:112-135), and the chunk's backward aggregate
//   D  (one CTA)    the smoothed means at the chunk boundaries
//   E  (parallel)   backward means, the new trajectory, the objective and the
//                   stopping maxima (ieks.cpp:49-77)
// Finalize: innovation statistics / sigma_hat (ieks.cpp:79-109), the
// smoothed covariances in Joseph form P^s_k = (I - E_k phi) P+_k (..)^T +
// E_k Q Q^T E_k^T + E_k P^s_{k+1} E_k^T (the ⊗_s covariance algebra,
// parallel.cpp:146-156), chunk aggregates chained like D, and the outputs
// (ieks.cpp:196-208) with cov_sqrt a pivoted-Cholesky factor of P^s.
//
// HBM layout: node-major, E_k (D x D) and g_k (D) per node, P+_k (D x D) in
// the finalize; the trajectory (N+1) x D row-major.
#pragma once

#include "big_la.cuh"
#include "fast.cuh"
#include "field.cuh"

namespace pode {
namespace big {

// Shared-memory step constants: node scales, the transition's binomial
// coefficients, the linearisation (f, Jacobian).
template <int D, int d>
struct StepSm {
  static constexpr int B = D / d;
  double tn[B], tni[B], tk[B], tki[B], ratio[B];
  double bin[B][B];
  double y[d], f[d], off[d];
  double jac[d * d];
  double red[kBW];
  int finite;
};

struct BigArgs {
  const double* grid;
  const double* eta;   // linearisation point, (padded + 1) x D row-major (node N at N * D)
  int64_t N;
  int L;
  int64_t nchunks;
  int ek0;
  DevProblem prob;
  DevError* err;
  const double* qq;    // sigma^2 Q_bar Q_bar^T (D x D)
  const double* q1u;   // unit-diffusion Q_bar block (B x B lower), for the objective
  const double* m0;    // T_0^-1 mu_0
  double* ws;          // per-chunk workspace
  int64_t ws_stride;   // doubles per chunk
  long long* phases;   // PODE_BIG_PHASES: per-phase clock64 totals of CTA 0 (debug; nullptr = off)
};

// Phase timer of CTA 0, thread 0 (between CTA barriers, so a phase's time
// is the CTA's).
struct PhaseClock {
  long long* out = nullptr;
  long long t = 0;
  __device__ explicit PhaseClock(long long* o) {
#ifdef __CUDA_ARCH__
    out = (blockIdx.x == 0 && threadIdx.x == 0) ? o : nullptr;
    t = clock64();
#endif
  }
  __device__ void mark(int i) {
#ifdef __CUDA_ARCH__
    if (out) {
      const long long n = clock64();
      out[i] += n - t;
      t = n;
    }
#endif
  }
};

template <int D, int d>
struct Big {
  static constexpr int B = D / d;
  static constexpr int q = B - 1;
  using Sm = StepSm<D, d>;

  // node scales T_n (ieks.cpp:28-33, incoming step; node 0 uses step 0)
  __device__ static void taus(const double* grid, int64_t n, double* t, double* ti) {
    const double h = (n == 0) ? grid[1] - grid[0] : grid[n] - grid[n - 1];
    const double rh = sqrt(h);
    double fact = 1.0;
    for (int i = q; i >= 0; --i) {
      const int k = q - i;
      if (k > 0) fact *= k;
      t[i] = rh * pow(h, double(k)) / fact;
      ti[i] = 1.0 / t[i];
    }
  }
  __device__ static double binom(int n, int k) {
    double num = 1.0, den = 1.0;
    for (int t = 0; t < k; ++t) {
      num *= double(n - t);
      den *= double(t + 1);
    }
    return num / den;
  }
  // step k -> k+1 constants into smem (thread 0), then sync
  __device__ static void step_consts(Sm& s, const double* grid, int64_t k) {
    if (threadIdx.x == 0) {
      taus(grid, k, s.tk, s.tki);
      taus(grid, k + 1, s.tn, s.tni);
      for (int i = 0; i < B; ++i) s.ratio[i] = s.tk[i] * s.tni[i];
      for (int a = 0; a < B; ++a)
        for (int i = 0; i < B; ++i) s.bin[a][i] = (i >= a) ? binom(q - a, i - a) * s.ratio[i] : 0.0;
    }
    __syncthreads();
  }
  // The transition acts blockwise (B x B upper-triangular bin per state
  // component), so every product below is a set of independent block tasks;
  // each thread keeps kU tasks (kU * B loads) in flight.  Strides lx / ly
  // address global or shared operands alike.  Y != X throughout.
  static constexpr int kU = 4;
  // Y = Phi X (rows): task (blk, column j)
  __device__ static void phi_rows(const Sm& s, const double* X, int lx, double* Y, int ly) {
    constexpr int T = d * D;
    for (int base = threadIdx.x; base < T; base += kU * kBT) {
      double x[kU][B];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int t = base + u * kBT, blk = t / D, j = t - blk * D;
#pragma unroll
        for (int i = 0; i < B; ++i) x[u][i] = t < T ? X[(blk * B + i) * lx + j] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int t = base + u * kBT, blk = t / D, j = t - blk * D;
        if (t < T) {
#pragma unroll
          for (int a = 0; a < B; ++a) {
            double acc = 0.0;
#pragma unroll
            for (int i = a; i < B; ++i) acc = fma(s.bin[a][i], x[u][i], acc);
            Y[(blk * B + a) * ly + j] = acc;
          }
        }
      }
    }
    __syncthreads();
  }
  // Y = Phi X + M on and below the diagonal, mirrored above (M: D x D,
  // stride D): the predicted covariance phi (P phi^T) + Q Q^T, exactly
  // symmetric (the two triangles of phi P phi^T would otherwise differ by
  // the association order); also written to Pg (stride D) when given.
  __device__ static void phi_rows_sym(const Sm& s, const double* X, int lx, const double* M, double* Y, int ly,
                                      double* Pg = nullptr) {
    constexpr int T = d * D;
    for (int base = threadIdx.x; base < T; base += kU * kBT) {
      double x[kU][B], mv[kU][B];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int t = base + u * kBT, blk = t / D, j = t - blk * D;
#pragma unroll
        for (int i = 0; i < B; ++i) {
          const bool lo = t < T && blk * B + i >= j;
          x[u][i] = lo ? X[(blk * B + i) * lx + j] : 0.0;
          mv[u][i] = lo ? M[(blk * B + i) * D + j] : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int t = base + u * kBT, blk = t / D, j = t - blk * D;
#pragma unroll
        for (int a = 0; a < B; ++a) {
          const int r = blk * B + a;
          if (t < T && r >= j) {
            double acc = 0.0;
#pragma unroll
            for (int i = a; i < B; ++i) acc = fma(s.bin[a][i], x[u][i], acc);
            acc += mv[u][a];
            Y[r * ly + j] = acc;
            Y[j * ly + r] = acc;
            if (Pg) {
              Pg[r * D + j] = acc;
              Pg[j * D + r] = acc;
            }
          }
        }
      }
    }
    __syncthreads();
  }
  // Y = X Phi^T (kT) or Y = X Phi (!kT): task (row r, blk)
  template <bool kT>
  __device__ static void phi_colwise(const Sm& s, const double* X, int lx, double* Y, int ly) {
    constexpr int T = D * d;
    for (int base = threadIdx.x; base < T; base += kU * kBT) {
      double x[kU][B];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int t = base + u * kBT, r = t / d, blk = t - r * d;
#pragma unroll
        for (int i = 0; i < B; ++i) x[u][i] = t < T ? X[r * lx + blk * B + i] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int t = base + u * kBT, r = t / d, blk = t - r * d;
        if (t < T) {
#pragma unroll
          for (int c = 0; c < B; ++c) {
            double acc = 0.0;
            if (kT) {  // Y[r][blk B + c] = sum_{i >= c} bin[c][i] X[r][blk B + i]
#pragma unroll
              for (int i = c; i < B; ++i) acc = fma(s.bin[c][i], x[u][i], acc);
            } else {   // Y[r][blk B + c] = sum_{i <= c} X[r][blk B + i] bin[i][c]
#pragma unroll
              for (int i = 0; i <= c; ++i) acc = fma(x[u][i], s.bin[i][c], acc);
            }
            Y[r * ly + blk * B + c] = acc;
          }
        }
      }
    }
    __syncthreads();
  }
  __device__ static void phi_cols(const Sm& s, const double* X, int lx, double* Y, int ly) {
    phi_colwise<true>(s, X, lx, Y, ly);
  }
  __device__ static void phi_right(const Sm& s, const double* X, int lx, double* Y, int ly) {
    phi_colwise<false>(s, X, lx, Y, ly);
  }
  __device__ static void phi_vec(const Sm& s, const double* x, double* y) {
    for (int r = threadIdx.x; r < D; r += kBT) {
      const int blk = r / B, a = r - blk * B;
      double acc = 0.0;
      for (int i = a; i < B; ++i) acc = fma(s.bin[a][i], x[blk * B + i], acc);
      y[r] = acc;
    }
    __syncthreads();
  }
  // EK1 / EK0 linearisation at eta[k+1] (statespace.cpp:65-103).  Pleiades
  // (the only registered field with d = 28) is evaluated body-parallel (one
  // thread per body owns its two acceleration rows of the Jacobian, the same
  // summation order as field.cuh); other fields on thread 0.
  __device__ static void linearize(Sm& s, const BigArgs& a, int64_t k1) {
    if (a.prob.kind == 5 && d == 28) {
      constexpr int NB = 7;
      for (int i = threadIdx.x; i < d * d; i += kBT) s.jac[i] = 0.0;
      if (threadIdx.x < d) s.y[threadIdx.x] = a.eta[k1 * D + threadIdx.x * B];
      if (threadIdx.x == 0) s.finite = 1;
      __syncthreads();
      const int t = threadIdx.x;
      if (t < NB) {  // body i: f[2NB+i], f[3NB+i] and Jacobian rows 2NB+i, 3NB+i
        const int i = t;
        double ax = 0.0, ay = 0.0;
        double* rx = s.jac + (2 * NB + i) * d;
        double* ry = s.jac + (3 * NB + i) * d;
        for (int j = 0; j < NB; ++j) {
          if (j == i) continue;
          const double dx = s.y[j] - s.y[i], dy = s.y[NB + j] - s.y[NB + i];
          const double r2 = dx * dx + dy * dy;
          const double r = sqrt(r2);
          const double r3 = r2 * r, r5 = r3 * r2;
          const double mj = static_cast<double>(j + 1);
          ax += (mj * dx) / r3;
          ay += (mj * dy) / r3;
          const double dxx = mj * (1.0 / r3 - 3.0 * dx * dx / r5);
          const double dxy = mj * (-3.0 * dx * dy / r5);
          const double dyy = mj * (1.0 / r3 - 3.0 * dy * dy / r5);
          rx[j] += dxx;
          rx[i] -= dxx;
          rx[NB + j] += dxy;
          rx[NB + i] -= dxy;
          ry[j] += dxy;
          ry[i] -= dxy;
          ry[NB + j] += dyy;
          ry[NB + i] -= dyy;
        }
        s.f[2 * NB + i] = ax;
        s.f[3 * NB + i] = ay;
      } else if (t < 2 * NB) {  // positions' rows: x_i' = vx_i, y_i' = vy_i
        const int i = t - NB;
        s.f[i] = s.y[2 * NB + i];
        s.f[NB + i] = s.y[3 * NB + i];
        s.jac[i * d + 2 * NB + i] = 1.0;
        s.jac[(NB + i) * d + 3 * NB + i] = 1.0;
      }
      __syncthreads();
      if (t < d) {
        bool fin = isfinite(s.f[t]);
        double jy = 0.0;
        for (int j = 0; j < d; ++j) {
          if (!a.ek0) fin &= isfinite(s.jac[t * d + j]);
          jy += s.jac[t * d + j] * s.y[j];
        }
        s.off[t] = a.ek0 ? s.f[t] : s.f[t] - jy;
        if (!fin) s.finite = 0;
      }
      __syncthreads();
      if (a.ek0) {
        for (int i = threadIdx.x; i < d * d; i += kBT) s.jac[i] = 0.0;
        __syncthreads();
      }
      return;
    }
    if (threadIdx.x == 0) {
      for (int j = 0; j < d; ++j) s.y[j] = a.eta[k1 * D + j * B];
      double jac[d * d];
      eval_field<d>(a.prob, s.y, s.f, jac, a.prob.kind == 7 ? a.grid[k1] : 0.0);
      bool fin = true;
      for (int i = 0; i < d; ++i) fin &= isfinite(s.f[i]);
      for (int i = 0; i < d * d; ++i) {
        if (!a.ek0) fin &= isfinite(jac[i]);
        s.jac[i] = a.ek0 ? 0.0 : jac[i];
      }
      for (int i = 0; i < d; ++i) {
        double jy = 0.0;
        for (int j = 0; j < d; ++j) jy += s.jac[i * d + j] * s.y[j];
        s.off[i] = a.ek0 ? s.f[i] : s.f[i] - jy;
      }
      s.finite = fin ? 1 : 0;
    }
    __syncthreads();
  }
  // HX (d x D) = H_bar X; H_bar row i = t1 e_{iB+1} - t0 sum_c jac[i][c] e_{cB}
  __device__ static void h_rows(const Sm& s, const double* X, double* HX, int lx = D) {
    const double t0 = s.tn[0], t1 = s.tn[1];
    for (int i = threadIdx.x >> 5; i < d; i += kBW)
      for (int j = threadIdx.x & 31; j < D; j += 32) {
        double acc = (1.0 * t1) * X[(i * B + 1) * lx + j];
        for (int c = 0; c < d; ++c) acc = fma((-s.jac[i * d + c]) * t0, X[(c * B) * lx + j], acc);
        HX[i * D + j] = acc;
      }
    __syncthreads();
  }
  // XH (n x d) = X H_bar^T for X with n rows of D
  __device__ static void h_cols(const Sm& s, int n, const double* X, double* XH, int lx = D, int lo = d) {
    const double t0 = s.tn[0], t1 = s.tn[1];
    for (int idx = threadIdx.x; idx < n * d; idx += kBT) {
      const int r = idx / d, i = idx - (idx / d) * d;
      double acc = (1.0 * t1) * X[r * lx + i * B + 1];
      for (int c = 0; c < d; ++c) acc = fma((-s.jac[i * d + c]) * t0, X[r * lx + c * B], acc);
      XH[r * lo + i] = acc;
    }
    __syncthreads();
  }
  // HX (d x D, stride lo) = H_bar X for X in shared memory (stride lx): the
  // Jacobian part as one DMMA product (jac x the rows cB of X), then the
  // t1 rows iB+1
  __device__ static void h_rows_smem(const Sm& s, const double* X, int lx, double* HX, int lo) {
    gemm_core<false>(d, D, d, -s.tn[0], s.jac, d, X, B * lx, 0.0, HX, lo);
    const double t1 = s.tn[1];
    for (int idx = threadIdx.x; idx < d * D; idx += kBT) {
      const int i = idx / D, j = idx - (idx / D) * D;
      HX[i * lo + j] = fma(t1, X[(i * B + 1) * lx + j], HX[i * lo + j]);
    }
    __syncthreads();
  }
  // z = H_bar v - offset (d)
  __device__ static void h_vec(const Sm& s, const double* v, double* z) {
    const double t0 = s.tn[0], t1 = s.tn[1];
    for (int i = threadIdx.x; i < d; i += kBT) {
      double acc = (1.0 * t1) * v[i * B + 1];
      for (int c = 0; c < d; ++c) acc = fma((-s.jac[i * d + c]) * t0, v[c * B], acc);
      z[i] = acc - s.off[i];
    }
    __syncthreads();
  }
};

// Dynamic shared memory of the kernels: b1 (offset 0: the staging area of
// the big_la.cuh routines and of cov_update_parts) and b2 (a resident D x D
// matrix, stride smem_ld(D)) after it; the chain kernels' LU needs
// D smem_ld(2 D + 1).
template <int D, int d = 28>
constexpr int b2_offset() {
  constexpr int ls = smem_ld(D), scratch = d * smem_ld(D) + 2 * d * smem_ld(d);
  return D * ls > scratch ? D * ls : scratch;
}
template <int D>
constexpr size_t big_smem_bytes(bool) {
  constexpr size_t two = size_t(b2_offset<D>()) + size_t(D) * smem_ld(D), lu = size_t(D) * smem_ld(2 * D + 1);
  return sizeof(double) * (two > lu ? two : lu);
}

// Per-chunk workspace slots (doubles), see the kernels.
template <int D, int d>
struct Slots {
  static constexpr int64_t DD = int64_t(D) * D;
  static constexpr int64_t dD = int64_t(d) * D;
  static constexpr int64_t kMats = 8;  // M0..M7
  static constexpr int64_t kSmall = 6 * dD + 2 * int64_t(d) * d + 8 * D + 4 * d;
  static constexpr int64_t kStride = kMats * DD + kSmall;
};

// The measurement update of one step in covariance form (kf_update with
// R = 0, sequential.cpp:41-67): from Pm (predicted) produce W = S^-1 H Pm
// (d x D) and Sinv (d x d); P+ = Pm - W^T W, K = W^T S^-1.
template <int D, int d>
__device__ bool cov_update_parts(StepSm<D, d>& s, const double* Pm, int lp, double* Sinv, double* W) {
  using G = Big<D, d>;
  constexpr int lh = smem_ld(D), l2 = smem_ld(d);
  double* hp = dyn_smem();         // H Pm (d x D), then W = S^-1 H Pm
  double* ss = hp + d * lh;        // S S^T = H Pm H^T (d x d), then S
  double* si = ss + d * l2;        // I, then S^-1
  G::h_rows_smem(s, Pm, lp, hp, lh);
  G::h_cols(s, d, hp, ss, lh, l2);
  for (int idx = threadIdx.x; idx < d * d; idx += kBT) si[(idx / d) * l2 + idx % d] = (idx / d == idx % d) ? 1.0 : 0.0;
  const bool sing = potrf_smem(d, ss, l2, s.red);  // (syncs)
  trsm_left_lower(d, D, ss, l2, hp, lh);           // W = S^-1 H Pm
  trsm_left_lower(d, d, ss, l2, si, l2);           // S^-1
  stage(d, D, hp, lh, W, D);
  stage(d, d, si, l2, Sinv, d);
  return sing;
}

// ------------------------------------------------------------- pass A ---
template <int D, int d>
__global__ void __launch_bounds__(kBT) k_big_fwd_reduce(BigArgs a, double* agg, int first) {
  using G = Big<D, d>;
  using S = Slots<D, d>;
  __shared__ StepSm<D, d> s;
  const int64_t c = blockIdx.x;
  const int64_t s0 = c * a.L, e = min(a.N, s0 + a.L);
  double* w = a.ws + c * a.ws_stride;
  double *Am = w, *Lam = w + 2 * S::DD, *Anew = w + 5 * S::DD;
  double* sm = w + S::kMats * S::DD;
  double *W = sm + S::dD, *HA = sm + 2 * S::dD, *Ub = sm + 3 * S::dD;
  double *Sd = sm + 6 * S::dD, *Sinv = Sd + d * d, *bv = Sinv + d * d, *bm = bv + D, *eta = bm + D, *u = eta + D,
         *ub = u + d;
  // P lives in shared memory (b2) for the whole chunk; b1 is the scratch
  // of the products (P phi^T, then the staging of the small solves).
  constexpr int ls = smem_ld(D);
  double* b1 = dyn_smem();
  double* b2 = b1 + b2_offset<D, d>();
  const bool chunk0 = c == 0 && first;
  for (int idx = threadIdx.x; idx < D * D; idx += kBT) {
    const int r = idx / D, j = idx - (idx / D) * D;
    Am[idx] = (!chunk0 && r == j) ? 1.0 : 0.0;
    b2[r * ls + j] = 0.0;
    Lam[idx] = 0.0;
  }
  for (int r = threadIdx.x; r < D; r += kBT) {
    bv[r] = chunk0 ? a.m0[r] : 0.0;
    eta[r] = 0.0;
  }
  __syncthreads();
  bool bad_sing = false;
  int64_t bad_lin = -1;
  for (int64_t k = s0; k < e; ++k) {
    G::step_consts(s, a.grid, k);
    G::phi_rows(s, Am, D, Anew, D);  // A- = phi A
    G::phi_vec(s, bv, bm);           // b- = phi b
    G::phi_cols(s, b2, ls, b1, ls);  // P phi^T
    G::phi_rows_sym(s, b1, ls, a.qq, b2, ls);  // Pm = phi P phi^T + Q Q^T
    G::linearize(s, a, k + 1);
    if (!s.finite && bad_lin < 0) bad_lin = k + 1;
    bad_sing |= cov_update_parts<D, d>(s, b2, ls, Sinv, W);  // scratch: b1
    G::h_rows(s, Anew, HA);  // H A-
    G::h_vec(s, bm, u);      // H b- - offset
    gemm<false, false>(d, D, d, 1.0, Sinv, d, HA, D, 0.0, Ub, D);  // Ubar = S^-1 H A-
    gemv<false>(d, d, 1.0, Sinv, d, u, 0.0, ub);                    // ubar = S^-1 u
    // A = A- - W^T Ubar; b = b- - W^T ubar; P = Pm - W^T W;
    // eta -= Ubar^T ubar; Lambda += Ubar^T Ubar
    gemm<true, false>(D, D, d, -1.0, W, D, Ub, D, 1.0, Anew, D);
    gemv<true>(D, d, -1.0, W, D, ub, 1.0, bm);
    gemm<true, false>(D, D, d, -1.0, W, D, W, D, 1.0, b2, ls);  // (P stays symmetric to rounding; the chains re-symmetrise)
    gemv<true>(D, d, -1.0, Ub, D, ub, 1.0, eta);
    gemm<true, false>(D, D, d, 1.0, Ub, D, Ub, D, 1.0, Lam, D);
    double* t = Am;  // rotate buffers: A <- Anew
    Am = Anew;
    Anew = t;
    copy(D, bm, bv);
  }
  if (threadIdx.x == 0) {
    if (bad_lin >= 0) raise_error(a.err, bad_lin, kErrLinearization);
    if (bad_sing) raise_error(a.err, s0, kErrSingular);
  }
  // aggregate c: A, P, Lambda (D x D each), b, eta
  double* o = agg + c * (3 * S::DD + 2 * D);
  for (int idx = threadIdx.x; idx < D * D; idx += kBT) {
    o[idx] = Am[idx];
    o[S::DD + idx] = b2[(idx / D) * ls + idx % D];
    o[2 * S::DD + idx] = Lam[idx];
  }
  for (int r = threadIdx.x; r < D; r += kBT) {
    o[3 * S::DD + r] = bv[r];
    o[3 * S::DD + D + r] = eta[r];
  }
}

// ---------------------------------------------------- pass B (one CTA) ---
// prefix[c] = (m, P) of the filtered marginal at the END of chunk c.
template <int D, int d>
__global__ void __launch_bounds__(kBT) k_big_chain_fwd(BigArgs a, const double* agg, double* prefix, double* scratch,
                                                       int first, const double* carry) {
  using S = Slots<D, d>;
  double *M = scratch, *X = scratch + S::DD, *T = X + int64_t(D) * (D + 1);
  double* m = T + S::DD;
  const int64_t stride = 3 * S::DD + 2 * D;
  // chunk 0: its aggregate absorbed the initial distribution (A = 0), or (a
  // shard) starts from the carry
  for (int64_t c = 0; c < a.nchunks; ++c) {
    const double* g = agg + c * stride;
    const double *Ac = g, *Pa = g + S::DD, *Lam = g + 2 * S::DD, *bc = g + 3 * S::DD, *ec = bc + D;
    double* out = prefix + c * (S::DD + D);  // m (D) then P (D x D)
    if (c == 0 && first) {
      copy(D, bc, out);
      copy(D * D, Pa, out + D);
      continue;
    }
    const double* pm = (c == 0) ? carry : prefix + (c - 1) * (S::DD + D);
    const double* Pcg = pm + D;
    // M = I + Pc Lambda; X = [Pc | m + Pc eta]
    gemm<false, false>(D, D, D, 1.0, Pcg, D, Lam, D, 0.0, M, D);
    gemv<false>(D, D, 1.0, Pcg, D, ec, 0.0, m);
    for (int idx = threadIdx.x; idx < D * (D + 1); idx += kBT) {
      const int r = idx / (D + 1), j = idx - r * (D + 1);
      X[idx] = j < D ? Pcg[r * D + j] : m[r] + pm[r];
      if (j == r) M[r * D + r] += 1.0;
    }
    __syncthreads();
    lu_solve(D, M, D, D + 1, X, D + 1);  // X = [P_s | m_s]
    // out.m = A m_s + b; out.P = A P_s A^T + Pa
    for (int r = threadIdx.x; r < D; r += kBT) m[r] = X[r * (D + 1) + D];
    __syncthreads();
    copy(D, bc, out);
    gemv<false>(D, D, 1.0, Ac, D, m, 1.0, out);
    gemm<false, false>(D, D, D, 1.0, Ac, D, X, D + 1, 0.0, T, D);          // A P_s
    copy(D * D, Pa, out + D);
    gemm<false, true>(D, D, D, 1.0, T, D, Ac, D, 1.0, out + D, D);         // + A P_s A^T
    symmetrize(D, out + D, D);
  }
}

// ------------------------------------------------------------- pass C ---
// kFinal: also stores P+_k (filtered covariance at every node, pf) and the
// whitened innovations sum (innov, one partial per chunk).
template <int D, int d, bool kFinal>
__global__ void __launch_bounds__(kBT) k_big_fwd_down(BigArgs a, const double* prefix, double* E_out, double* g_out,
                                                      double* g_term, double* bagg, double* pf, double* pterm,
                                                      double* innov, int first, int last, const double* carry) {
  using G = Big<D, d>;
  using S = Slots<D, d>;
  __shared__ StepSm<D, d> s;
  const int64_t c = blockIdx.x;
  const int64_t s0 = c * a.L, e = min(a.N, s0 + a.L);
  double* w = a.ws + c * a.ws_stride;
  double *Pm = w + 2 * S::DD, *EA = w + 6 * S::DD, *EAn = w + 7 * S::DD;
  double* sm = w + S::kMats * S::DD;
  double* W = sm + S::dD;
  double *Sd = sm + 6 * S::dD, *Sinv = Sd + d * d, *m = Sinv + d * d, *mm = m + D, *gk = mm + D, *gA = gk + D,
         *z = gA + D, *zb = z + d;
  // Two shared-memory D x D matrices carry the step: P (filtered covariance)
  // lives in b2 between steps.  Per step: b1 <- Y = P phi^T; b2 <- Pm =
  // phi Y + Q Q^T (also to global); b2 <- L (Pm = L L^T); b1 <- Y L^-T L^-1
  // = E; b2 <- Pm (from global) for the measurement update; b2 <- P+.
  constexpr int ls = smem_ld(D);
  double* b1 = dyn_smem();
  double* b2 = b1 + b2_offset<D, d>();
  const double* pin = (c == 0) ? (first ? nullptr : carry) : prefix + (c - 1) * (S::DD + D);
  if (pin) {
    stage(D, D, pin + D, D, b2, ls);
  } else {
    for (int idx = threadIdx.x; idx < D * D; idx += kBT) b2[(idx / D) * ls + idx % D] = 0.0;
  }
  for (int r = threadIdx.x; r < D; r += kBT) m[r] = pin ? pin[r] : a.m0[r];
  __syncthreads();
  bool bad_sing = false;
  int64_t bad_lin = -1;
  double inn = 0.0;
  for (int64_t k = s0; k < e; ++k) {
    PhaseClock pc(a.phases);
    G::step_consts(s, a.grid, k);
    if constexpr (kFinal) stage(D, D, b2, ls, pf + k * S::DD, D);
    pc.mark(0);
    G::phi_cols(s, b2, ls, b1, ls);
    G::phi_rows_sym(s, b1, ls, a.qq, b2, ls, Pm);
    pc.mark(1);
    bad_sing |= potrf_smem(D, b2, ls, s.red);
    pc.mark(2);
    trsm_right_lower_t(D, D, b2, ls, b1, ls);
    pc.mark(3);
    trsm_right_lower_n(D, D, b2, ls, b1, ls);
    pc.mark(4);
    double* Ek = E_out + k * S::DD;
    stage(D, D, b1, ls, Ek, D);
    pc.mark(5);
    G::phi_vec(s, m, mm);                                              // m- = phi m
    gemv<false>(D, D, -1.0, b1, ls, mm, 0.0, gk);                      // -E m-
    for (int r = threadIdx.x; r < D; r += kBT) {
      gk[r] += m[r];                                                   // g = m - E phi m
      g_out[k * D + r] = gk[r];
    }
    __syncthreads();
    pc.mark(6);
    if constexpr (!kFinal) {
      // backward aggregate (E, g) <- (E E_k, E g_k + g) (⊗_s on means)
      if (k == s0) {
        stage(D, D, b1, ls, EA, D);
        copy(D, gk, gA);
      } else {
        gemv<false>(D, D, 1.0, EA, D, gk, 1.0, gA);
        gemm_core<false>(D, D, D, 1.0, EA, D, b1, ls, 0.0, EAn, D);
        double* t = EA;
        EA = EAn;
        EAn = t;
      }
    }
    pc.mark(7);
    // measurement update at node k+1
    G::linearize(s, a, k + 1);
    if (!s.finite && bad_lin < 0) bad_lin = k + 1;
    stage(D, D, Pm, D, b2, ls);
    pc.mark(8);
    bad_sing |= cov_update_parts<D, d>(s, b2, ls, Sinv, W);  // scratch: b1
    pc.mark(9);
    G::h_vec(s, mm, z);                             // H m- - offset
    gemv<false>(d, d, 1.0, Sinv, d, z, 0.0, zb);    // S^-1 z
    if constexpr (kFinal) {
      if (threadIdx.x == 0)
        for (int i = 0; i < d; ++i) inn = fma(zb[i], zb[i], inn);
    }
    copy(D, mm, m);
    gemv<true>(D, d, -1.0, W, D, zb, 1.0, m);       // m+ = m- - W^T S^-1 z
    gemm<true, false>(D, D, d, -1.0, W, D, W, D, 1.0, b2, ls);  // P+ = Pm - W^T W (staging: b1)
    pc.mark(10);
  }
  if (e == a.N) {  // terminal node N: E = 0, g = m_f(N)
    copy(D, m, g_term);
    if constexpr (kFinal) stage(D, D, b2, ls, pterm, D);
  }
  if constexpr (!kFinal) {
    const bool term = e == a.N && last;
    double* ob = bagg + c * (S::DD + D);
    if (term) gemv<false>(D, D, 1.0, EA, D, m, 1.0, gA);
    for (int idx = threadIdx.x; idx < D * D; idx += kBT) ob[idx] = term ? 0.0 : EA[idx];
    for (int r = threadIdx.x; r < D; r += kBT) ob[S::DD + r] = gA[r];
  }
  if (threadIdx.x == 0) {
    if (kFinal) {  // the k_finish3 partial layout (sum, 0, 0)
      innov[c * 3 + 0] = inn;
      innov[c * 3 + 1] = 0.0;
      innov[c * 3 + 2] = 0.0;
    }
    if (bad_lin >= 0) raise_error(a.err, bad_lin, kErrLinearization);
    if (bad_sing) raise_error(a.err, s0, kErrSingular);
  }
}

// ---------------------------------------------------- pass D (one CTA) ---
// suffix[c] = smoothed mean at the start node of chunk c (the last chunk's
// aggregate absorbed the terminal element).
template <int D>
__global__ void __launch_bounds__(kBT) k_big_chain_bwd(int64_t nc, const double* bagg, double* suffix,
                                                       const double* right) {
  constexpr int64_t DD = int64_t(D) * D;
  for (int64_t c = nc - 1; c >= 0; --c) {
    const double* g = bagg + c * (DD + D);
    const double* nxt = (c == nc - 1) ? right : suffix + (c + 1) * D;
    for (int i = threadIdx.x; i < D; i += kBT) {
      double acc = g[DD + i];
      if (nxt)
        for (int k = 0; k < D; ++k) acc = fma(g[i * D + k], nxt[k], acc);
      suffix[c * D + i] = acc;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------- pass E ---
// Backward means, new trajectory (original coordinates), objective terms
// (unit-diffusion metric, block-diagonal Q_bar: one thread per block) and
// stopping maxima; one (obj, dmax, emax) partial per chunk.
template <int D, int d, bool kInitial>
__global__ void __launch_bounds__(kBT) k_big_bwd_down(BigArgs a, const double* E_in, const double* g_in,
                                                      const double* g_term, const double* suffix,
                                                      const double* eta_old, double* eta_new, double* part, int last) {
  using G = Big<D, d>;
  constexpr int B = D / d;
  __shared__ double mu[D], nm[D], bar_next[D], bar[D], pb[D];
  __shared__ double tk[B], tki[B], tn[B], ratio[B], bin[B][B], red[kBW];
  const int64_t c = blockIdx.x;
  const int64_t s0 = c * a.L, e = min(a.N, s0 + a.L);
  const bool lastc = c == a.nchunks - 1;
  double obj = 0.0, dmax = 0.0, emax = 0.0;
  if (threadIdx.x == 0) G::taus(a.grid, e, tn, tki);  // tki: T_e^-1 here
  __syncthreads();
  for (int r = threadIdx.x; r < D; r += kBT) {
    const double old_e = eta_old[e * D + r];
    double eta_e;
    if (kInitial) {
      eta_e = old_e;
      mu[r] = 0.0;
    } else {
      mu[r] = lastc ? g_term[r] : suffix[(c + 1) * D + r];
      eta_e = tn[r % B] * mu[r];
    }
    if (lastc) {
      if (!kInitial) eta_new[e * D + r] = eta_e;
      if (last) {
        dmax = fmax(dmax, fabs(eta_e - old_e));
        emax = fmax(emax, fabs(eta_e));
      }
    }
    bar_next[r] = tki[r % B] * eta_e;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < B; ++i) tn[i] = tki[i];  // T_{k+1}^-1
  __syncthreads();
  for (int64_t k = e - 1; k >= s0; --k) {
    if (threadIdx.x == 0) {
      G::taus(a.grid, k, tk, tki);
      for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tn[i];
      for (int aa = 0; aa < B; ++aa)
        for (int i = 0; i < B; ++i) bin[aa][i] = (i >= aa) ? G::binom(B - 1 - aa, i - aa) * ratio[i] : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < D; r += kBT) {
      const double oldk = eta_old[k * D + r];
      double etak;
      if (kInitial) {
        etak = oldk;
      } else {
        double acc = g_in[k * D + r];
        const double* Er = E_in + (k * D + r) * D;
        for (int j = 0; j < D; ++j) acc = fma(Er[j], mu[j], acc);
        nm[r] = acc;
        etak = tk[r % B] * acc;
        eta_new[k * D + r] = etak;
      }
      dmax = fmax(dmax, fabs(etak - oldk));
      emax = fmax(emax, fabs(etak));
      bar[r] = tki[r % B] * etak;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < D; r += kBT) {
      const int blk = r / B, aa = r - blk * B;
      double acc = 0.0;
      for (int i = aa; i < B; ++i) acc = fma(bin[aa][i], bar[blk * B + i], acc);
      pb[r] = bar_next[r] - acc;
      if (!kInitial) mu[r] = nm[r];
    }
    __syncthreads();
    // || Qunit^-1/2 (bar_{k+1} - phi bar_k) ||^2, Q_bar = I_d (x) Q1: one block per thread
    for (int blk = threadIdx.x; blk < d; blk += kBT) {
      double w[B];
      for (int i = 0; i < B; ++i) {
        double acc = pb[blk * B + i];
        for (int k2 = 0; k2 < i; ++k2) acc = fma(-a.q1u[i * B + k2], w[k2], acc);
        w[i] = acc / a.q1u[i * B + i];
        obj = fma(w[i], w[i], obj);
      }
    }
    for (int r = threadIdx.x; r < D; r += kBT) bar_next[r] = bar[r];
    if (threadIdx.x == 0)
      for (int i = 0; i < B; ++i) tn[i] = tki[i];
    __syncthreads();
  }
  obj = block_sum(obj, red);
  dmax = block_max(dmax, red);
  emax = block_max(emax, red);
  if (threadIdx.x == 0) {
    part[c * 3 + 0] = obj;
    part[c * 3 + 1] = dmax;
    part[c * 3 + 2] = emax;
  }
}

// ------------------------------------------------- finalize (once) ---
// M1_k = (I - E_k phi) P+_k (I - E_k phi)^T + E_k Q Q^T E_k^T: the
// covariance of the smoothing element at node k (Joseph form).
// M = (I - E phi) P+ (I - E phi)^T (T1, T2 scratch; all D x D, stride D).
template <int D, int d>
__device__ void smooth_joseph(StepSm<D, d>& s, const double* Ek, const double* Pf, double* T1, double* T2,
                              double* M) {
  using G = Big<D, d>;
  G::phi_right(s, Ek, D, T1, D);  // E phi  (phi_k = node k -> k+1)
  axpby_eye(D, -1.0, T1, 0.0, nullptr, 1.0, T1);
  gemm<false, false>(D, D, D, 1.0, T1, D, Pf, D, 0.0, T2, D);   // (I - E phi) P+
  gemm<false, true>(D, D, D, 1.0, T2, D, T1, D, 0.0, M, D);     // .. (I - E phi)^T
}

// F2: per chunk the smoothing-covariance aggregate (Eagg, Lagg): P^s(s) =
// Eagg P^s(e) Eagg^T + Lagg (the last chunk absorbs P^s(N) = P+(N)).
template <int D, int d>
__global__ void __launch_bounds__(kBT) k_big_fin_fold(BigArgs a, const double* E_in, const double* pf,
                                                      const double* pterm, double* sagg, int last) {
  using G = Big<D, d>;
  using S = Slots<D, d>;
  __shared__ StepSm<D, d> s;
  const int64_t c = blockIdx.x;
  const int64_t s0 = c * a.L, e = min(a.N, s0 + a.L);
  const bool term = c == a.nchunks - 1 && last;
  double* w = a.ws + c * a.ws_stride;
  double *EA = w, *LA = w + S::DD, *M1 = w + 2 * S::DD, *T1 = w + 3 * S::DD, *T2 = w + 4 * S::DD,
         *EAn = w + 5 * S::DD, *LAn = w + 6 * S::DD;
  for (int idx = threadIdx.x; idx < D * D; idx += kBT) {
    EA[idx] = (!term && idx / D == idx % D) ? 1.0 : 0.0;
    LA[idx] = term ? pterm[idx] : 0.0;
  }
  __syncthreads();
  for (int64_t k = e - 1; k >= s0; --k) {
    G::step_consts(s, a.grid, k);
    const double* Ek = E_in + k * S::DD;
    // Lagg <- (I - E phi) P+ (I - E phi)^T + E (Q Q^T + Lagg) E^T
    smooth_joseph<D, d>(s, Ek, pf + k * S::DD, T1, T2, LAn);
    axpby_eye(D, 1.0, a.qq, 1.0, LA, 0.0, M1);
    gemm<false, false>(D, D, D, 1.0, Ek, D, M1, D, 0.0, T1, D);
    gemm<false, true>(D, D, D, 1.0, T1, D, Ek, D, 1.0, LAn, D);
    gemm<false, false>(D, D, D, 1.0, Ek, D, EA, D, 0.0, EAn, D);   // E Eagg
    double* t = EA;
    EA = EAn;
    EAn = t;
    t = LA;
    LA = LAn;
    LAn = t;
  }
  double* o = sagg + c * 2 * S::DD;
  for (int idx = threadIdx.x; idx < D * D; idx += kBT) {
    o[idx] = EA[idx];
    o[S::DD + idx] = LA[idx];
  }
}

// F3 (one CTA): P^s at every chunk's start node, from the right.
template <int D>
__global__ void __launch_bounds__(kBT) k_big_chain_fin(int64_t nc, const double* sagg, double* ps, double* T,
                                                       const double* right) {
  constexpr int64_t DD = int64_t(D) * D;
  for (int64_t c = nc - 1; c >= 0; --c) {
    const double* g = sagg + c * 2 * DD;
    const double* nxt = (c == nc - 1) ? right : ps + (c + 1) * DD;
    double* out = ps + c * DD;
    copy(D * D, g + DD, out);
    if (nxt) {
      gemm<false, false>(D, D, D, 1.0, g, D, nxt, D, 0.0, T, D);
      gemm<false, true>(D, D, D, 1.0, T, D, g, D, 1.0, out, D);
    }
    symmetrize(D, out, D);
  }
}

// Pivoted Cholesky of the symmetric PSD n x n A (shared memory, stride la,
// both triangles; destroyed): A = Pi L L^T Pi^T with the largest remaining
// diagonal as pivot; a pivot <= 1e-15 max diag ends the factorisation
// (remaining columns zero).  Blocked: 8-column panels, each column one
// symmetric row/column swap and one left-looking column update inside the
// panel (2 barriers), the trailing update a DMMA rank-8 product on full
// tiles (the trailing block stays exactly symmetric for the swaps).  On
// return L is in A's lower triangle (pivot order), perm[i] = original index
// of pivot row i; returns the rank.
__device__ int psd_factor_smem(int n, double* A, int la, int* perm, double* red) {
  __shared__ double s_dg[128];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gr = lane >> 2, tg = lane & 3;
  double mloc = 0.0;
  for (int i = threadIdx.x; i < n; i += kBT) {
    perm[i] = i;
    s_dg[i] = A[i * la + i];
    mloc = fmax(mloc, A[i * la + i]);
  }
  const double tol = 1e-15 * block_max(mloc, red);  // (syncs)
  int rank = n;
  for (int j0 = 0; j0 < n && rank == n; j0 += 8) {
    const int w = min(8, n - j0);
    for (int c = 0; c < w; ++c) {
      const int j = j0 + c;
      // pivot: every warp finds it (no broadcast barrier)
      double best = -1.0;
      int bi = j;
      for (int i = j + lane; i < n; i += 32) {
        const double v = s_dg[i];
        if (v > best) {
          best = v;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
          best = ov;
          bi = oi;
        }
      }
      if (!(best > tol)) {  // CTA-uniform: rank j
        rank = j;
        break;
      }
      const int p = bi;
      if (p != j) {  // rows j <-> p (all columns), then (below) columns per row
        for (int t = threadIdx.x; t < n; t += kBT) {
          const double x = A[j * la + t];
          A[j * la + t] = A[p * la + t];
          A[p * la + t] = x;
        }
        if (threadIdx.x == 0) {
          const double x = s_dg[j];
          s_dg[j] = s_dg[p];
          s_dg[p] = x;
          const int q = perm[j];
          perm[j] = perm[p];
          perm[p] = q;
        }
      }
      __syncthreads();
      // thread per row i >= j: swap its columns j <-> p, then
      // L_ij = (A_ij - sum_{c' in panel, < j} L_ic' L_jc') / L_jj
      const double l = sqrt(s_dg[j]), inv = 1.0 / l;
      for (int i = j + threadIdx.x; i < n; i += kBT) {
        double v = A[i * la + p];
        if (p != j) {
          A[i * la + p] = A[i * la + j];
        }
        if (i == j) {
          A[i * la + j] = l;
        } else {
          for (int c2 = j0; c2 < j; ++c2) v = fma(-A[i * la + c2], A[j * la + c2], v);
          v *= inv;
          A[i * la + j] = v;
          s_dg[i] -= v * v;
        }
      }
      __syncthreads();
    }
    if (rank < n) break;
    // trailing update A22 -= L21 L21^T (full tiles), rank w, on DMMA
    const int r0b = j0 + w, M = n - r0b;
    if (M > 0) {
      const int tiles = (M + 7) / 8;
      for (int q = warp; q < tiles * tiles; q += kBW) {
        const int ti = q / tiles, tj = q - ti * tiles;
        const int rr = r0b + ti * 8 + gr, cc = r0b + tj * 8 + 2 * tg, rb = r0b + tj * 8 + gr;
        double c0 = (rr < n && cc < n) ? A[rr * la + cc] : 0.0;
        double c1 = (rr < n && cc + 1 < n) ? A[rr * la + cc + 1] : 0.0;
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4) {
          if (kk < w) {
            const int k = j0 + kk + tg;
            const double a = (rr < n && kk + tg < w) ? -A[rr * la + k] : 0.0;
            const double b = (rb < n && kk + tg < w) ? A[rb * la + k] : 0.0;
            dmma(c0, c1, a, b, c0, c1);
          }
        }
        if (rr < n && cc < n) A[rr * la + cc] = c0;
        if (rr < n && cc + 1 < n) A[rr * la + cc + 1] = c1;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  return rank;
}

struct BigOut {
  double* means;
  double* cov;
  double* sol_m;
  double* sol_c;
};

// F4: P^s_k = M1_k + E_k P^s_{k+1} E_k^T from the chunk's end, with the
// calibrated outputs (ieks.cpp:196-208).
template <int D, int d>
__global__ void __launch_bounds__(kBT) k_big_fin_bwd(BigArgs a, const double* E_in, const double* pf,
                                                     const double* pterm, const double* ps, const double* eta_out,
                                                     const double* innov_tot, double count, BigOut o, int last) {
  using G = Big<D, d>;
  using S = Slots<D, d>;
  constexpr int B = D / d;
  __shared__ StepSm<D, d> s;
  __shared__ int perm[D];
  __shared__ double tt[B], tti[B];
  const int64_t c = blockIdx.x;
  const int64_t s0 = c * a.L, e = min(a.N, s0 + a.L);
  const bool lastc = c == a.nchunks - 1;
  double* w = a.ws + c * a.ws_stride;
  double *Pn = w, *T1 = w + 2 * S::DD, *T2 = w + 3 * S::DD, *Pk = w + 4 * S::DD, *T3 = w + 5 * S::DD;
  constexpr int ls = smem_ld(D);
  double* b1 = dyn_smem();
  const double sig = sqrt(innov_tot[0] / count);
  stage(D, D, lastc ? pterm : ps + (c + 1) * S::DD, D, Pn, D);
  auto emit = [&](int64_t n, const double* Pnode) {
    if (threadIdx.x == 0) G::taus(a.grid, n, tt, tti);
    if (o.cov) {  // F = Pi L, row perm[i] of F = row i of L, scaled by T_n sigma
      stage(D, D, Pnode, D, b1, ls);
      const int rank = psd_factor_smem(D, b1, ls, perm, s.red);
      double* oc = o.cov + n * S::DD;
      for (int base = threadIdx.x; base < D * D; base += 4 * kBT) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int idx = base + u * kBT;
          if (idx < D * D) {
            const int i = idx / D, cc = idx - i * D, pi = perm[i];
            oc[pi * D + cc] = (cc <= i && cc < rank) ? tt[pi % B] * b1[i * ls + cc] * sig : 0.0;
          }
        }
      }
    }
    for (int r = threadIdx.x; r < D; r += kBT) {
      if (o.means) o.means[n * D + r] = eta_out[n * D + r];
      if (o.sol_m && r % B == 0) o.sol_m[n * d + r / B] = eta_out[n * D + r];
    }
    for (int idx = threadIdx.x; idx < d * d; idx += kBT) {
      const int i = idx / d, j = idx - (idx / d) * d;
      if (o.sol_c) o.sol_c[n * d * d + idx] = (tt[0] * sig) * (tt[0] * sig) * Pnode[(i * B) * D + j * B];
    }
    __syncthreads();
  };
  if (lastc && last) emit(e, Pn);
  for (int64_t k = e - 1; k >= s0; --k) {
    G::step_consts(s, a.grid, k);
    const double* Ek = E_in + k * S::DD;
    // P^s_k = (I - E phi) P+ (I - E phi)^T + E (Q Q^T + P^s_{k+1}) E^T
    smooth_joseph<D, d>(s, Ek, pf + k * S::DD, T1, T2, Pk);
    axpby_eye(D, 1.0, a.qq, 1.0, Pn, 0.0, T3);
    gemm<false, false>(D, D, D, 1.0, Ek, D, T3, D, 0.0, T2, D);   // E (Q Q^T + P^s_{k+1})
    gemm<false, true>(D, D, D, 1.0, T2, D, Ek, D, 1.0, Pk, D);    // .. E^T
    symmetrize(D, Pk, D);
    emit(k, Pk);
    double* t = Pn;
    Pn = Pk;
    Pk = t;
  }
}

}  // namespace big
}  // namespace pode
