// Lane-serial small-matrix fp64 kernels: one time-chunk (or one scan
// element) per THREAD, every matrix in registers, no cross-lane traffic.
//
// Why: a square-root Kalman step at D <= 8 is ~10^3 FMAs of short, mostly
// independent row updates.  Spreading one step over D lanes (group.cuh)
// costs ~3x more shuffle / shared-memory / select instructions than FMAs and
// leaves every lane waiting on the pivot chain; running 32 independent
// chunks per warp instead keeps the FP64 pipe fed with pure DFMA streams and
// needs no synchronisation at all.  Register pressure is the price; spills
// (if any) stay in L1.
//
// Algebra restated (row form of Eigen's Householder QR of the transpose,
// proj/src/linalg.cpp:9-27): kf_predict / kf_update (sequential.cpp:30-67),
// make_filtering_element + ⊗_f (parallel.cpp:5-100), make_smoothing_element
// (parallel.cpp:112-135), ⊗_s on (E, g) (parallel.cpp:146-156).
#pragma once

#include <cfloat>

#include "engine.cuh"
#include "field.cuh"
#include "fast.cuh"

namespace pode {
namespace lane {

#ifndef PODE_LANE_THREADS
#define PODE_LANE_THREADS 128
#endif
constexpr int kLaneThreads = PODE_LANE_THREADS;
// Pass E is HBM-bound: more resident warps would keep more loads in flight
// (register cap 64K / (128 * kBwdMinBlocks)); 3 and 4 spilled, so 2.
#ifndef PODE_BWD_MIN_BLOCKS
#define PODE_BWD_MIN_BLOCKS 2
#endif
constexpr int kBwdMinBlocks = PODE_BWD_MIN_BLOCKS;
// Passes A and C: resident 128-thread blocks per SM the register allocation
// targets (1 = up to 255 registers).
#ifndef PODE_LANE_MIN_BLOCKS
#define PODE_LANE_MIN_BLOCKS 1
#endif
constexpr int kLaneMinBlocks = PODE_LANE_MIN_BLOCKS;
// Register budget of passes A and C: the launch bounds above, or an explicit
// cap (PODE_LANE_MAXNREG, developer A/B builds).
#ifdef PODE_LANE_MAXNREG
#define PODE_LANE_BOUNDS __maxnreg__(PODE_LANE_MAXNREG)
#else
#define PODE_LANE_BOUNDS __launch_bounds__(kLaneThreads, kLaneMinBlocks)
#endif

// Householder LQ of an R x K row-major register matrix over the first P
// pivots: row p is reflected against columns p..K-1 and every later row is
// updated (Eigen convention: beta = -sign(c0) ||x||, tau = (beta - c0) / beta,
// essential = tail / (c0 - beta); identity when ||tail||^2 <= DBL_MIN).
// S < K: the right block (columns >= S) is lower triangular, so columns
// > S + p are structurally zero at pivot p and skipped (group.cuh live_col).
template <int R, int K, int P, int S = K>
__device__ __forceinline__ void lq(double (&m)[R][K]) {
#pragma unroll
  for (int p = 0; p < P; ++p) {
    double t0 = 0.0, t1 = 0.0;
#pragma unroll
    for (int j = p + 1; j < K; ++j) {
      if (!live_col(j, p, S)) continue;
      if ((j - p) & 1)
        t0 = fma(m[p][j], m[p][j], t0);
      else
        t1 = fma(m[p][j], m[p][j], t1);
    }
    const double tail = t0 + t1;
    double tau, beta, inv;
    householder_coefs(m[p][p], tail, tau, beta, inv);  // branch-free (group.cuh)
    double ess[K];
#pragma unroll
    for (int j = p + 1; j < K; ++j) ess[j] = live_col(j, p, S) ? m[p][j] * inv : 0.0;
#pragma unroll
    for (int r = p + 1; r < R; ++r) {
      double w0 = m[r][p], w1 = 0.0;
#pragma unroll
      for (int j = p + 1; j < K; ++j) {
        if (!live_col(j, p, S)) continue;
        if ((j - p) & 1)
          w1 = fma(m[r][j], ess[j], w1);
        else
          w0 = fma(m[r][j], ess[j], w0);
      }
      const double tw = tau * (w0 + w1);
      m[r][p] -= tw;
#pragma unroll
      for (int j = p + 1; j < K; ++j)
        if (live_col(j, p, S)) m[r][j] = fma(-tw, ess[j], m[r][j]);
    }
    // when tau == 0 (tail below DBL_MIN) this is the identity with beta = c0;
    // the tail is dropped, as Eigen's triangular view of R drops it
    m[p][p] = beta;
#pragma unroll
    for (int j = p + 1; j < K; ++j) m[p][j] = 0.0;
  }
}

template <int D>
__device__ __forceinline__ bool singular_diag(const double (&l)[D][D], int n) {
  double mx = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i)
    if (i < n) mx = fmax(mx, fabs(l[i][i]));
  bool s = false;
#pragma unroll
  for (int i = 0; i < D; ++i)
    if (i < n) s |= fabs(l[i][i]) <= 1e-13 * mx;
  return s;
}

// The transition's block structure: phi_n = phi_bar diag(ratio), phi_bar
// block-diagonal binomial (prior.cpp:99-107; ieks.cpp:37-45).
template <int D, int d>
struct Model {
  static constexpr int B = D / d;
  static constexpr int q = B - 1;

  __device__ static double binom(int n, int k) {
    double num = 1.0, den = 1.0;
    for (int t = 0; t < k; ++t) {
      num *= double(n - t);
      den *= double(t + 1);
    }
    return num / den;
  }

  // phi entry (a -> i within a block) = phi_bar[a][i] * ratio[i]
  __device__ static void phi_coefs(const double (&ratio)[B], double (&pc)[B][B]) {
#pragma unroll
    for (int a = 0; a < B; ++a)
#pragma unroll
      for (int i = 0; i < B; ++i) pc[a][i] = (i >= a) ? binom(q - a, i - a) * ratio[i] : 0.0;
  }

  // y = phi x on columns [0, NC) (in place safe: row a of a block reads
  // rows >= a).
  template <int K, int NC = K>
  __device__ static void phi_rows(const double (&pc)[B][B], double (&x)[D][K]) {
#pragma unroll
    for (int blk = 0; blk < d; ++blk)
#pragma unroll
      for (int a = 0; a < B; ++a) {
        double o[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) o[j] = pc[a][a] * x[blk * B + a][j];
#pragma unroll
        for (int i = a + 1; i < B; ++i)
#pragma unroll
          for (int j = 0; j < NC; ++j) o[j] = fma(pc[a][i], x[blk * B + i][j], o[j]);
#pragma unroll
        for (int j = 0; j < NC; ++j) x[blk * B + a][j] = o[j];
      }
  }

  __device__ static void phi_vec(const double (&pc)[B][B], double (&x)[D]) {
#pragma unroll
    for (int blk = 0; blk < d; ++blk)
#pragma unroll
      for (int a = 0; a < B; ++a) {
        double o = pc[a][a] * x[blk * B + a];
#pragma unroll
        for (int i = a + 1; i < B; ++i) o = fma(pc[a][i], x[blk * B + i], o);
        x[blk * B + a] = o;
      }
  }

  // Linearisation (statespace.cpp:65-103) at the full state eta (original
  // coordinates); H_bar row i = (E_1 - F_y E_0)[i] diag(T_{n}).
  struct Lin {
    double jac[d][d];
    double off[d];
    bool finite;
  };
  __device__ static Lin linearize(const DevProblem& prob, const double (&y)[d], int ek0, double t) {
    Lin l;
    double f[d], jac[d * d];
    eval_field<d>(prob, y, f, jac, t);
    bool fin = true;
#pragma unroll
    for (int j = 0; j < d; ++j) fin &= isfinite(f[j]);
#pragma unroll
    for (int i = 0; i < d; ++i)
#pragma unroll
      for (int j = 0; j < d; ++j) {
        if (!ek0) fin &= isfinite(jac[i * d + j]);
        l.jac[i][j] = ek0 ? 0.0 : jac[i * d + j];
      }
    l.finite = fin;
#pragma unroll
    for (int i = 0; i < d; ++i) {
      double jy = 0.0;
#pragma unroll
      for (int j = 0; j < d; ++j) jy += l.jac[i][j] * y[j];
      l.off[i] = ek0 ? f[i] : f[i] - jy;
    }
    return l;
  }

  // rows of H_bar X (d x K)
  template <int K>
  __device__ static void h_rows(const Lin& l, const double (&t)[B], const double (&x)[D][K], double (&o)[d][K]) {
#pragma unroll
    for (int i = 0; i < d; ++i) {
#pragma unroll
      for (int j = 0; j < K; ++j) o[i][j] = (1.0 * t[1]) * x[i * B + 1][j];
#pragma unroll
      for (int c = 0; c < d; ++c) {
        const double coef = (-l.jac[i][c]) * t[0];
#pragma unroll
        for (int j = 0; j < K; ++j) o[i][j] = fma(coef, x[c * B][j], o[i][j]);
      }
    }
  }
  __device__ static void h_vec(const Lin& l, const double (&t)[B], const double (&x)[D], double (&o)[d]) {
#pragma unroll
    for (int i = 0; i < d; ++i) {
      double v = (1.0 * t[1]) * x[i * B + 1];
#pragma unroll
      for (int c = 0; c < d; ++c) v = fma((-l.jac[i][c]) * t[0], x[c * B], v);
      o[i] = v;
    }
  }

  // Square-root update against the noiseless d-row observation
  // (sequential.cpp:41-67, R = 0): Psi = tria([[H C-], [C-]]) over D
  // columns.  Produces S (d x d), the gain K (D x d) and C+ (in cm).
  struct Upd {
    double s[d][d];
    double sinv[d];
    double k[D][d];
    bool singular;
  };
  __device__ static Upd update(const Lin& l, const double (&t)[B], double (&cm)[D][D]) {
    Upd u;
    double psi[d + D][D];
    double hc[d][D];
    h_rows<D>(l, t, cm, hc);
#pragma unroll
    for (int i = 0; i < d; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) psi[i][j] = hc[i][j];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int j = 0; j < D; ++j) psi[d + r][j] = cm[r][j];
    lq<d + D, D, D>(psi);
    double mx = 0.0;
#pragma unroll
    for (int i = 0; i < d; ++i) mx = fmax(mx, fabs(psi[i][i]));
    bool sg = false;
#pragma unroll
    for (int i = 0; i < d; ++i) {
      sg |= fabs(psi[i][i]) <= 1e-13 * mx;
#pragma unroll
      for (int j = 0; j < d; ++j) u.s[i][j] = (j <= i) ? psi[i][j] : 0.0;
      u.sinv[i] = rcp_nr(psi[i][i]);
    }
    u.singular = sg;
    // K = Psi21 S^-1 (x S = Psi21[r]) ; C+ = Psi22 (shifted by d columns)
#pragma unroll
    for (int r = 0; r < D; ++r) {
#pragma unroll
      for (int i = d - 1; i >= 0; --i) {
        double acc = psi[d + r][i];
#pragma unroll
        for (int k = i + 1; k < d; ++k) acc = fma(-u.k[r][k], u.s[k][i], acc);
        u.k[r][i] = acc * u.sinv[i];
      }
#pragma unroll
      for (int j = 0; j < D; ++j) cm[r][j] = (j <= r && j < D - d) ? psi[d + r][d + j] : 0.0;
    }
    return u;
  }

  __device__ static void s_solve(const Upd& u, const double (&v)[d], double (&w)[d]) {
#pragma unroll
    for (int i = 0; i < d; ++i) {
      double acc = v[i];
#pragma unroll
      for (int k = 0; k < i; ++k) acc = fma(-u.s[i][k], w[k], acc);
      w[i] = acc * u.sinv[i];
    }
  }

  // C- = tria([phi C, Q]) (kf_predict, sequential.cpp:30-39); on return
  // pm holds phi C (before the sweep, for callers that need it).
  __device__ static void predict_cov(const double (&pc)[B][B], const double (&c)[D][D], const double* qrow,
                                     double (&cm)[D][D]) {
    double m[D][2 * D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        m[r][j] = c[r][j];
        m[r][D + j] = qrow[r * D + j];
      }
    phi_rows<2 * D, D>(pc, m);  // phi acts on the left half only
    lq<D, 2 * D, D, D>(m);      // right block Q^1/2: lower triangular
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int j = 0; j < D; ++j) cm[r][j] = (j <= r) ? m[r][j] : 0.0;
  }

  // T_n = diag(sqrt(h) h^k / k!), k = q - i, for the incoming step h
  // (ieks.cpp:28-33), and its inverse from one division:
  // T^-1 = k! h^-k / sqrt(h) (1 / sqrt(h) = sqrt(h) / h).
  __device__ static void taus_h(double h, double (&t)[B], double (&ti)[B]) {
    const double rh = sqrt(h), ih = 1.0 / h, irh = rh * ih;
    double hp = 1.0, ihp = 1.0, fact = 1.0;
#pragma unroll
    for (int k = 0; k <= q; ++k) {
      if (k > 0) {
        hp *= h;
        ihp *= ih;
        fact *= k;
      }
      t[q - k] = k <= 2 ? rh * hp / fact : rh * hp * (1.0 / fact);  // (1/1, 1/2 exact)
      ti[q - k] = irh * ihp * fact;
    }
  }
  // origin: local node 0 is global node 0 (its scale uses the first step).
  __device__ static double step_h(const double* grid, int origin, int64_t n) {
    return (n == 0 && origin) ? grid[1] - grid[0] : grid[n] - grid[n - 1];
  }
  __device__ static void taus(const double* grid, int origin, int64_t n, double (&t)[B], double (&ti)[B]) {
    taus_h(step_h(grid, origin, n), t, ti);
  }
};

// Per-node smoothing elements (E_n, g_n) in a chunk-interleaved
// structure-of-arrays layout: entry x of node n = c L + t (chunk c, local
// step t) lives at (t * X + x) * nc + c, X = D*D for E and D for g, so the
// 32 lanes of a warp (32 consecutive chunks) touch 32 consecutive doubles on
// every access.  The terminal node N (E = 0, g = m_f(N)) is kept in `term`.
struct ElemSoA {
  double* e;
  double* g;
  double* term;
  int64_t nc;
  int L;
};

// The trajectory eta in the same chunk-interleaved layout: component r of
// node k = c L + t (k < N) at (t * D + r) * nc + c; node N in `term`.
template <int D>
__device__ __forceinline__ int64_t eta_index(int64_t k, int r, int L, int64_t nc) {
  const int64_t c = k / L;
  return ((k - c * L) * D + r) * nc + c;
}

template <int D>
__device__ __forceinline__ double eta_at(const double* base, const double* term, int64_t k, int r, int64_t N,
                                         int L, int64_t nc) {
  return (k == N) ? term[r] : base[eta_index<D>(k, r, L, nc)];
}

// y = E_0 eta at node k = s + t of chunk c (t = L: the next chunk's first
// node; k = N: the node-N slot), without an integer division.
template <int D, int d>
__device__ __forceinline__ void gather_y(const FastArgs& a, const LinPoint& lp, int64_t c, int64_t t, int64_t k,
                                         double (&y)[d]) {
  constexpr int B = D / d;
  const bool at_n = k == a.N;
  const bool wrap = t == a.L;
  const int64_t cc = wrap ? c + 1 : c, tt = wrap ? 0 : t;
#pragma unroll
  for (int j = 0; j < d; ++j) y[j] = at_n ? lp.term[j * B] : lp.eta[(tt * D + j * B) * a.nchunks + cc];
}

// Prefetch of gather_y's addresses (node k = s + t of chunk c) a step or two
// ahead (PODE_Y_PREFETCH=1: L1, 2: L2 evict_last).  Off by default: FHN 2^20
// ms per iteration, three interleaved runs each, 0.822 (off) vs 0.829 (L1)
// vs 0.829 (L2) — the sunk load's latency is covered by the other warp.
#ifndef PODE_Y_PREFETCH
#define PODE_Y_PREFETCH 0
#endif
template <int D, int d>
__device__ __forceinline__ void prefetch_y(const FastArgs& a, const LinPoint& lp, int64_t c, int64_t t, int64_t k) {
  if constexpr (PODE_Y_PREFETCH) {
    constexpr int B = D / d;
    if (k > a.N) return;
    const bool at_n = k == a.N;
    const bool wrap = t == a.L;
    const int64_t cc = wrap ? c + 1 : c, tt = wrap ? 0 : t;
#pragma unroll
    for (int j = 0; j < d; ++j) {
      const double* p = at_n ? lp.term + j * B : lp.eta + (tt * D + j * B) * a.nchunks + cc;
      if constexpr (PODE_Y_PREFETCH == 2)
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
      else
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
    }
  }
}

template <int D>
__device__ __forceinline__ void soa_st(const ElemSoA& s, int64_t c, int64_t t, const double (&E)[D][D],
                                       const double (&g)[D]) {
#pragma unroll
  for (int r = 0; r < D; ++r) {
#pragma unroll
    for (int j = 0; j < D; ++j) s.e[((t * D + r) * D + j) * s.nc + c] = E[r][j];
    s.g[(t * D + r) * s.nc + c] = g[r];
  }
}

template <int D>
__device__ __forceinline__ void soa_ld(const ElemSoA& s, int64_t c, int64_t t, double (&E)[D][D],
                                       double (&g)[D]) {
#pragma unroll
  for (int r = 0; r < D; ++r) {
#pragma unroll
    for (int j = 0; j < D; ++j) E[r][j] = s.e[((t * D + r) * D + j) * s.nc + c];
    g[r] = s.g[(t * D + r) * s.nc + c];
  }
}

template <int D>
__device__ __forceinline__ void ld_mat(const double* p, double (&m)[D][D]) {
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int j = 0; j < D; ++j) m[r][j] = p[r * D + j];
}
template <int D>
__device__ __forceinline__ void st_mat(double* p, const double (&m)[D][D]) {
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int j = 0; j < D; ++j) p[r * D + j] = m[r][j];
}

// Dynamic shared memory of pass C (the fused backward-aggregate slots).
template <int D>
constexpr size_t fwd_down_smem() {
  return sizeof(double) * (D * D + D) * kLaneThreads;
}

// Pass A keeps the chunk's A (D x D) in per-thread shared-memory slots when
// A, C and J together exceed the register file (D >= 8: 1 KB of spills).
template <int D>
constexpr bool fwd_reduce_a_smem() {
  return D >= 8;
}
template <int D>
constexpr size_t fwd_reduce_smem() {
  return fwd_reduce_a_smem<D>() ? sizeof(double) * D * D * kLaneThreads : 0;
}

// A D x D matrix per node in the chunk-interleaved layout of ElemSoA::e.
template <int D>
__device__ __forceinline__ void mat_st(double* base, int64_t nc, int64_t c, int64_t t, const double (&m)[D][D]) {
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int j = 0; j < D; ++j) base[((t * D + r) * D + j) * nc + c] = m[r][j];
}
template <int D>
__device__ __forceinline__ void mat_ld(const double* base, int64_t nc, int64_t c, int64_t t, double (&m)[D][D]) {
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int j = 0; j < D; ++j) m[r][j] = base[((t * D + r) * D + j) * nc + c];
}

// Block sum of one value per thread (fixed tree order) -> part[3 b] (the
// k_finish3 partial layout, maxima 0).  Every thread of the block must call it.
__device__ __forceinline__ void block_sum_partial(double* red, double v, double* part) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int st = kLaneThreads / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x * 3 + 0] = red[0];
    part[blockIdx.x * 3 + 1] = 0.0;
    part[blockIdx.x * 3 + 2] = 0.0;
  }
}

// ------------------------------------------------------------- pass A ---
// One thread per chunk: fold the chunk's filtering elements into the
// aggregate (A, b, C, eta, J) (see fast.cuh for the algebra).
template <int D, int d, bool kBatch = false>
__global__ void PODE_LANE_BOUNDS k_lane_fwd_reduce(const FastArgs a, FastConst<D> cst, FEd agg) {
  using M = Model<D, d>;
  constexpr int B = M::B;
  const int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (c >= a.nchunks) return;
  const SegPos sp = seg_pos<kBatch>(a, c);
  if (kBatch && sp.cl >= sp.nreal) {  // padding chunk: the identity aggregate
#pragma unroll
    for (int r = 0; r < D; ++r) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        agg.a[c * D * D + r * D + j] = (r == j) ? 1.0 : 0.0;
        agg.c[c * D * D + r * D + j] = 0.0;
        agg.j[c * D * D + r * D + j] = 0.0;
      }
      agg.b[c * D + r] = 0.0;
      agg.eta[c * D + r] = 0.0;
    }
    return;
  }
  if (kBatch && a.active != nullptr && !a.active[sp.seg]) return;  // converged IVP: its aggregates are not read
  const LinPoint lp = lin_point_seg<D, kBatch>(a, sp.seg);
  const DevProblem& prob = kBatch ? a.probs[sp.seg] : a.prob;
  const bool head = sp.cl == 0 && a.first;
  const int64_t s = sp.cl * a.L;
  const int64_t e = min(a.N, s + a.L);
  constexpr bool kAS = fwd_reduce_a_smem<D>();
  extern __shared__ double smem_a[];
  // A in registers, or (kAS) in this thread's conflict-free smem slots
  double A[kAS ? 1 : D][kAS ? 1 : D];
  auto sa = [&](int r, int j) -> double& { return smem_a[(r * D + j) * kLaneThreads + threadIdx.x]; };
  double C[D][D], J[D][D], b[D], eta[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if constexpr (kAS)
        sa(r, j) = (!head && r == j) ? 1.0 : 0.0;
      else
        A[r][j] = (!head && r == j) ? 1.0 : 0.0;
      C[r][j] = 0.0;
      J[r][j] = 0.0;
    }
    b[r] = head ? (kBatch ? a.m0s[sp.seg * D + r] : cst.m0[r]) : 0.0;
    eta[r] = 0.0;
  }
  double tk[B], tki[B];
  M::taus(a.grid, a.first, s, tk, tki);
  bool bad_sing = false;
  int64_t bad_lin = -1;
  // node times one step ahead (the grid load's latency overlaps a step)
  double gcur = a.grid[s], gnext = a.grid[s + 1];
  for (int64_t k = s; k < e; ++k) {
    double tn[B], tni[B], ratio[B], pc[B][B];
    const double h = gnext - gcur;
    gcur = gnext;
    if (k + 2 <= a.N) gnext = a.grid[k + 2];
    M::taus_h(h, tn, tni);
#pragma unroll
    for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tni[i];
    M::phi_coefs(ratio, pc);
    // predict
    if constexpr (kAS) {  // A <- phi A one block of B rows at a time
#pragma unroll
      for (int blk = 0; blk < d; ++blk) {
        double x[B][D];
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int j = 0; j < D; ++j) x[i][j] = sa(blk * B + i, j);
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int j = 0; j < D; ++j) {
            double o = pc[i][i] * x[i][j];
#pragma unroll
            for (int i2 = i + 1; i2 < B; ++i2) o = fma(pc[i][i2], x[i2][j], o);
            sa(blk * B + i, j) = o;
          }
      }
    } else {
      M::template phi_rows<D>(pc, A);
    }
    M::phi_vec(pc, b);
    double cm[D][D];
    M::predict_cov(pc, C, cst.q, cm);
    // update at node k+1
    double ylin[d];  // (a one-step-ahead load costs pass A more in spills than it saves)
    if (k + 1 < e) prefetch_y<D, d>(a, lp, c, k + 2 - s, k + 2);
    gather_y<D, d>(a, lp, c, k + 1 - s, k + 1, ylin);
    const typename M::Lin lin = M::linearize(prob, ylin, a.ek0, gcur);  // t_{k+1} (only PODE_POLE reads it)
    if (!lin.finite && bad_lin < 0) bad_lin = k + 1;
    const typename M::Upd u = M::update(lin, tn, cm);
    bad_sing |= u.singular;
    double U[d][D], uu[d];
    if constexpr (kAS) {  // h_rows on the smem rows cB and iB+1
#pragma unroll
      for (int i = 0; i < d; ++i) {
#pragma unroll
        for (int j = 0; j < D; ++j) U[i][j] = (1.0 * tn[1]) * sa(i * B + 1, j);
#pragma unroll
        for (int c2 = 0; c2 < d; ++c2) {
          const double coef = (-lin.jac[i][c2]) * tn[0];
#pragma unroll
          for (int j = 0; j < D; ++j) U[i][j] = fma(coef, sa(c2 * B, j), U[i][j]);
        }
      }
    } else {
      M::template h_rows<D>(lin, tn, A, U);
    }
    M::h_vec(lin, tn, b, uu);
#pragma unroll
    for (int i = 0; i < d; ++i) uu[i] -= lin.off[i];
    // A+ = A- - K U, b+ = b- - K u
#pragma unroll
    for (int r = 0; r < D; ++r) {
#pragma unroll
      for (int i = 0; i < d; ++i) {
#pragma unroll
        for (int j = 0; j < D; ++j) {
          if constexpr (kAS)
            sa(r, j) = fma(-u.k[r][i], U[i][j], sa(r, j));
          else
            A[r][j] = fma(-u.k[r][i], U[i][j], A[r][j]);
        }
        b[r] = fma(-u.k[r][i], uu[i], b[r]);
      }
    }
    // Ubar = S^-1 U, ubar = S^-1 u; eta -= Ubar^T ubar; J = tria([J, Ubar^T])
    double ub[d], X[D][d];
    M::s_solve(u, uu, ub);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double col[d], w[d];
#pragma unroll
      for (int i = 0; i < d; ++i) col[i] = U[i][j];
      M::s_solve(u, col, w);
      double de = 0.0;
#pragma unroll
      for (int i = 0; i < d; ++i) {
        X[j][i] = w[i];
        de = fma(w[i], ub[i], de);
      }
      eta[j] -= de;
    }
    // structured Householder sweep: row p of [J | X] is nonzero only in
    // columns <= p and the d extra columns.
#pragma unroll
    for (int p = 0; p < D; ++p) {
      double tail = 0.0;
#pragma unroll
      for (int i = 0; i < d; ++i) tail = fma(X[p][i], X[p][i], tail);
      double tau, beta, inv;
      householder_coefs(J[p][p], tail, tau, beta, inv);
      double ess[d];
#pragma unroll
      for (int i = 0; i < d; ++i) ess[i] = X[p][i] * inv;
#pragma unroll
      for (int r = p + 1; r < D; ++r) {
        double w = J[r][p];
#pragma unroll
        for (int i = 0; i < d; ++i) w = fma(X[r][i], ess[i], w);
        const double tw = tau * w;
        J[r][p] -= tw;
#pragma unroll
        for (int i = 0; i < d; ++i) X[r][i] = fma(-tw, ess[i], X[r][i]);
      }
      J[p][p] = beta;
    }
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int j = 0; j < D; ++j) C[r][j] = (j <= r) ? cm[r][j] : 0.0;
#pragma unroll
    for (int i = 0; i < B; ++i) {
      tk[i] = tn[i];
      tki[i] = tni[i];
    }
  }
  if (bad_lin >= 0) raise_error(a.err, bad_lin, kErrLinearization);
  if (bad_sing) raise_error(a.err, s, kErrSingular);
  if constexpr (kAS) {
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int j = 0; j < D; ++j) agg.a[c * D * D + r * D + j] = sa(r, j);
  } else {
    st_mat<D>(agg.a + c * D * D, A);
  }
  st_mat<D>(agg.c + c * D * D, C);
  st_mat<D>(agg.j + c * D * D, J);
#pragma unroll
  for (int r = 0; r < D; ++r) {
    agg.b[c * D + r] = b[r];
    agg.eta[c * D + r] = eta[r];
  }
}

// ------------------------------------------------------------- pass C ---
// One thread per chunk: square-root Kalman filter from the chunk's incoming
// filtered marginal; smoothing elements E_n, g_n (parallel.cpp:112-135) of
// every node (chunk-interleaved layout, ElemSoA).
// kFinal (once, after convergence): also stores the filtered factor C_f(k)
// of every node (cf, chunk-interleaved like E; node N in cterm) and reduces
// the whitened innovations ||S^-1 (H m- - offset)||^2 (innovation_stats,
// ieks.cpp:79-104) into one partial per block.
template <int D, int d, bool kFinal, bool kBatch>
__device__ __forceinline__ double fwd_down_chunk(const FastArgs& a, const FastConst<D>& cst, const FEd& prefix,
                                                 const ElemSoA& elems, double* cf, double* cterm, int64_t c,
                                                 double* sacc, const SEd& bagg, const SegPos& sp) {
  using M = Model<D, d>;
  constexpr int B = M::B;
  double innov = 0.0;
  const LinPoint lp = lin_point_seg<D, kBatch>(a, sp.seg);
  const DevProblem& prob = kBatch ? a.probs[sp.seg] : a.prob;
  const int64_t s = sp.cl * a.L;
  const int64_t e = min(a.N, s + a.L);
  double m[D], C[D][D];
  if (sp.cl == 0 && a.first) {
#pragma unroll
    for (int r = 0; r < D; ++r) {
      m[r] = kBatch ? a.m0s[sp.seg * D + r] : cst.m0[r];
#pragma unroll
      for (int j = 0; j < D; ++j) C[r][j] = 0.0;
    }
  } else if (sp.cl == 0) {  // shard > 0: the filtered marginal folded from the left
    ld_mat<D>(a.carry + D, C);
#pragma unroll
    for (int r = 0; r < D; ++r) m[r] = a.carry[r];
  } else {
    ld_mat<D>(prefix.c + (c - 1) * D * D, C);
#pragma unroll
    for (int r = 0; r < D; ++r) m[r] = prefix.b[(c - 1) * D + r];
  }
  double tk[B], tki[B];
  M::taus(a.grid, a.first, s, tk, tki);
  bool bad_sing = false;
  int64_t bad_lin = -1;
  // the linearisation point and the node time of the next step are loaded
  // one step ahead, so their global-memory latency overlaps the current
  // step's arithmetic
  double ynext[d];
  gather_y<D, d>(a, lp, c, 1, s + 1, ynext);
  double gcur = a.grid[s], gnext = a.grid[s + 1];
  for (int64_t k = s; k < e; ++k) {
    double tn[B], tni[B], ratio[B], pc[B][B];
    const double h = gnext - gcur;
    gcur = gnext;
    if (k + 2 <= a.N) gnext = a.grid[k + 2];
    M::taus_h(h, tn, tni);
#pragma unroll
    for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tni[i];
    M::phi_coefs(ratio, pc);
    // Y = C (phi C)^T = C C^T phi^T; C- = tria([phi C, Q]); E = Y C-^-T C-^-1
    if constexpr (kFinal) mat_st<D>(cf, a.nchunks, c, k - s, C);
    double pcC[D][D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int j = 0; j < D; ++j) pcC[r][j] = C[r][j];
    M::template phi_rows<D>(pc, pcC);
    double Y[D][D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int x = 0; x <= r; ++x) acc = fma(C[r][x], pcC[j][x], acc);
        Y[r][j] = acc;
      }
    double cm[D][D];
    M::predict_cov(pc, C, cst.q, cm);
    bad_sing |= singular_diag<D>(cm, D);
    double rd[D];
#pragma unroll
    for (int i = 0; i < D; ++i) rd[i] = rcp_nr(cm[i][i]);
    double E[D][D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double z[D];
#pragma unroll
      for (int i = 0; i < D; ++i) {  // z C-^T = Y[r]  (forward)
        double acc = Y[r][i];
#pragma unroll
        for (int k2 = 0; k2 < i; ++k2) acc = fma(-cm[i][k2], z[k2], acc);
        z[i] = acc * rd[i];
      }
#pragma unroll
      for (int i = D - 1; i >= 0; --i) {  // E[r] C- = z  (backward)
        double acc = z[i];
#pragma unroll
        for (int k2 = i + 1; k2 < D; ++k2) acc = fma(-E[r][k2], cm[k2][i], acc);
        E[r][i] = acc * rd[i];
      }
    }
    double mm[D];
#pragma unroll
    for (int r = 0; r < D; ++r) mm[r] = m[r];
    M::phi_vec(pc, mm);
    double gk[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) acc = fma(E[r][j], mm[j], acc);
      gk[r] = m[r] - acc;
    }
    soa_st<D>(elems, c, k - s, E, gk);
    if constexpr (!kFinal) {
      // pass C2 fused: the chunk's backward aggregate (E, g) <- (E E_k, E g_k + g)
      // in time order (⊗_s on means, parallel.cpp:146-156), accumulated in
      // this thread's shared-memory slots
      auto ae = [&](int r, int j) -> double& { return sacc[(r * D + j) * kLaneThreads + threadIdx.x]; };
      auto ag = [&](int r) -> double& { return sacc[(D * D + r) * kLaneThreads + threadIdx.x]; };
      if (k == s) {
#pragma unroll
        for (int r = 0; r < D; ++r) {
#pragma unroll
          for (int j = 0; j < D; ++j) ae(r, j) = E[r][j];
          ag(r) = gk[r];
        }
      } else {
#pragma unroll
        for (int r = 0; r < D; ++r) {
          double row[D], o[D], og = ag(r);
#pragma unroll
          for (int x = 0; x < D; ++x) {
            row[x] = ae(r, x);
            o[x] = 0.0;
          }
#pragma unroll
          for (int x = 0; x < D; ++x) {
#pragma unroll
            for (int j = 0; j < D; ++j) o[j] = fma(row[x], E[x][j], o[j]);
            og = fma(row[x], gk[x], og);
          }
#pragma unroll
          for (int j = 0; j < D; ++j) ae(r, j) = o[j];
          ag(r) = og;
        }
      }
    }
    // measurement update at node k+1
    double ylin[d];
#pragma unroll
    for (int i = 0; i < d; ++i) ylin[i] = ynext[i];
    if (k + 2 < e) prefetch_y<D, d>(a, lp, c, k + 3 - s, k + 3);
    if (k + 1 < e) gather_y<D, d>(a, lp, c, k + 2 - s, k + 2, ynext);
    const typename M::Lin lin = M::linearize(prob, ylin, a.ek0, gcur);  // t_{k+1} (only PODE_POLE reads it)
    if (!lin.finite && bad_lin < 0) bad_lin = k + 1;
    const typename M::Upd u = M::update(lin, tn, cm);
    bad_sing |= u.singular;
    double z[d];
    M::h_vec(lin, tn, mm, z);
#pragma unroll
    for (int i = 0; i < d; ++i) z[i] -= lin.off[i];
    if constexpr (kFinal) {
      double w[d];
      M::s_solve(u, z, w);
#pragma unroll
      for (int i = 0; i < d; ++i) innov = fma(w[i], w[i], innov);
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double v = mm[r];
#pragma unroll
      for (int i = 0; i < d; ++i) v = fma(-u.k[r][i], z[i], v);
      m[r] = v;
#pragma unroll
      for (int j = 0; j < D; ++j) C[r][j] = (j <= r) ? cm[r][j] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < B; ++i) {
      tk[i] = tn[i];
      tki[i] = tni[i];
    }
  }
  if (e == a.N) {  // terminal node N: E = 0, g = m_f(N) (parallel.cpp:137-144)
#pragma unroll
    for (int r = 0; r < D; ++r) elems.term[sp.seg * D + r] = m[r];
    if constexpr (kFinal) st_mat<D>(cterm + sp.seg * D * D, C);
  }
  if constexpr (!kFinal) {  // store the backward aggregate (the last shard's last chunk absorbs the terminal)
    const bool term = e == a.N && a.last;
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double og = sacc[(D * D + r) * kLaneThreads + threadIdx.x];
      if (term) {
#pragma unroll
        for (int x = 0; x < D; ++x) og = fma(sacc[(r * D + x) * kLaneThreads + threadIdx.x], m[x], og);
      }
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double v = sacc[(r * D + j) * kLaneThreads + threadIdx.x];
        bagg.e[c * D * D + r * D + j] = term ? 0.0 : v;
      }
      bagg.g[c * D + r] = og;
    }
  }
  if (bad_lin >= 0) raise_error(a.err, bad_lin, kErrLinearization);
  if (bad_sing) raise_error(a.err, s, kErrSingular);
  return innov;
}

template <int D, int d, bool kFinal = false, bool kBatch = false>
__global__ void PODE_LANE_BOUNDS k_lane_fwd_down(const FastArgs a, FastConst<D> cst, FEd prefix,
                                                                ElemSoA elems, double* cf = nullptr,
                                                                double* cterm = nullptr, double* part = nullptr,
                                                                SEd bagg = SEd{}) {
  __shared__ double red[kFinal ? kLaneThreads : 1];
  extern __shared__ double sacc[];  // !kFinal: (D*D + D) x kLaneThreads aggregate slots
  const int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  double innov = 0.0;
  if (c < a.nchunks) {
    const SegPos sp = seg_pos<kBatch>(a, c);
    if (kBatch && sp.cl >= sp.nreal) {  // padding chunk: identity backward aggregate
      if constexpr (!kFinal) {
#pragma unroll
        for (int r = 0; r < D; ++r) {
#pragma unroll
          for (int j = 0; j < D; ++j) bagg.e[c * D * D + r * D + j] = (r == j) ? 1.0 : 0.0;
          bagg.g[c * D + r] = 0.0;
        }
      }
    } else if (!kBatch || a.active == nullptr || a.active[sp.seg]) {
      innov = fwd_down_chunk<D, d, kFinal, kBatch>(a, cst, prefix, elems, cf, cterm, c, sacc, bagg, sp);
    }
  }
  if constexpr (kFinal) block_sum_partial(red, innov, part);  // every thread reaches the barriers
}

// ------------------------------------------------- finalize (once) ---
// Smoothing-element covariance factor in Joseph form,
//   L_k = tria([(I - E_k phi_k) C_f(k), E_k Q^1/2]),
// L L^T = P_f - E P^- E^T: the same Gaussian as the lower-right block of the
// reference's tria (make_smoothing_element, parallel.cpp:112-135).
template <int D, int d>
__device__ __forceinline__ void smooth_factor(const double (&pc)[D / d][D / d], const double (&E)[D][D],
                                              const double (&cf)[D][D], const double* q, double (&lk)[D][D]) {
  using M = Model<D, d>;
  double x[D][D];
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int j = 0; j < D; ++j) x[r][j] = cf[r][j];
  M::template phi_rows<D>(pc, x);
  double m[D][2 * D];
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double acc = cf[r][j], acq = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        acc = fma(-E[r][k], x[k][j], acc);
        if (k >= j) acq = fma(E[r][k], q[k * D + j], acq);  // Q^1/2 lower triangular
      }
      m[r][j] = acc;
      m[r][D + j] = acq;
    }
  lq<D, 2 * D, D>(m);
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int j = 0; j < D; ++j) lk[r][j] = (j <= r) ? m[r][j] : 0.0;
}

// l <- tria([E l, lk]) (⊗_s covariance part, parallel.cpp:146-156; lk lower).
template <int D>
__device__ __forceinline__ void smooth_combine_factor(const double (&E)[D][D], const double (&lk)[D][D],
                                                      double (&l)[D][D]) {
  double m[D][2 * D];
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) acc = fma(E[r][k], l[k][j], acc);
      m[r][j] = acc;
      m[r][D + j] = lk[r][j];
    }
  lq<D, 2 * D, D, D>(m);
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int j = 0; j < D; ++j) l[r][j] = (j <= r) ? m[r][j] : 0.0;
}

// F2: each chunk's full smoothing aggregate e_s ⊗ .. ⊗ e_{e-1} (⊗ the
// terminal element for the last chunk) as (E, g, L), folded backwards; the
// per-node L_k are formed on the fly from (E_k, C_f(k)).
template <int D, int d, bool kBatch = false>
__global__ void __launch_bounds__(kLaneThreads) k_lane_fin_fold(FastArgs a, FastConst<D> cst, ElemSoA elems,
                                                                const double* cf, const double* cterm, SEd agg) {
  using M = Model<D, d>;
  constexpr int B = M::B;
  const int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (c >= a.nchunks) return;
  const SegPos sp = seg_pos<kBatch>(a, c);
  if (kBatch && sp.cl >= sp.nreal) {  // padding chunk: the identity (E, g, L) = (I, 0, 0)
#pragma unroll
    for (int r = 0; r < D; ++r) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        agg.e[c * D * D + r * D + j] = (r == j) ? 1.0 : 0.0;
        agg.l[c * D * D + r * D + j] = 0.0;
      }
      agg.g[c * D + r] = 0.0;
    }
    return;
  }
  const int64_t s = sp.cl * a.L;
  const int64_t e = min(a.N, s + a.L);
  const bool last = sp.cl == sp.nreal - 1 && a.last;
  double ea[D][D], la[D][D], ga[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
    ga[r] = last ? elems.term[sp.seg * D + r] : 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      ea[r][j] = (!last && r == j) ? 1.0 : 0.0;
      la[r][j] = last ? cterm[sp.seg * D * D + r * D + j] : 0.0;
    }
  }
  double tn[B], tni[B];
  M::taus(a.grid, a.first, e, tn, tni);
  BwdGrid bg(a.grid, a.first, e - 1);
  for (int64_t k = e - 1; k >= s; --k) {
    double tk[B], tki[B], ratio[B], pc[B][B];
    M::taus_h(bg.step(k), tk, tki);
#pragma unroll
    for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tni[i];
    M::phi_coefs(ratio, pc);
    double E[D][D], gk[D], cfk[D][D], lk[D][D];
    soa_ld<D>(elems, c, k - s, E, gk);
    mat_ld<D>(cf, a.nchunks, c, k - s, cfk);
    smooth_factor<D, d>(pc, E, cfk, cst.q, lk);
    smooth_combine_factor<D>(E, lk, la);
    double ne[D][D], ng[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double acc = gk[r];
#pragma unroll
      for (int x = 0; x < D; ++x) acc = fma(E[r][x], ga[x], acc);
      ng[r] = acc;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double v = 0.0;
#pragma unroll
        for (int x = 0; x < D; ++x) v = fma(E[r][x], ea[x][j], v);
        ne[r][j] = v;
      }
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
      ga[r] = ng[r];
#pragma unroll
      for (int j = 0; j < D; ++j) ea[r][j] = ne[r][j];
    }
#pragma unroll
    for (int i = 0; i < B; ++i) {
      tn[i] = tk[i];
      tni[i] = tki[i];
    }
  }
  st_mat<D>(agg.e + c * D * D, ea);
  st_mat<D>(agg.l + c * D * D, la);
#pragma unroll
  for (int r = 0; r < D; ++r) agg.g[c * D + r] = ga[r];
}

// Calibrated outputs of node n (ieks.cpp:196-208): means = eta, cov_sqrt =
// T_n L^s_n sigma_rel, and their solution-component projections.
struct FinOut {
  double* means;
  double* cov;
  double* sol_m;
  double* sol_c;
};

template <int D, int d>
__device__ __forceinline__ void write_node(const FinOut& o, int64_t n, const double (&t)[D / d],
                                           const double (&ls)[D][D], const double (&eta)[D], double sig) {
  constexpr int B = D / d;
  if (o.means) {
#pragma unroll
    for (int r = 0; r < D; ++r) o.means[n * D + r] = eta[r];
  }
  if (o.cov) {
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int j = 0; j < D; ++j) o.cov[(n * D + r) * D + j] = t[r % B] * ls[r][j] * sig;
  }
  if (o.sol_m) {
#pragma unroll
    for (int i = 0; i < d; ++i) o.sol_m[n * d + i] = eta[i * B];
  }
  if (o.sol_c) {
#pragma unroll
    for (int i = 0; i < d; ++i)
#pragma unroll
      for (int j = 0; j < d; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) acc += (t[0] * ls[i * B][k] * sig) * (t[0] * ls[j * B][k] * sig);
        o.sol_c[(n * d + i) * d + j] = acc;
      }
  }
}

// F4: backward smoothed-factor recursion L^s_k = tria([E_k L^s_{k+1}, L_k])
// from each chunk's incoming factor (the reverse scan of the F2 aggregates;
// the last chunk starts from C_f(N)), fused with the output projection.
template <int D, int d, bool kBatch = false>
__global__ void __launch_bounds__(kLaneThreads) k_lane_fin_bwd(FastArgs a, FastConst<D> cst, ElemSoA elems,
                                                               const double* cf, const double* cterm, SEd suffix,
                                                               const double* eta_out, const double* eta_out_term,
                                                               const double* innov, double count, FinOut o) {
  using M = Model<D, d>;
  constexpr int B = M::B;
  const int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (c >= a.nchunks) return;
  const SegPos sp = seg_pos<kBatch>(a, c);
  if (kBatch && sp.cl >= sp.nreal) return;
  if constexpr (kBatch) {  // IVP seg's newest trajectory: pair[it_b & 1]
    eta_out = (a.seg_it[sp.seg] & 1) ? a.pair1 : a.pair0;
    eta_out_term = eta_out + a.term_off + sp.seg * D;
  }
  const int64_t s = sp.cl * a.L;
  const int64_t e = min(a.N, s + a.L);
  const int64_t out0 = sp.seg * (a.N + 1);  // output node offset of this IVP
  const bool last = sp.cl == sp.nreal - 1;  // cterm: C_f(N), or the right carry's factor (shards)
  const double sig = sqrt(innov[sp.seg] / count);
  double ls[D][D];
  ld_mat<D>(last ? cterm + sp.seg * D * D : suffix.l + (c + 1) * D * D, ls);
  double tn[B], tni[B];
  M::taus(a.grid, a.first, e, tn, tni);
  if (last && a.last) {
    double eta[D];
#pragma unroll
    for (int r = 0; r < D; ++r) eta[r] = eta_out_term[r];
    write_node<D, d>(o, out0 + e, tn, ls, eta, sig);
  }
  BwdGrid bg(a.grid, a.first, e - 1);
  for (int64_t k = e - 1; k >= s; --k) {
    double tk[B], tki[B], ratio[B], pc[B][B];
    M::taus_h(bg.step(k), tk, tki);
#pragma unroll
    for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tni[i];
    M::phi_coefs(ratio, pc);
    double E[D][D], gk[D], cfk[D][D], lk[D][D];
    soa_ld<D>(elems, c, k - s, E, gk);
    mat_ld<D>(cf, a.nchunks, c, k - s, cfk);
    smooth_factor<D, d>(pc, E, cfk, cst.q, lk);
    smooth_combine_factor<D>(E, lk, ls);
    double eta[D];
#pragma unroll
    for (int r = 0; r < D; ++r) eta[r] = eta_out[((k - s) * D + r) * a.nchunks + c];
    write_node<D, d>(o, out0 + k, tk, ls, eta, sig);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      tn[i] = tk[i];
      tni[i] = tki[i];
    }
  }
}

// ------------------------------------------------------------- pass E ---
// One thread per chunk: backward mean recursion m_n = g_n + E_n m_{n+1}
// from the chunk's incoming smoothed mean; new trajectory (original
// coordinates) and per-chunk objective / stopping partials.
// eta_old / eta_new (and their node-N slots) are in the chunk-interleaved
// layout of eta_at; the next step's (E, g, eta_old) are prefetched while the
// current step computes.
template <int D, int d, bool kInitial, bool kBatch = false>
__global__ void __launch_bounds__(kLaneThreads, kBwdMinBlocks) k_lane_bwd_down(FastArgs a, FastConst<D> cst, ElemSoA elems,
                                                                SEd suffix, const double* eta_old,
                                                                const double* old_term, double* eta_new,
                                                                double* new_term, double* part) {
  using M = Model<D, d>;
  constexpr int B = M::B;
  __shared__ double red[3][kLaneThreads];
  const int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t nc = a.nchunks;
  const SegPos sp = seg_pos<kBatch>(a, c < nc ? c : nc - 1);
  const bool okc = c < nc && (!kBatch || (sp.cl < sp.nreal && a.active[sp.seg]));
  double obj = 0.0, dmax = 0.0, emax = 0.0;
  if (a.it_dev != nullptr) {  // graph-loop mode: buffers by iteration parity
    const int par = *a.it_dev & 1;
    eta_old = par ? a.pair1 : a.pair0;
    old_term = eta_old + a.term_off;
    eta_new = par ? a.pair0 : a.pair1;
    new_term = eta_new + a.term_off;
  }
  if (okc) {
    if constexpr (kBatch) {  // this IVP's node-N slots
      old_term += sp.seg * D;
      new_term += sp.seg * D;
    }
    const int64_t s = sp.cl * a.L;
    const int64_t e = min(a.N, s + a.L);
    const bool last = sp.cl == sp.nreal - 1;
    double mu[D], te[B], tei[B];
    M::taus(a.grid, a.first, e, te, tei);
    double bar_next[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double eta_e;
      const double old_e = (e == a.N) ? old_term[r] : eta_old[r * nc + c + 1];  // the next chunk's node 0
      if (kInitial) {
        eta_e = old_e;
        mu[r] = 0.0;
      } else {
        mu[r] = last ? elems.term[sp.seg * D + r] : suffix.g[(c + 1) * D + r];
        eta_e = te[r % B] * mu[r];
      }
      if (last) {
        if (!kInitial) new_term[r] = eta_e;  // shards: the halo node, owned by the next shard
        if (a.last) {
          dmax = fmax(dmax, fabs(eta_e - old_e));
          emax = fmax(emax, fabs(eta_e));
        }
      }
      bar_next[r] = tei[r % B] * eta_e;
    }
    double tn[B];
#pragma unroll
    for (int i = 0; i < B; ++i) tn[i] = tei[i];  // T_{k+1}^-1
    // Register prefetch of the next step's (E, g, eta_old) where two D x D
    // blocks fit beside the recursion (D <= 7); at D = 8, 9 it spilled
    // (632 B of stack at D = 8), so those load at the top of each step from
    // the L2 lines prefetched below.
    constexpr bool kRegPre = D * D <= 49;
    constexpr int DP = kRegPre ? D : 1;
    double En[DP][DP], gn[DP], on[DP];
    if constexpr (kRegPre) {
      if (e - 1 >= s) {
        if (!kInitial) soa_ld<DP>(elems, c, e - 1 - s, En, gn);
#pragma unroll
        for (int r = 0; r < D; ++r) on[r] = eta_old[((e - 1 - s) * D + r) * nc + c];
      }
    }
    BwdGrid bg(a.grid, a.first, e - 1);
    for (int64_t k = e - 1; k >= s; --k) {
      double E[D][D], gk[D], oldk[D];
      if constexpr (kRegPre) {
#pragma unroll
        for (int r = 0; r < D; ++r) {
          gk[r] = gn[r];
          oldk[r] = on[r];
#pragma unroll
          for (int j = 0; j < D; ++j) E[r][j] = En[r][j];
        }
        if (k - 1 >= s) {
          if (!kInitial) soa_ld<DP>(elems, c, k - 1 - s, En, gn);
#pragma unroll
          for (int r = 0; r < D; ++r) on[r] = eta_old[((k - 1 - s) * D + r) * nc + c];
        }
      } else {
        if (!kInitial) soa_ld<D>(elems, c, k - s, E, gk);
#pragma unroll
        for (int r = 0; r < D; ++r) oldk[r] = eta_old[((k - s) * D + r) * nc + c];
      }
      if (!kInitial && k - 2 >= s) {
        // L2 prefetch of step k-2 for the whole warp (its 32 chunks span <= 3
        // lines per entry), so the register prefetch above hits L2: more
        // loads in flight without more registers.
        constexpr int X = D * D + 2 * D;
        const int lane = threadIdx.x & 31;
        const int64_t cw = c - lane, t2 = k - 2 - s;
        for (int q = lane; q < 3 * X; q += 32) {
          const int x = q / 3, part = q - 3 * (q / 3);
          const int64_t cc = min(nc - 1, cw + (part == 0 ? 0 : (part == 1 ? 16 : 31)));
          const double* addr = x < D * D ? elems.e + (t2 * D * D + x) * nc + cc
                                         : (x < D * D + D ? elems.g + (t2 * D + (x - D * D)) * nc + cc
                                                          : eta_old + (t2 * D + (x - D * D - D)) * nc + cc);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(addr));
        }
      }
      double tk[B], tki[B];
      M::taus_h(bg.step(k), tk, tki);
      double etak[D];
      if (kInitial) {
#pragma unroll
        for (int r = 0; r < D; ++r) etak[r] = oldk[r];
      } else {
        double nm[D];
#pragma unroll
        for (int r = 0; r < D; ++r) {
          double acc = gk[r];
#pragma unroll
          for (int j = 0; j < D; ++j) acc = fma(E[r][j], mu[j], acc);
          nm[r] = acc;
        }
#pragma unroll
        for (int r = 0; r < D; ++r) {
          mu[r] = nm[r];
          etak[r] = tk[r % B] * nm[r];
          eta_new[((k - s) * D + r) * nc + c] = etak[r];
        }
      }
      double bar[D];
#pragma unroll
      for (int r = 0; r < D; ++r) {
        dmax = fmax(dmax, fabs(etak[r] - oldk[r]));
        emax = fmax(emax, fabs(etak[r]));
        bar[r] = tki[r % B] * etak[r];
      }
      // objective term: || Qunit^-1/2 (bar_{k+1} - phi_k bar_k) ||^2
      double ratio[B], pc[B][B], pb[D];
#pragma unroll
      for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tn[i];
      M::phi_coefs(ratio, pc);
#pragma unroll
      for (int r = 0; r < D; ++r) pb[r] = bar[r];
      M::phi_vec(pc, pb);
      double w[D], acc2 = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double acc = bar_next[i] - pb[i];
#pragma unroll
        for (int k2 = 0; k2 < i; ++k2) acc = fma(-cst.qunit[i * D + k2], w[k2], acc);
        w[i] = acc * cst.qunit_rdiag[i];
        acc2 = fma(w[i], w[i], acc2);
      }
      obj += acc2;
#pragma unroll
      for (int r = 0; r < D; ++r) bar_next[r] = bar[r];
#pragma unroll
      for (int i = 0; i < B; ++i) tn[i] = tki[i];
    }
  }
  red[0][threadIdx.x] = obj;
  red[1][threadIdx.x] = dmax;
  red[2][threadIdx.x] = emax;
  __syncthreads();
  for (int st = kLaneThreads / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      red[0][threadIdx.x] += red[0][threadIdx.x + st];
      red[1][threadIdx.x] = fmax(red[1][threadIdx.x], red[1][threadIdx.x + st]);
      red[2][threadIdx.x] = fmax(red[2][threadIdx.x], red[2][threadIdx.x + st]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x * 3 + 0] = red[0][0];
    part[blockIdx.x * 3 + 1] = red[1][0];
    part[blockIdx.x * 3 + 2] = red[2][0];
  }
}

}  // namespace lane
}  // namespace pode
