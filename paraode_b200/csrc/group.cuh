// Group-of-lanes dense fp64 linear algebra for small state dimensions D.
//
// Execution model (B200, sm_100a): a warp is split into 32/D "groups" of D
// consecutive lanes; each group owns one element / one time-chunk.  Lane r of
// a group holds ROW r of every D x D matrix (and of every 2D-row stacked
// matrix, in two slots) in registers, and entry r of every D-vector.  Rows
// are shared inside the group through a per-group shared-memory scratch tile
// (publish -> __syncwarp -> broadcast reads), so a D x D product costs D^2
// FMAs per lane and D^2/2 128-bit broadcast loads instead of D^2 shuffles.
// Lanes left over when D does not divide 32 form a phantom group that
// computes on junk and never stores.
//
// The arithmetic restates the reference's square-root operators
// (proj/src/linalg.cpp tria = Householder QR of M^T, Eigen's sign convention;
// proj/src/sequential.cpp, proj/src/parallel.cpp) in row form: an LQ of the
// stacked matrix with one Householder reflector per pivot row.
#pragma once

#include <cuda_runtime.h>
#include <cfloat>
#include <cstdint>

namespace pode {

template <int K>
struct Rw {
  double v[K];
  __device__ __forceinline__ double& operator[](int i) { return v[i]; }
  __device__ __forceinline__ double operator[](int i) const { return v[i]; }
};

template <int K>
__device__ __forceinline__ Rw<K> zeros() {
  Rw<K> o;
#pragma unroll
  for (int j = 0; j < K; ++j) o[j] = 0.0;
  return o;
}

// Per-group scratch: a (2D) x (2D) tile plus two D-vectors.
template <int D>
struct Scratch {
  static constexpr int kTile = 4 * D * D;
  // vector area: [0,D) factor inverse diagonal, [D,2D) gather slot,
  // [2D,3D) spare slot, [3D, 5D+2) LQ reflector.
  static constexpr int kRaw = kTile + 6 * D + 4;
  // Group stride = 2 (mod 16) doubles: the groups of a warp then start on
  // distinct 4-word bank slots, so the group-broadcast reads of mm/publish
  // (every group reading its own tile) are one wavefront instead of up to
  // three (ncu: ~50 % of shared-load wavefronts were bank conflicts), and
  // every tile stays 16-byte aligned for double2 rows.
  static constexpr int kDoubles = kRaw + (18 - kRaw % 16) % 16;
};

template <int D>
struct Grp {
  static constexpr int kPerWarp = 32 / D;             // real groups per warp
  static constexpr int kSlots = kPerWarp + ((32 % D) ? 1 : 0);  // + phantom
  int r;       // row owned by this lane (0..D-1)
  int gw;      // group index inside the warp (kPerWarp = phantom)
  double* sc;  // group scratch tile
  double* vs;  // group scratch vector area (>= 4 D doubles)

  __device__ __forceinline__ static Grp make(double* warp_scratch) {
    Grp g;
    const int lane = threadIdx.x & 31;
    g.gw = lane / D;
    g.r = lane - g.gw * D;
    g.sc = warp_scratch + g.gw * Scratch<D>::kDoubles;
    g.vs = g.sc + Scratch<D>::kTile;
    return g;
  }
  __device__ __forceinline__ bool real() const { return gw < kPerWarp; }
};

__device__ __forceinline__ void wsync() { __syncwarp(); }

// ----------------------------------------------------------- publishing ---
// Tile rows of even length move as double2 (16-byte shared accesses; tiles
// and row starts are 16-byte aligned then), odd ones element-wise.
template <int K>
__device__ __forceinline__ void st_tile_row(double* p, const Rw<K>& x) {
  if constexpr (K % 2 == 0) {
#pragma unroll
    for (int j = 0; j < K / 2; ++j) reinterpret_cast<double2*>(p)[j] = make_double2(x[2 * j], x[2 * j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) p[j] = x[j];
  }
}
template <int K>
__device__ __forceinline__ Rw<K> ld_tile_row(const double* p) {
  Rw<K> x;
  if constexpr (K % 2 == 0) {
#pragma unroll
    for (int j = 0; j < K / 2; ++j) {
      const double2 v = reinterpret_cast<const double2*>(p)[j];
      x[2 * j] = v.x;
      x[2 * j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) x[j] = p[j];
  }
  return x;
}

// Writes this lane's row into the tile (row stride K) bracketed by warp
// barriers: the leading one protects readers of the previous contents.
template <int D, int K>
__device__ __forceinline__ void publish(const Grp<D>& g, const Rw<K>& row) {
  wsync();
  st_tile_row<K>(g.sc + g.r * K, row);
  wsync();
}

// Two stacked row sets: rows 0..D-1 = a, D..2D-1 = b (stride K).
template <int D, int K>
__device__ __forceinline__ void publish2(const Grp<D>& g, const Rw<K>& a, const Rw<K>& b) {
  wsync();
  st_tile_row<K>(g.sc + g.r * K, a);
  st_tile_row<K>(g.sc + (D + g.r) * K, b);
  wsync();
}

template <int D>
__device__ __forceinline__ void publish_vec(const Grp<D>& g, double x, int slot = 1) {
  wsync();
  g.vs[slot * D + g.r] = x;
  wsync();
}

// --------------------------------------------------------- vector forms ---
template <int D>
__device__ __forceinline__ Rw<D> gather_vec(const Grp<D>& g, double x) {
  publish_vec(g, x);
  return ld_tile_row<D>(g.vs + D);
}

// y = A x  (A rows on lanes, x distributed) -> y_r on lane r.
template <int D>
__device__ __forceinline__ double matvec(const Grp<D>& g, const Rw<D>& a, double x) {
  const Rw<D> xv = gather_vec(g, x);
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) acc = fma(a[k], xv[k], acc);
  return acc;
}

// y = A^T x -> y_r = sum_k A[k][r] x_k.
template <int D>
__device__ __forceinline__ double matvec_t(const Grp<D>& g, const Rw<D>& a, double x) {
  wsync();
  st_tile_row<D>(g.sc + g.r * D, a);
  g.vs[D + g.r] = x;
  wsync();
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) acc = fma(g.sc[k * D + g.r], g.vs[D + k], acc);
  return acc;
}

// Sum over the group of a per-lane value (every lane gets the total, summed
// in lane order so all lanes agree bitwise).
template <int D>
__device__ __forceinline__ double group_sum(const Grp<D>& g, double x) {
  const Rw<D> v = gather_vec(g, x);
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) s += v[k];
  return s;
}

template <int D>
__device__ __forceinline__ double group_max(const Grp<D>& g, double x) {
  const Rw<D> v = gather_vec(g, x);
  double s = v[0];
#pragma unroll
  for (int k = 1; k < D; ++k) s = fmax(s, v[k]);
  return s;
}

// --------------------------------------------------------- matrix forms ---
// C = A B
template <int D, int K>
__device__ __forceinline__ Rw<K> mm(const Grp<D>& g, const Rw<D>& a, const Rw<K>& b) {
  publish<D, K>(g, b);
  Rw<K> c = zeros<K>();
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double ak = a[k];
    const Rw<K> bk = ld_tile_row<K>(g.sc + k * K);
#pragma unroll
    for (int j = 0; j < K; ++j) c[j] = fma(ak, bk[j], c[j]);
  }
  return c;
}

// C = A B^T  (C[r][j] = row_r(A) . row_j(B))
template <int D>
__device__ __forceinline__ Rw<D> mm_nt(const Grp<D>& g, const Rw<D>& a, const Rw<D>& b) {
  publish<D, D>(g, b);
  Rw<D> c;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const Rw<D> bj = ld_tile_row<D>(g.sc + j * D);
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) acc = fma(a[k], bj[k], acc);
    c[j] = acc;
  }
  return c;
}

// C = A^T B  (C[r][j] = sum_k A[k][r] B[k][j])
template <int D>
__device__ __forceinline__ Rw<D> mm_tn(const Grp<D>& g, const Rw<D>& a, const Rw<D>& b) {
  publish2<D, D>(g, a, b);
  Rw<D> c = zeros<D>();
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double akr = g.sc[k * D + g.r];
    const Rw<D> bk = ld_tile_row<D>(g.sc + (D + k) * D);
#pragma unroll
    for (int j = 0; j < D; ++j) c[j] = fma(akr, bk[j], c[j]);
  }
  return c;
}

// Row r of A^T.
template <int D>
__device__ __forceinline__ Rw<D> transpose(const Grp<D>& g, const Rw<D>& a) {
  publish<D, D>(g, a);
  Rw<D> t;
#pragma unroll
  for (int j = 0; j < D; ++j) t[j] = g.sc[j * D + g.r];
  return t;
}

// ------------------------------------------------------------------ LQ ---
// Householder LQ ("tria") of a stacked matrix held in rows:
//   rows 0..NT-1      : top[] on lanes 0..NT-1 (lanes >= NT must hold zeros)
//   rows NT..NT+NB-1  : bot[] on lanes 0..NB-1 (NB <= D; other lanes zero)
// with K columns.  Pivot p eliminates row p against column p for
// p < min(NT + NB, K), exactly as Eigen's unblocked HouseholderQR does on the
// transpose (beta = -sign(c0) ||x||, essential = tail / (c0 - beta),
// tau = (beta - c0) / beta; tau = 0 when ||tail||^2 <= DBL_MIN).  On return
// the rows hold L (lower triangular in pivot order); L L^T = M M^T.
// Sum of squares of x[lo..K) with four independent accumulators (short
// dependency chains; every lane evaluates it identically).
// Structural sparsity of the stacked trias [L | T] used here: when the right
// block (columns >= S) is lower triangular in every row, then before pivot p
// every row is zero in columns > S + p (each pivot row's reflector only
// reaches S + p, by induction), so those columns are skipped.  S = K means
// no structure.  (Pure zeros are skipped: the arithmetic is unchanged.)
__device__ __forceinline__ constexpr bool live_col(int j, int p, int S) { return j < S || j <= S + p; }

template <int K, int S = K>
__device__ __forceinline__ double sumsq_from(const Rw<K>& x, int lo, int p) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int j = lo; j < K; ++j) {
    if (!live_col(j, p, S)) continue;
    const int s = (j - lo) & 3;
    if (s == 0) a0 = fma(x[j], x[j], a0);
    if (s == 1) a1 = fma(x[j], x[j], a1);
    if (s == 2) a2 = fma(x[j], x[j], a2);
    if (s == 3) a3 = fma(x[j], x[j], a3);
  }
  return (a0 + a1) + (a2 + a3);
}

template <int K, int S = K>
__device__ __forceinline__ double dot_from(const Rw<K>& x, const Rw<K>& y, int lo, double init, int p) {
  double a0 = init, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int j = lo; j < K; ++j) {
    if (!live_col(j, p, S)) continue;
    const int s = (j - lo) & 3;
    if (s == 0) a0 = fma(x[j], y[j], a0);
    if (s == 1) a1 = fma(x[j], y[j], a1);
    if (s == 2) a2 = fma(x[j], y[j], a2);
    if (s == 3) a3 = fma(x[j], y[j], a3);
  }
  return (a0 + a1) + (a2 + a3);
}

// Householder reflector of x[p..K) in Eigen's convention; every lane of the
// group computes it redundantly from the shuffled pivot row (no owner-only
// serial section, no shared-memory round trip).
template <int K>
struct Reflector {
  double tau, beta;
  Rw<K> ess;  // ess[j], j > p
};

// Branch-free fp64 reciprocal square root and reciprocal: the MUFU
// approximation refined by Newton steps to full double precision (no
// IEEE slow-path calls, so a whole Householder sweep stays one basic block).
// Inputs are positive normal numbers here (guarded by the callers).
// PODE_NEWTON_ITERS refinements (the MUFU seed has ~2^-23 relative error,
// Newton squares it: two steps reach 2^-46 -> 2^-92, below fp64 rounding).
#ifndef PODE_NEWTON_ITERS
#define PODE_NEWTON_ITERS 2
#endif
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
#pragma unroll
  for (int i = 0; i < PODE_NEWTON_ITERS; ++i) y = y * fma(-hx * y, y, 1.5);
  return y;
}

__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < PODE_NEWTON_ITERS; ++i) {
    const double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
  }
  return y;
}

// Householder coefficients of x = [c0, tail] (Eigen's makeHouseholder):
// beta = -sign(c0) ||x||, tau = (beta - c0) / beta, inv = 1 / (c0 - beta);
// (tau, beta, inv) = (0, c0, 0) when ||tail||^2 <= DBL_MIN.  Branch-free.
__device__ __forceinline__ void householder_coefs(double c0, double tail, double& tau, double& beta, double& inv) {
  const bool live = tail > DBL_MIN;
  const double n2 = fma(c0, c0, tail);
  const double r = rsqrt_nr(live ? n2 : 1.0);  // 1 / ||x||
  const double sgn = (c0 >= 0.0) ? -1.0 : 1.0;
  const double b = sgn * (n2 * r);              // -sign(c0) ||x||
  const double rb = sgn * r;                    // 1 / beta
  const double ic = rcp_nr(live ? (c0 - b) : 1.0);
  tau = live ? (b - c0) * rb : 0.0;
  beta = live ? b : c0;
  inv = live ? ic : 0.0;
}

template <int K, int S = K>
__device__ __forceinline__ Reflector<K> make_reflector(const Rw<K>& x, int p) {
  Reflector<K> h;
  const double tail = sumsq_from<K, S>(x, p + 1, p);
  double inv;
  householder_coefs(x[p], tail, h.tau, h.beta, inv);
#pragma unroll
  for (int j = p + 1; j < K; ++j) h.ess[j] = live_col(j, p, S) ? x[j] * inv : 0.0;
  return h;
}

// y <- y (I - tau v v^T), v = [1, ess] on columns p..K-1.
template <int K, int S = K>
__device__ __forceinline__ void apply_reflector(const Reflector<K>& h, int p, Rw<K>& y) {
  const double w = dot_from<K, S>(y, h.ess, p + 1, y[p], p);
  const double tw = h.tau * w;
  y[p] -= tw;
#pragma unroll
  for (int j = p + 1; j < K; ++j)
    if (live_col(j, p, S)) y[j] = fma(-tw, h.ess[j], y[j]);
}

// Row p of a register row set, fetched from its owner lane.
template <int D, int K, int S = K>
__device__ __forceinline__ Rw<K> shfl_row(const Grp<D>& g, const Rw<K>& row, int owner, int from) {
  const int src = (threadIdx.x & 31) - g.r + owner;
  Rw<K> x;
#pragma unroll
  for (int j = 0; j < K; ++j)
    x[j] = (j >= from && live_col(j, from, S)) ? __shfl_sync(0xffffffffu, row[j], src) : 0.0;
  return x;
}

template <int D, int NT, int NB, int K, int S = K>
__device__ __forceinline__ void lq(const Grp<D>& g, Rw<K>& top, Rw<K>& bot) {
  constexpr int kPivots = (NT + NB < K) ? (NT + NB) : K;
#pragma unroll
  for (int p = 0; p < kPivots; ++p) {
    const bool in_top = p < NT;
    const int owner = in_top ? p : p - NT;
    const Reflector<K> h = make_reflector<K, S>(shfl_row<D, K, S>(g, in_top ? top : bot, owner, p), p);
    const double tau = h.tau;
    const double beta = h.beta;
    const Rw<K>& ess = h.ess;
    // Apply H = I - tau v v^T (v = [1, ess]) from the right to every row but
    // the pivot row; rows already reduced have zeros from column p on, so the
    // update leaves them unchanged.
    (void)tau;
    (void)ess;
    // Rows already reduced have zeros from column p on, so applying the
    // reflector to every row leaves them unchanged; the pivot row itself
    // becomes [.., beta, 0, ..] (branch-free select, no divergence).
    const bool own = g.r == owner;
    if (in_top) {
      apply_reflector<K, S>(h, p, top);
      apply_reflector<K, S>(h, p, bot);
      if (own) {
        top[p] = beta;
#pragma unroll
        for (int j = p + 1; j < K; ++j) top[j] = 0.0;
      }
    } else {
      apply_reflector<K, S>(h, p, bot);
      if (own) {
        bot[p] = beta;
#pragma unroll
        for (int j = p + 1; j < K; ++j) bot[j] = 0.0;
      }
    }
  }
}

// Two independent LQs of D x K row sets run in one pivot sweep (their
// reflectors are independent, so the two dependency chains overlap).
template <int D, int K, int S = K>
__device__ __forceinline__ void lq_pair(const Grp<D>& g, Rw<K>& a, Rw<K>& b) {
  constexpr int kPivots = (D < K) ? D : K;
#pragma unroll
  for (int p = 0; p < kPivots; ++p) {
    const Reflector<K> ha = make_reflector<K, S>(shfl_row<D, K, S>(g, a, p, p), p);
    const Reflector<K> hb = make_reflector<K, S>(shfl_row<D, K, S>(g, b, p, p), p);
    apply_reflector<K, S>(ha, p, a);
    apply_reflector<K, S>(hb, p, b);
    if (g.r == p) {
      a[p] = ha.beta;
      b[p] = hb.beta;
#pragma unroll
      for (int j = p + 1; j < K; ++j) {
        a[j] = 0.0;
        b[j] = 0.0;
      }
    }
  }
}

// Single row set: tria of a D x K matrix (K >= D) -> rows of L (first D cols).
template <int D, int K, int S = K>
__device__ __forceinline__ Rw<D> tria(const Grp<D>& g, Rw<K> m) {
  Rw<K> none = zeros<K>();
  lq<D, 0, D, K, S>(g, none, m);
  Rw<D> o;
#pragma unroll
  for (int j = 0; j < D; ++j) o[j] = m[j];
  return o;
}

// sqrt_sum(A, B) = tria([A B]) for D x D factors (general B).
template <int D>
__device__ __forceinline__ Rw<D> sqrt_sum(const Grp<D>& g, const Rw<D>& a, const Rw<D>& b) {
  Rw<2 * D> m;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    m[j] = a[j];
    m[D + j] = b[j];
  }
  return tria<D, 2 * D>(g, m);
}

// sqrt_sum for a lower-triangular B (skips its structural zeros).
template <int D>
__device__ __forceinline__ Rw<D> sqrt_sum_lt(const Grp<D>& g, const Rw<D>& a, const Rw<D>& b) {
  Rw<2 * D> m;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    m[j] = a[j];
    m[D + j] = b[j];
  }
  return tria<D, 2 * D, D>(g, m);
}

// ----------------------------------------------------- triangular solves ---
// The factor L (lower, D x D) is published once; every lane then solves its
// own row — no cross-lane dependency chain.
//   solve_xlt: x L^T = b  (x = b L^-T; forward substitution with L)
//   solve_xl : x L   = b  (x = b L^-1;  back substitution with L^T)
template <int D, int K>
__device__ __forceinline__ void publish_factor(const Grp<D>& g, const Rw<K>& l_row) {
  wsync();
  st_tile_row<D>(g.sc + g.r * D, l_row);
  g.vs[g.r] = 1.0 / l_row[g.r];
  wsync();
}

template <int D, int KB>
__device__ __forceinline__ Rw<KB> solve_xlt(const Grp<D>& g, const Rw<KB>& b) {
  // x L^T = b  <=>  L x^T = b^T, KB = D.
  Rw<KB> x;
#pragma unroll
  for (int i = 0; i < KB; ++i) {
    double acc = b[i];
#pragma unroll
    for (int k = 0; k < i; ++k) acc = fma(-g.sc[i * D + k], x[k], acc);
    x[i] = acc * g.vs[i];
  }
  return x;
}

template <int D, int KB>
__device__ __forceinline__ Rw<KB> solve_xl(const Grp<D>& g, const Rw<KB>& b) {
  // x L = b  <=>  L^T x^T = b^T (upper), KB = D.
  Rw<KB> x;
#pragma unroll
  for (int i = KB - 1; i >= 0; --i) {
    double acc = b[i];
#pragma unroll
    for (int k = i + 1; k < KB; ++k) acc = fma(-g.sc[k * D + i], x[k], acc);
    x[i] = acc * g.vs[i];
  }
  return x;
}

// Redundant per-lane forward substitution of a distributed vector against
// the published factor: returns the full solution w = L^-1 v on every lane.
template <int D>
__device__ __forceinline__ Rw<D> solve_vec_lower_all(const Grp<D>& g, const Rw<D>& v) {
  Rw<D> w;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double acc = v[i];
#pragma unroll
    for (int k = 0; k < i; ++k) acc = fma(-g.sc[i * D + k], w[k], acc);
    w[i] = acc * g.vs[i];
  }
  return w;
}

// Singularity test of a published-or-owned triangular factor
// (proj/src/linalg.cpp:54-62): |L_ii| <= 1e-13 max_j |L_jj|.
template <int D>
__device__ __forceinline__ bool singular_diag(const Grp<D>& g, double diag, int n_valid) {
  const double a = (g.r < n_valid) ? fabs(diag) : 0.0;
  const double mx = group_max(g, a);
  const double mine = group_max(g, (g.r < n_valid && a <= 1e-13 * mx) ? 1.0 : 0.0);
  return mine > 0.0;
}

// Entry idx of a register row without dynamic register indexing.
template <int K>
__device__ __forceinline__ double pick(const Rw<K>& x, int idx) {
  double v = 0.0;
#pragma unroll
  for (int j = 0; j < K; ++j) v = (j == idx) ? x[j] : v;
  return v;
}

template <int K>
__device__ __forceinline__ bool row_finite(const Rw<K>& x) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < K; ++j) ok &= isfinite(x[j]);
  return ok;
}

}  // namespace pode
