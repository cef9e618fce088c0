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
  static constexpr int kDoubles = kTile + 6 * D + 4;
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
// Writes this lane's row into the tile (row stride K) bracketed by warp
// barriers: the leading one protects readers of the previous contents.
template <int D, int K>
__device__ __forceinline__ void publish(const Grp<D>& g, const Rw<K>& row) {
  wsync();
#pragma unroll
  for (int j = 0; j < K; ++j) g.sc[g.r * K + j] = row[j];
  wsync();
}

// Two stacked row sets: rows 0..D-1 = a, D..2D-1 = b (stride K).
template <int D, int K>
__device__ __forceinline__ void publish2(const Grp<D>& g, const Rw<K>& a, const Rw<K>& b) {
  wsync();
#pragma unroll
  for (int j = 0; j < K; ++j) {
    g.sc[g.r * K + j] = a[j];
    g.sc[(D + g.r) * K + j] = b[j];
  }
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
  Rw<D> o;
#pragma unroll
  for (int k = 0; k < D; ++k) o[k] = g.vs[D + k];
  return o;
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
#pragma unroll
  for (int j = 0; j < D; ++j) g.sc[g.r * D + j] = a[j];
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
#pragma unroll
    for (int j = 0; j < K; ++j) c[j] = fma(ak, g.sc[k * K + j], c[j]);
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
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) acc = fma(a[k], g.sc[j * D + k], acc);
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
#pragma unroll
    for (int j = 0; j < D; ++j) c[j] = fma(akr, g.sc[(D + k) * D + j], c[j]);
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
template <int D, int NT, int NB, int K>
__device__ __forceinline__ void lq(const Grp<D>& g, Rw<K>& top, Rw<K>& bot) {
  constexpr int kPivots = (NT + NB < K) ? (NT + NB) : K;
  double* vb = g.vs + 3 * D;  // reflector: vb[0] = tau, vb[1 + j] = essential_j (j > p)
#pragma unroll
  for (int p = 0; p < kPivots; ++p) {
    const bool in_top = p < NT;
    const int owner = in_top ? p : p - NT;
    wsync();
    if (g.r == owner) {
      const Rw<K>& row = in_top ? top : bot;
      double tail = 0.0;
#pragma unroll
      for (int j = p + 1; j < K; ++j) tail = fma(row[j], row[j], tail);
      const double c0 = row[p];
      double tau = 0.0, beta = c0, inv = 0.0;
      if (tail > DBL_MIN) {
        beta = sqrt(fma(c0, c0, tail));
        if (c0 >= 0.0) beta = -beta;
        inv = 1.0 / (c0 - beta);
        tau = (beta - c0) / beta;
      }
      vb[0] = tau;
#pragma unroll
      for (int j = p + 1; j < K; ++j) vb[1 + j] = row[j] * inv;
      vb[1] = beta;
    }
    wsync();
    const double tau = vb[0];
    const double beta = vb[1];
    Rw<K> ess;
#pragma unroll
    for (int j = p + 1; j < K; ++j) ess[j] = vb[1 + j];
    // Apply H = I - tau v v^T (v = [1, ess]) from the right to every row but
    // the pivot row; rows already reduced have zeros from column p on, so the
    // update leaves them unchanged.
    auto apply = [&](Rw<K>& y) {
      double w = y[p];
#pragma unroll
      for (int j = p + 1; j < K; ++j) w = fma(y[j], ess[j], w);
      const double tw = tau * w;
      y[p] -= tw;
#pragma unroll
      for (int j = p + 1; j < K; ++j) y[j] = fma(-tw, ess[j], y[j]);
    };
    if (in_top) {
      if (g.r == owner) {
        top[p] = beta;
#pragma unroll
        for (int j = p + 1; j < K; ++j) top[j] = 0.0;
      } else {
        apply(top);
      }
      apply(bot);
    } else {
      if (g.r == owner) {
        bot[p] = beta;
#pragma unroll
        for (int j = p + 1; j < K; ++j) bot[j] = 0.0;
      } else {
        apply(bot);
      }
    }
  }
}

// Single row set: tria of a D x K matrix (K >= D) -> rows of L (first D cols).
template <int D, int K>
__device__ __forceinline__ Rw<D> tria(const Grp<D>& g, Rw<K> m) {
  Rw<K> none = zeros<K>();
  lq<D, 0, D, K>(g, none, m);
  Rw<D> o;
#pragma unroll
  for (int j = 0; j < D; ++j) o[j] = m[j];
  return o;
}

// sqrt_sum(A, B) = tria([A B]) for D x D factors.
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

// ----------------------------------------------------- triangular solves ---
// The factor L (lower, D x D) is published once; every lane then solves its
// own row — no cross-lane dependency chain.
//   solve_xlt: x L^T = b  (x = b L^-T; forward substitution with L)
//   solve_xl : x L   = b  (x = b L^-1;  back substitution with L^T)
template <int D, int K>
__device__ __forceinline__ void publish_factor(const Grp<D>& g, const Rw<K>& l_row) {
  wsync();
#pragma unroll
  for (int j = 0; j < D; ++j) g.sc[g.r * D + j] = l_row[j];
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
