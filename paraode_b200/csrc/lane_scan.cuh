// Lane-serial associative scans over element arrays: one chunk of L
// elements per THREAD (reduce-then-scan, the tree of engine.cuh with the
// combine evaluated by a single lane).  Used for the chunk-aggregate scans of
// the fused IEKS iteration, where only a few thousand elements remain and
// the critical path is the latency of one combine.
//
//   ⊗_f (parallel.cpp:67-100): Xi = tria([[C_i^T J_j, I], [J_j, 0]]) — only
//   the first D pivots are formed (they give Xi11, Xi21; the remaining block
//   R satisfies R R^T = Xi22 Xi22^T and enters J only through another tria).
//   ⊗_s on means (E, g) (parallel.cpp:146-156).
#pragma once

#include "lane.cuh"

namespace pode {
namespace lane {

template <int D>
struct LF {  // filtering element in registers (full row-major matrices)
  double a[D][D], c[D][D], j[D][D], b[D], eta[D];
};

template <int D>
__device__ __forceinline__ void load_f(const FEd& x, int64_t i, LF<D>& e) {
  ld_mat<D>(x.a + i * D * D, e.a);
  ld_mat<D>(x.c + i * D * D, e.c);
  ld_mat<D>(x.j + i * D * D, e.j);
#pragma unroll
  for (int r = 0; r < D; ++r) {
    e.b[r] = x.b[i * D + r];
    e.eta[r] = x.eta[i * D + r];
  }
}

template <int D>
__device__ __forceinline__ void store_f(const FEd& x, int64_t i, const LF<D>& e) {
  st_mat<D>(x.a + i * D * D, e.a);
  st_mat<D>(x.c + i * D * D, e.c);
  st_mat<D>(x.j + i * D * D, e.j);
#pragma unroll
  for (int r = 0; r < D; ++r) {
    x.b[i * D + r] = e.b[r];
    x.eta[i * D + r] = e.eta[r];
  }
}

// out = li ⊗_f rj; returns false if Xi11 is singular.  Not inlined: the
// unrolled body is large enough that ptxas allocates registers far better
// for it as a separate function (the operands then live in L1-resident
// local memory).
template <int D>
__device__ __noinline__ bool combine_f(const LF<D>& li, const LF<D>& rj, LF<D>& out) {
  double m[2 * D][2 * D];
  // top rows [C_i^T J_j, I], bottom rows [J_j, 0]
#pragma unroll
  for (int r = 0; r < D; ++r) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int x = 0; x < D; ++x) acc = fma(li.c[x][r], rj.j[x][c], acc);
      m[r][c] = acc;
      m[r][D + c] = (r == c) ? 1.0 : 0.0;
      m[D + r][c] = rj.j[r][c];
      m[D + r][D + c] = 0.0;
    }
  }
  lq<2 * D, 2 * D, D>(m);
  double xi11[D][D];
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int c = 0; c < D; ++c) xi11[r][c] = (c <= r) ? m[r][c] : 0.0;
  const bool sing = singular_diag<D>(xi11, D);
  double rd[D];
#pragma unroll
  for (int i = 0; i < D; ++i) rd[i] = rcp_nr(xi11[i][i]);
  // W = C_i Xi11^-T  (row r: w Xi11^T = C_i[r], forward substitution)
  double w[D][D];
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double acc = li.c[r][i];
#pragma unroll
      for (int k = 0; k < i; ++k) acc = fma(-xi11[i][k], w[r][k], acc);
      w[r][i] = acc * rd[i];
    }
  // G = I - W Xi21^T
  double g[D][D];
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double acc = (r == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) acc = fma(-w[r][k], m[D + c][k], acc);
      g[r][c] = acc;
    }
  // AG = A_j G; A = AG A_i
  double ag[D][D];
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) acc = fma(rj.a[r][k], g[k][c], acc);
      ag[r][c] = acc;
    }
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) acc = fma(ag[r][k], li.a[k][c], acc);
      out.a[r][c] = acc;
    }
  // b = AG (b_i + C_i (C_i^T eta_j)) + b_j
  double t1[D], t3[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) acc = fma(li.c[k][r], rj.eta[k], acc);
    t1[r] = acc;
  }
#pragma unroll
  for (int r = 0; r < D; ++r) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) acc = fma(li.c[r][k], t1[k], acc);
    t3[r] = li.b[r] + acc;
  }
#pragma unroll
  for (int r = 0; r < D; ++r) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) acc = fma(ag[r][k], t3[k], acc);
    out.b[r] = acc + rj.b[r];
  }
  // eta = (G A_i)^T (eta_j - J_j (J_j^T b_i)) + eta_i
  double u1[D], u3[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) acc = fma(rj.j[k][r], li.b[k], acc);
    u1[r] = acc;
  }
#pragma unroll
  for (int r = 0; r < D; ++r) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) acc = fma(rj.j[r][k], u1[k], acc);
    u3[r] = rj.eta[r] - acc;
  }
  double gu[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {  // G^T u3
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) acc = fma(g[k][r], u3[k], acc);
    gu[r] = acc;
  }
#pragma unroll
  for (int r = 0; r < D; ++r) {  // A_i^T (G^T u3) + eta_i
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) acc = fma(li.a[k][r], gu[k], acc);
    out.eta[r] = acc + li.eta[r];
  }
  // C = tria([A_j W, C_j])
  {
    double s[D][2 * D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) acc = fma(rj.a[r][k], w[k][c], acc);
        s[r][c] = acc;
        s[r][D + c] = rj.c[r][c];
      }
    lq<D, 2 * D, D>(s);
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) out.c[r][c] = (c <= r) ? s[r][c] : 0.0;
  }
  // J = tria([A_i^T R, J_i]),  R = bottom-right block after the D pivots
  {
    double s[D][2 * D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) acc = fma(li.a[k][r], m[D + k][D + c], acc);
        s[r][c] = acc;
        s[r][D + c] = li.j[r][c];
      }
    lq<D, 2 * D, D>(s);
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) out.j[r][c] = (c <= r) ? s[r][c] : 0.0;
  }
  return !sing;
}

template <int D>
struct LFOps {
  using El = LF<D>;
  using Arr = FEd;
  __device__ static void load(const Arr& x, int64_t i, El& e) { load_f<D>(x, i, e); }
  __device__ static void store(const Arr& x, int64_t i, const El& e) { store_f<D>(x, i, e); }
  __device__ static bool combine(const El& l, const El& r, El& o) { return combine_f<D>(l, r, o); }
};

template <int D>
struct LM {  // mean-only smoothing element (E, g)
  double e[D][D], g[D];
};

template <int D>
struct LMOps {
  using El = LM<D>;
  using Arr = SEd;
  __device__ static void load(const Arr& x, int64_t i, El& e) {
    ld_mat<D>(x.e + i * D * D, e.e);
#pragma unroll
    for (int r = 0; r < D; ++r) e.g[r] = x.g[i * D + r];
  }
  __device__ static void store(const Arr& x, int64_t i, const El& e) {
    st_mat<D>(x.e + i * D * D, e.e);
#pragma unroll
    for (int r = 0; r < D; ++r) x.g[i * D + r] = e.g[r];
  }
  __device__ static bool combine(const El& l, const El& rr, El& o) {
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double og = l.g[r];
#pragma unroll
      for (int c = 0; c < D; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) acc = fma(l.e[r][k], rr.e[k][c], acc);
        o.e[r][c] = acc;
      }
#pragma unroll
      for (int k = 0; k < D; ++k) og = fma(l.e[r][k], rr.g[k], og);
      o.g[r] = og;
    }
    return true;
  }
};

template <int D, class Op>
__global__ void __launch_bounds__(kLaneThreads) k_lscan_reduce(typename Op::Arr x, int64_t n, int L,
                                                               typename Op::Arr agg, DevError* err) {
  const int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t lo = c * L;
  if (lo >= n) return;
  const int64_t hi = min(n, lo + L);
  typename Op::El acc, e, tmp;
  Op::load(x, lo, acc);
  bool bad = false;
  for (int64_t k = lo + 1; k < hi; ++k) {
    Op::load(x, k, e);
    bad |= !Op::combine(acc, e, tmp);
    acc = tmp;
  }
  if (bad) raise_error(err, lo, kErrSingular);
  Op::store(agg, c, acc);
}

template <int D, class Op, bool kReverse>
__global__ void __launch_bounds__(kLaneThreads) k_lscan_down(typename Op::Arr x, int64_t n, int L,
                                                             typename Op::Arr aggs, int64_t nchunks,
                                                             typename Op::Arr out, DevError* err) {
  const int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t lo = c * L;
  if (lo >= n) return;
  const int64_t hi = min(n, lo + L);
  const int64_t carry = kReverse ? c + 1 : c - 1;
  const bool have_carry = carry >= 0 && carry < nchunks;
  typename Op::El acc, e, tmp;
  bool bad = false;
  if (!kReverse) {
    if (have_carry) {
      Op::load(aggs, carry, acc);
      Op::load(x, lo, e);
      bad |= !Op::combine(acc, e, tmp);
      acc = tmp;
    } else {
      Op::load(x, lo, acc);
    }
    Op::store(out, lo, acc);
    for (int64_t k = lo + 1; k < hi; ++k) {
      Op::load(x, k, e);
      bad |= !Op::combine(acc, e, tmp);
      acc = tmp;
      Op::store(out, k, acc);
    }
  } else {
    if (have_carry) {
      Op::load(aggs, carry, acc);
      Op::load(x, hi - 1, e);
      bad |= !Op::combine(e, acc, tmp);
      acc = tmp;
    } else {
      Op::load(x, hi - 1, acc);
    }
    Op::store(out, hi - 1, acc);
    for (int64_t k = hi - 2; k >= lo; --k) {
      Op::load(x, k, e);
      bad |= !Op::combine(e, acc, tmp);
      acc = tmp;
      Op::store(out, k, acc);
    }
  }
  if (bad) raise_error(err, lo, kErrSingular);
}

// Recursive reduce-then-scan with lane-serial combines (chunk length Lup at
// every level).  Returns the tally of combines and of the critical path.
template <int D, class Op, bool kReverse>
struct LaneScan {
  static void run(pode_context* ctx, typename Op::Arr in, typename Op::Arr out, int64_t n, int level, int Lup,
                  ScanTally& t) {
    DevError* err = reinterpret_cast<DevError*>(ctx->d_err);
    const unsigned th = kLaneThreads;
    if (n <= Lup) {
      k_lscan_down<D, Op, kReverse><<<1, th, 0, ctx->stream>>>(in, n, static_cast<int>(n), in, 0, out, err);
      note_launch(ctx, "lscan_down");
      t.combines += n - 1;
      t.depth += n - 1;
      return;
    }
    const int L = Lup;
    const int64_t nc = (n + L - 1) / L;
    typename Op::Arr agg = alloc(ctx, "lscan_agg_" + std::to_string(level), nc);
    const unsigned blocks = static_cast<unsigned>((nc + th - 1) / th);
    k_lscan_reduce<D, Op><<<blocks, th, 0, ctx->stream>>>(in, n, L, agg, err);
    note_launch(ctx, "lscan_reduce");
    t.combines += n - nc;
    t.depth += L - 1;
    run(ctx, agg, agg, nc, level + 1, Lup, t);
    k_lscan_down<D, Op, kReverse><<<blocks, th, 0, ctx->stream>>>(in, n, L, agg, nc, out, err);
    note_launch(ctx, "lscan_down");
    t.combines += n - 1;
    t.depth += L;
  }

  static typename Op::Arr alloc(pode_context* ctx, const std::string& tag, int64_t n) {
    if constexpr (std::is_same_v<typename Op::Arr, FEd>) {
      double* base = ctx->ws.arr<double>(tag + "_f", size_t(n) * (3 * D * D + 2 * D));
      FEd e;
      e.a = base;
      e.c = e.a + n * D * D;
      e.j = e.c + n * D * D;
      e.b = e.j + n * D * D;
      e.eta = e.b + n * D;
      return e;
    } else {
      double* base = ctx->ws.arr<double>(tag + "_m", size_t(n) * (D * D + D));
      return SEd{base, base + n * D * D, nullptr};
    }
  }
};

}  // namespace lane
}  // namespace pode
