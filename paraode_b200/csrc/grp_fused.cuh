// Group-of-D-lanes fused IEKS passes, for state dimensions the lane-serial
// passes (lane.cuh) cannot hold in registers (D = 10..16; rigid body IWP(4)
// is D = 15).  Same algebra, same driver (fast_driver.cuh), one chunk per
// GROUP of D consecutive lanes instead of one per thread: lane r owns row r
// of every D x D matrix and entry r of every D-vector, rows move through the
// group's shared-memory tile and pivot rows by shuffle (group.cuh).
//
// Restated reference operators (row form of Eigen's Householder QR of the
// transpose, proj/src/linalg.cpp:9-27): kf_predict / kf_update
// (sequential.cpp:30-67) folded into chunk aggregates = make_filtering_element
// + ⊗_f (parallel.cpp:5-100); make_smoothing_element (parallel.cpp:112-135);
// ⊗_s on (E, g) (parallel.cpp:146-156); the objective and stopping maxima
// (ieks.cpp:49-77); innovation statistics and outputs (ieks.cpp:79-109,
// 190-208).
//
// HBM layout is node-major (a group touches D contiguous doubles per row):
// eta[k D + r], E[(k D + r) D + j], g[k D + r], C_f[(k D + r) D + j] for
// local node k < nc L; node N in the separate term slot, as in lane.cuh.
#pragma once

#include "lane.cuh"

namespace pode {
namespace grp {

// Resident blocks per SM the heavy passes are compiled for (register cap
// 64K / (128 * n)); 2 = 255 registers.
#ifndef PODE_GRP_MIN_BLOCKS
#define PODE_GRP_MIN_BLOCKS 2
#endif
constexpr int kGrpMinBlocks = PODE_GRP_MIN_BLOCKS;

// Per-lane view of the block-binomial transition (prior.cpp:99-107):
// row r = blk B + a of Phi_n has entries bin(q - a, i - a) ratio[i] at
// columns blk B + i, i >= a.
template <int D, int d>
struct GM {
  using LM = lane::Model<D, d>;
  static constexpr int B = D / d;
  static constexpr int q = B - 1;
  struct Lane {
    int blk, a;
    double bin[B];
  };
  __device__ static Lane lane_of(int r) {
    Lane l;
    l.blk = r / B;
    l.a = r - l.blk * B;
#pragma unroll
    for (int i = 0; i < B; ++i) l.bin[i] = (i >= l.a) ? LM::binom(q - l.a, i - l.a) : 0.0;
    return l;
  }

  // row r of Phi X
  template <int K>
  __device__ static Rw<K> phi_rows(const Grp<D>& g, const Lane& ln, const double (&ratio)[B], const Rw<K>& x) {
    publish<D, K>(g, x);
    Rw<K> o = zeros<K>();
#pragma unroll
    for (int i = 0; i < B; ++i) {
      if (i < ln.a) continue;
      const double coef = ln.bin[i] * ratio[i];
      const Rw<K> row = ld_tile_row<K>(g.sc + (ln.blk * B + i) * K);
#pragma unroll
      for (int j = 0; j < K; ++j) o[j] = fma(coef, row[j], o[j]);
    }
    return o;
  }

  // entry i of the Jacobian row owned by this lane (i = g.r < d), column c
  __device__ static double jac_of(const typename LM::Lin& l, int i, int c) {
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < d; ++k) v = (k == i) ? l.jac[k][c] : v;
    return v;
  }

  // rows of H_bar X on lanes 0..d-1 (zeros elsewhere); H_bar row i =
  // (E_1 - F_y E_0)[i] diag(T_n) (statespace.cpp:65-88, ieks.cpp:160-164)
  template <int K>
  __device__ static Rw<K> h_rows(const Grp<D>& g, const typename LM::Lin& l, const double (&t)[B], const Rw<K>& x) {
    publish<D, K>(g, x);
    Rw<K> o = zeros<K>();
    if (g.r < d) {
      const Rw<K> x1 = ld_tile_row<K>(g.sc + (g.r * B + 1) * K);
#pragma unroll
      for (int j = 0; j < K; ++j) o[j] = (1.0 * t[1]) * x1[j];
#pragma unroll
      for (int c = 0; c < d; ++c) {
        const double coef = (-jac_of(l, g.r, c)) * t[0];
        const Rw<K> xc = ld_tile_row<K>(g.sc + (c * B) * K);
#pragma unroll
        for (int j = 0; j < K; ++j) o[j] = fma(coef, xc[j], o[j]);
      }
    }
    return o;
  }

  // Square-root update against the noiseless d-row observation
  // (sequential.cpp:41-67, R = 0): Psi = tria([[H C-], [C-]]).  On return cm
  // holds C+ (row r), k the gain row K[r] (d entries), s / sinv the factor S
  // (every lane).
  struct Upd {
    double s[d][d];
    double sinv[d];
    double k[d];
    bool singular;
  };
  __device__ static Upd update(const Grp<D>& g, const typename LM::Lin& l, const double (&t)[B], Rw<D>& cm) {
    Upd u;
    Rw<D> top = h_rows<D>(g, l, t, cm);
    Rw<D> bot = cm;
    lq<D, d, D, D>(g, top, bot);
    u.singular = singular_diag(g, pick(top, g.r < d ? g.r : D), d);
    Rw<D> srow = zeros<D>();
#pragma unroll
    for (int j = 0; j < d; ++j) srow[j] = (g.r < d) ? top[j] : 0.0;
    publish_factor<D, D>(g, srow);
#pragma unroll
    for (int i = 0; i < d; ++i) {
#pragma unroll
      for (int j = 0; j < d; ++j) u.s[i][j] = (j <= i) ? g.sc[i * D + j] : 0.0;
      u.sinv[i] = g.vs[i];
    }
    // K[r] S = Psi21[r]  (back substitution)
#pragma unroll
    for (int i = d - 1; i >= 0; --i) {
      double acc = bot[i];
#pragma unroll
      for (int k = i + 1; k < d; ++k) acc = fma(-u.k[k], u.s[k][i], acc);
      u.k[i] = acc * u.sinv[i];
    }
    // C+ = Psi22 (shifted by d columns)
#pragma unroll
    for (int j = 0; j < D; ++j) cm[j] = (j < D - d && j <= g.r) ? bot[d + (j < D - d ? j : 0)] : 0.0;
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

  // H_bar v - offset for a full vector v (every lane, static indices)
  __device__ static void innov(const typename LM::Lin& l, const double (&t)[B], const double (&v)[D], double (&z)[d]) {
    LM::h_vec(l, t, v, z);
#pragma unroll
    for (int i = 0; i < d; ++i) z[i] -= l.off[i];
  }
};

// Entry i of a small register array with a runtime (lane-dependent) index,
// without dynamic register indexing.
template <int B>
__device__ __forceinline__ double entry(const double (&t)[B], int i) {
  double v = 0.0;
#pragma unroll
  for (int k = 0; k < B; ++k) v = (k == i) ? t[k] : v;
  return v;
}

template <int K>
__device__ __forceinline__ Rw<K> sel(bool take, const Rw<K>& a, const Rw<K>& b) {
  Rw<K> o;
#pragma unroll
  for (int j = 0; j < K; ++j) o[j] = take ? a[j] : b[j];
  return o;
}

// The full D-vector on every lane of the group from entry r on lane r.
template <int D>
__device__ __forceinline__ void gather_full(const Grp<D>& g, double x, double (&v)[D]) {
  const Rw<D> f = gather_vec(g, x);
#pragma unroll
  for (int j = 0; j < D; ++j) v[j] = f[j];
}

// Node-major layout helpers (local node k = c L + t).
__device__ __forceinline__ int64_t node_of(const FastArgs& a, int64_t c, int64_t t) { return c * a.L + t; }

template <int D, int d>
__device__ __forceinline__ void load_y(const FastArgs& a, const LinPoint& lp, int64_t k, double (&y)[d]) {
  constexpr int B = D / d;
#pragma unroll
  for (int j = 0; j < d; ++j) y[j] = (k == a.N) ? lp.term[j * B] : lp.eta[k * D + j * B];
}

// ------------------------------------------------------------- pass A ---
template <int D, int d>
__global__ void __launch_bounds__(kThreads, kGrpMinBlocks) k_grp_fwd_reduce(const FastArgs a, FastConst<D> cst, FEd agg) {
  using M = GM<D, d>;
  using LM = typename M::LM;
  constexpr int B = M::B;
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t c = group_index<D>(g);
  const bool okc = g.real() && c < a.nchunks;
  const int64_t cc = okc ? c : 0;  // idle groups shadow chunk 0 (warp-uniform group ops), store nothing
  const typename M::Lane ln = M::lane_of(g.r);
  const LinPoint lp = lin_point(a);
  const int64_t s = cc * a.L;
  const int64_t e = min(a.N, s + a.L);
  const int r = g.r;
  const bool first = cc == 0 && a.first;
  Rw<D> A, C, J;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    A[j] = (!first && r == j) ? 1.0 : 0.0;
    C[j] = 0.0;
    J[j] = 0.0;
  }
  double b = first ? cst.m0[r < D ? r : 0] : 0.0, eta = 0.0;
  Rw<D> q;
#pragma unroll
  for (int j = 0; j < D; ++j) q[j] = cst.q[(r < D ? r : 0) * D + j];
  double tk[B], tki[B];
  LM::taus(a.grid, a.first, s, tk, tki);
  double gcur = a.grid[s], gnext = a.grid[s + 1], hlast = 0.0;
  bool bad_sing = false;
  int64_t bad_lin = -1;
  // every group of a warp runs L steps (group ops synchronise the warp); a
  // step past the chunk's end recomputes its last step and is discarded
  for (int t = 0; t < a.L; ++t) {
    const bool act = s + t < e;
    const int64_t k = act ? s + t : e - 1;
    double tn[B], tni[B], ratio[B], pc[B][B];
    // h_{k+1} from node times loaded a step ahead (a step past the chunk's
    // end repeats the last step's h)
    const double h = act ? gnext - gcur : hlast;
    hlast = h;
    if (act) {
      gcur = gnext;
      if (k + 2 <= a.N) gnext = a.grid[k + 2];
    }
    LM::taus_h(h, tn, tni);
#pragma unroll
    for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tni[i];
    LM::phi_coefs(ratio, pc);
    // predict
    Rw<D> An = M::template phi_rows<D>(g, ln, ratio, A);
    double bf[D];
    gather_full<D>(g, b, bf);
    LM::phi_vec(pc, bf);
    Rw<D> cm = sqrt_sum_lt(g, M::template phi_rows<D>(g, ln, ratio, C), q);  // C- = tria([phi C, Q])
    // update at node k+1
    double y[d];
    load_y<D, d>(a, lp, k + 1, y);
    const typename LM::Lin lin = LM::linearize(a.prob, y, a.ek0, gcur);  // t_{k+1} (only PODE_POLE reads it)
    if (act && !lin.finite && bad_lin < 0) bad_lin = k + 1;
    const typename M::Upd u = M::update(g, lin, tn, cm);
    bad_sing |= act && u.singular;
    double uu[d];
    M::innov(lin, tn, bf, uu);
    const Rw<D> U = M::template h_rows<D>(g, lin, tn, An);  // rows of H_bar A- on lanes < d
    // A+ = A- - K U, b+ = b- - K u
    publish<D, D>(g, U);
    double col[d];
    double bn = entry<D>(bf, r);
#pragma unroll
    for (int i = 0; i < d; ++i) {
      const Rw<D> Ui = ld_tile_row<D>(g.sc + i * D);
#pragma unroll
      for (int j = 0; j < D; ++j) An[j] = fma(-u.k[i], Ui[j], An[j]);
      bn = fma(-u.k[i], uu[i], bn);
      col[i] = g.sc[i * D + r];  // column r of U
    }
    // Ubar = S^-1 U (column r -> X[r]), ubar = S^-1 u; eta -= Ubar^T ubar
    double ub[d], X[d];
    M::s_solve(u, uu, ub);
    M::s_solve(u, col, X);
    double de = 0.0;
#pragma unroll
    for (int i = 0; i < d; ++i) de = fma(X[i], ub[i], de);
    // J = tria([X, J]) (J only enters through J J^T; the right block J is
    // lower triangular: structured sweep)
    Rw<D + d> xj;
#pragma unroll
    for (int i = 0; i < d; ++i) xj[i] = X[i];
#pragma unroll
    for (int j = 0; j < D; ++j) xj[d + j] = J[j];
    const Rw<D> Jn = tria<D, D + d, d>(g, xj);
    A = sel(act, An, A);
    C = sel(act, cm, C);
    J = sel(act, Jn, J);
    b = act ? bn : b;
    eta = act ? eta - de : eta;
#pragma unroll
    for (int i = 0; i < B; ++i) {
      tk[i] = act ? tn[i] : tk[i];
      tki[i] = act ? tni[i] : tki[i];
    }
  }
  if (!okc) return;
  if (r == 0 && bad_lin >= 0) raise_error(a.err, bad_lin, kErrLinearization);
  if (r == 0 && bad_sing) raise_error(a.err, s, kErrSingular);
  st_row<D>(agg.a, c, r, true, A);
  st_row<D>(agg.c, c, r, true, C);
  st_row<D>(agg.j, c, r, true, J);
  agg.b[c * D + r] = b;
  agg.eta[c * D + r] = eta;
}

// ------------------------------------------------------------- pass C ---
// kFinal: also stores C_f(k) (cf, node-major) and reduces the whitened
// innovations into one partial per block (part[3 b]).
template <int D, int d, bool kFinal>
__global__ void __launch_bounds__(kThreads, kGrpMinBlocks) k_grp_fwd_down(const FastArgs a, FastConst<D> cst, FEd prefix,
                                                           lane::ElemSoA elems, double* cf, double* cterm,
                                                           double* part, SEd bagg) {
  using M = GM<D, d>;
  using LM = typename M::LM;
  constexpr int B = M::B;
  extern __shared__ double smem[];
  __shared__ double red[kThreads];
  const Grp<D> g = make_group<D>(smem);
  const int64_t c = group_index<D>(g);
  const bool okc = g.real() && c < a.nchunks;
  const int64_t cc = okc ? c : 0;
  const typename M::Lane ln = M::lane_of(g.r);
  const LinPoint lp = lin_point(a);
  const int64_t s = cc * a.L;
  const int64_t e = min(a.N, s + a.L);
  const int r = g.r;
  const int rr = r < D ? r : 0;
  double innov = 0.0;
  double m;
  Rw<D> C;
  if (cc == 0 && a.first) {
    m = cst.m0[rr];
    C = zeros<D>();
  } else if (cc == 0) {
    m = a.carry[rr];
    C = ld_row<D>(a.carry + D, 0, rr, true);
  } else {
    m = prefix.b[(cc - 1) * D + rr];
    C = ld_row<D>(prefix.c, cc - 1, rr, true);
  }
  Rw<D> q;
#pragma unroll
  for (int j = 0; j < D; ++j) q[j] = cst.q[rr * D + j];
  double tk[B], tki[B];
  LM::taus(a.grid, a.first, s, tk, tki);
  double gcur = a.grid[s], gnext = a.grid[s + 1], hlast = 0.0;
  bool bad_sing = false;
  int64_t bad_lin = -1;
  Rw<D> EA = zeros<D>();
  double gA = 0.0;
  for (int t = 0; t < a.L; ++t) {
    const bool act = s + t < e;
    const bool st_ok = act && okc;
    const int64_t k = act ? s + t : e - 1;
    double tn[B], tni[B], ratio[B], pc[B][B];
    // h_{k+1} from node times loaded a step ahead (a step past the chunk's
    // end repeats the last step's h)
    const double h = act ? gnext - gcur : hlast;
    hlast = h;
    if (act) {
      gcur = gnext;
      if (k + 2 <= a.N) gnext = a.grid[k + 2];
    }
    LM::taus_h(h, tn, tni);
#pragma unroll
    for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tni[i];
    LM::phi_coefs(ratio, pc);
    if constexpr (kFinal) {
      if (st_ok) st_row<D>(cf, k, rr, true, C);
    }
    // Y = C (phi C)^T; C- = tria([phi C, Q]); E = Y C-^-T C-^-1
    const Rw<D> pcC = M::template phi_rows<D>(g, ln, ratio, C);
    const Rw<D> Y = mm_nt(g, C, pcC);
    Rw<D> cm = sqrt_sum_lt(g, pcC, q);
    const bool sing_pred = singular_diag(g, pick(cm, rr), D);  // every lane (group sync inside)
    bad_sing |= act && sing_pred;
    publish_factor<D, D>(g, cm);
    const Rw<D> z = solve_xlt<D, D>(g, Y);
    const Rw<D> E = solve_xl<D, D>(g, z);
    double mv[D];
    gather_full<D>(g, m, mv);
    LM::phi_vec(pc, mv);
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) acc = fma(E[j], mv[j], acc);
    const double gk = m - acc;
    if (st_ok) {
      st_row<D>(elems.e, k, rr, true, E);
      elems.g[k * D + rr] = gk;
    }
    if constexpr (!kFinal) {
      // the chunk's backward aggregate (E, g) <- (E E_k, E g_k + g) in time
      // order (⊗_s on means, parallel.cpp:146-156), in registers
      double gf[D];
      gather_full<D>(g, gk, gf);
      double og = gA;
#pragma unroll
      for (int x = 0; x < D; ++x) og = fma(EA[x], gf[x], og);
      const Rw<D> ee = mm(g, EA, E);
      EA = (t == 0) ? E : sel(act, ee, EA);
      gA = (t == 0) ? gk : (act ? og : gA);
    }
    // measurement update at node k+1
    double y[d];
    load_y<D, d>(a, lp, k + 1, y);
    const typename LM::Lin lin = LM::linearize(a.prob, y, a.ek0, gcur);  // t_{k+1} (only PODE_POLE reads it)
    if (act && !lin.finite && bad_lin < 0) bad_lin = k + 1;
    const typename M::Upd u = M::update(g, lin, tn, cm);
    bad_sing |= act && u.singular;
    double zz[d];
    M::innov(lin, tn, mv, zz);
    if constexpr (kFinal) {
      double w[d];
      M::s_solve(u, zz, w);
      if (act && r == 0)
#pragma unroll
        for (int i = 0; i < d; ++i) innov = fma(w[i], w[i], innov);
    }
    double mr = entry<D>(mv, r);
#pragma unroll
    for (int i = 0; i < d; ++i) mr = fma(-u.k[i], zz[i], mr);
    m = act ? mr : m;
    C = sel(act, cm, C);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      tk[i] = act ? tn[i] : tk[i];
      tki[i] = act ? tni[i] : tki[i];
    }
  }
  if (okc && e == a.N) {  // terminal node N: E = 0, g = m_f(N) (parallel.cpp:137-144)
    elems.term[rr] = m;
    if constexpr (kFinal) st_row<D>(cterm, 0, rr, true, C);
  }
  if constexpr (!kFinal) {  // the last shard's last chunk absorbs the terminal element
    const bool term = e == a.N && a.last;
    double mf[D];
    gather_full<D>(g, m, mf);
    double og = gA;
    if (term) {
#pragma unroll
      for (int x = 0; x < D; ++x) og = fma(EA[x], mf[x], og);
    }
    if (okc) {
#pragma unroll
      for (int j = 0; j < D; ++j) bagg.e[(c * D + r) * D + j] = term ? 0.0 : EA[j];
      bagg.g[c * D + r] = og;
    }
  }
  if (okc && r == 0 && bad_lin >= 0) raise_error(a.err, bad_lin, kErrLinearization);
  if (okc && r == 0 && bad_sing) raise_error(a.err, s, kErrSingular);
  if constexpr (kFinal) lane::block_sum_partial(red, okc ? innov : 0.0, part);
}

// ------------------------------------------------------------- pass E ---
template <int D, int d, bool kInitial>
__global__ void __launch_bounds__(kThreads) k_grp_bwd_down(FastArgs a, FastConst<D> cst, lane::ElemSoA elems,
                                                           SEd suffix, const double* eta_old, const double* old_term,
                                                           double* eta_new, double* new_term, double* part) {
  using M = GM<D, d>;
  using LM = typename M::LM;
  constexpr int B = M::B;
  extern __shared__ double smem[];
  __shared__ double red[3][kThreads];
  const Grp<D> g = make_group<D>(smem);
  const int64_t c = group_index<D>(g);
  const bool okc = g.real() && c < a.nchunks;
  const int64_t cc = okc ? c : 0;
  const int r = g.r;
  const int rr = r < D ? r : 0;
  if (a.it_dev != nullptr) {  // graph-loop mode: buffers by iteration parity
    const int par = *a.it_dev & 1;
    eta_old = par ? a.pair1 : a.pair0;
    old_term = eta_old + a.term_off;
    eta_new = par ? a.pair0 : a.pair1;
    new_term = eta_new + a.term_off;
  }
  double obj = 0.0, dmax = 0.0, emax = 0.0;
  const int64_t s = cc * a.L;
  const int64_t e = min(a.N, s + a.L);
  const bool last = cc == a.nchunks - 1;
  double te[B], tei[B];
  LM::taus(a.grid, a.first, e, te, tei);
  const double tr_e = entry<B>(te, rr % B);
  const double tri_e = entry<B>(tei, rr % B);
  const double old_e = (e == a.N) ? old_term[rr] : eta_old[e * D + rr];
  double mu, eta_e;
  if (kInitial) {
    eta_e = old_e;
    mu = 0.0;
  } else {
    mu = last ? elems.term[rr] : suffix.g[(cc + 1) * D + rr];
    eta_e = tr_e * mu;
  }
  if (okc && last) {
    if (!kInitial) new_term[rr] = eta_e;  // shards: the halo node, owned by the next shard
    if (a.last) {
      dmax = fmax(dmax, fabs(eta_e - old_e));
      emax = fmax(emax, fabs(eta_e));
    }
  }
  double bar_next[D];
  gather_full<D>(g, tri_e * eta_e, bar_next);
  double tn[B];
#pragma unroll
  for (int i = 0; i < B; ++i) tn[i] = tei[i];  // T_{k+1}^-1
  for (int t = a.L - 1; t >= 0; --t) {
    const bool act = s + t < e;
    const int64_t k = act ? s + t : s;
    double tk[B], tki[B];
    LM::taus(a.grid, a.first, k, tk, tki);
    const double oldk = eta_old[k * D + rr];
    double etak, mun = mu;
    if (kInitial) {
      etak = oldk;
    } else {
      double muf[D];
      gather_full<D>(g, mu, muf);
      const Rw<D> E = ld_row<D>(elems.e, k, rr, true);
      double acc = elems.g[k * D + rr];
#pragma unroll
      for (int j = 0; j < D; ++j) acc = fma(E[j], muf[j], acc);
      mun = acc;
      etak = entry<B>(tk, rr % B) * acc;
      if (act && okc) eta_new[k * D + rr] = etak;
    }
    if (act && okc) {
      dmax = fmax(dmax, fabs(etak - oldk));
      emax = fmax(emax, fabs(etak));
    }
    double bar[D];
    gather_full<D>(g, entry<B>(tki, rr % B) * etak, bar);
    // objective term || Qunit^-1/2 (bar_{k+1} - phi_k bar_k) ||^2 (lane 0)
    double ratio[B], pc[B][B], pb[D];
#pragma unroll
    for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tn[i];
    LM::phi_coefs(ratio, pc);
#pragma unroll
    for (int j = 0; j < D; ++j) pb[j] = bar[j];
    LM::phi_vec(pc, pb);
    double w[D], acc2 = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double acc = bar_next[i] - pb[i];
#pragma unroll
      for (int k2 = 0; k2 < i; ++k2) acc = fma(-cst.qunit[i * D + k2], w[k2], acc);
      w[i] = acc * cst.qunit_rdiag[i];
      acc2 = fma(w[i], w[i], acc2);
    }
    if (act && okc && r == 0) obj += acc2;
    if (act) {
      mu = mun;
#pragma unroll
      for (int j = 0; j < D; ++j) bar_next[j] = bar[j];
#pragma unroll
      for (int i = 0; i < B; ++i) tn[i] = tki[i];
    }
  }
  red[0][threadIdx.x] = obj;
  red[1][threadIdx.x] = dmax;
  red[2][threadIdx.x] = emax;
  __syncthreads();
  for (int st = kThreads / 2; st > 0; st >>= 1) {
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

// ------------------------------------------------- finalize (once) ---
// L_k = tria([(I - E_k phi_k) C_f(k), E_k Q^1/2]) (Joseph form of the
// lower-right block of make_smoothing_element, parallel.cpp:112-135).
template <int D, int d>
__device__ __forceinline__ Rw<D> smooth_factor(const Grp<D>& g, const typename GM<D, d>::Lane& ln,
                                               const double (&ratio)[D / d], const Rw<D>& E, const Rw<D>& cf,
                                               const Rw<D>& q) {
  const Rw<D> pcf = GM<D, d>::template phi_rows<D>(g, ln, ratio, cf);
  const Rw<D> epc = mm(g, E, pcf);
  const Rw<D> eq = mm(g, E, q);
  Rw<D> left;
#pragma unroll
  for (int j = 0; j < D; ++j) left[j] = cf[j] - epc[j];
  return sqrt_sum(g, left, eq);
}

template <int D, int d>
__global__ void __launch_bounds__(kThreads) k_grp_fin_fold(FastArgs a, FastConst<D> cst, lane::ElemSoA elems,
                                                           const double* cf, const double* cterm, SEd agg) {
  using M = GM<D, d>;
  using LM = typename M::LM;
  constexpr int B = M::B;
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t c = group_index<D>(g);
  const bool okc = g.real() && c < a.nchunks;
  const int64_t cc = okc ? c : 0;
  const typename M::Lane ln = M::lane_of(g.r);
  const int r = g.r;
  const int rr = r < D ? r : 0;
  const int64_t s = cc * a.L;
  const int64_t e = min(a.N, s + a.L);
  const bool last = cc == a.nchunks - 1 && a.last;
  Rw<D> ea, la;
  double ga = last ? elems.term[rr] : 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    ea[j] = (!last && r == j) ? 1.0 : 0.0;
    la[j] = last ? cterm[rr * D + j] : 0.0;
  }
  Rw<D> q;
#pragma unroll
  for (int j = 0; j < D; ++j) q[j] = cst.q[rr * D + j];
  double tn[B], tni[B];
  LM::taus(a.grid, a.first, e, tn, tni);
  for (int t = a.L - 1; t >= 0; --t) {
    const bool act = s + t < e;
    const int64_t k = act ? s + t : s;
    double tk[B], tki[B], ratio[B];
    LM::taus(a.grid, a.first, k, tk, tki);
#pragma unroll
    for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tni[i];
    const Rw<D> E = ld_row<D>(elems.e, k, rr, true);
    const double gk = elems.g[k * D + rr];
    const Rw<D> cfk = ld_row<D>(cf, k, rr, true);
    const Rw<D> lk = smooth_factor<D, d>(g, ln, ratio, E, cfk, q);
    const Rw<D> ln2 = sqrt_sum_lt(g, mm(g, E, la), lk);  // tria([E l, lk]) (⊗_s, parallel.cpp:146-156)
    const double gn = matvec(g, E, ga) + gk;
    const Rw<D> en = mm(g, E, ea);
    la = sel(act, ln2, la);
    ga = act ? gn : ga;
    ea = sel(act, en, ea);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      tn[i] = act ? tk[i] : tn[i];
      tni[i] = act ? tki[i] : tni[i];
    }
  }
  if (!okc) return;
  st_row<D>(agg.e, c, r, true, ea);
  st_row<D>(agg.l, c, r, true, la);
  agg.g[c * D + r] = ga;
}

// Calibrated outputs of node n (ieks.cpp:196-208), row r on lane r.
template <int D, int d>
__device__ __forceinline__ void write_node(const Grp<D>& g, bool ok, const lane::FinOut& o, int64_t n,
                                           const double (&t)[D / d], const Rw<D>& ls, double eta, double sig) {
  constexpr int B = D / d;
  const int r = g.r;
  const double tr = entry<B>(t, r < D ? r % B : 0);
  if (ok && o.means) o.means[n * D + r] = eta;
  if (ok && o.cov) {
#pragma unroll
    for (int j = 0; j < D; ++j) o.cov[(n * D + r) * D + j] = tr * ls[j] * sig;
  }
  if (ok && o.sol_m && r % B == 0) o.sol_m[n * d + r / B] = eta;
  if (o.sol_c) {
    publish<D, D>(g, ls);
    if (ok && r < d * d) {
      const int i = r / d, j = r - (r / d) * d;
      const Rw<D> li = ld_tile_row<D>(g.sc + (i * B) * D);
      const Rw<D> lj = ld_tile_row<D>(g.sc + (j * B) * D);
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) acc += (t[0] * li[k] * sig) * (t[0] * lj[k] * sig);
      o.sol_c[(n * d + i) * d + j] = acc;
    }
  }
}

template <int D, int d>
__global__ void __launch_bounds__(kThreads) k_grp_fin_bwd(FastArgs a, FastConst<D> cst, lane::ElemSoA elems,
                                                          const double* cf, const double* cterm, SEd suffix,
                                                          const double* eta_out, const double* eta_out_term,
                                                          const double* innov, double count, lane::FinOut o) {
  using M = GM<D, d>;
  using LM = typename M::LM;
  constexpr int B = M::B;
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t c = group_index<D>(g);
  const bool okc = g.real() && c < a.nchunks;
  const int64_t cc = okc ? c : 0;
  const typename M::Lane ln = M::lane_of(g.r);
  const int rr = g.r < D ? g.r : 0;
  const int64_t s = cc * a.L;
  const int64_t e = min(a.N, s + a.L);
  const bool last = cc == a.nchunks - 1;
  const double sig = sqrt(innov[0] / count);
  Rw<D> ls = ld_row<D>(last ? cterm : suffix.l, last ? 0 : cc + 1, rr, true);
  Rw<D> q;
#pragma unroll
  for (int j = 0; j < D; ++j) q[j] = cst.q[rr * D + j];
  double tn[B], tni[B];
  LM::taus(a.grid, a.first, e, tn, tni);
  // node N (the last chunk of the last shard); every group calls write_node
  // (it synchronises the warp), only that one writes
  write_node<D, d>(g, okc && last && a.last, o, e, tn, ls, eta_out_term[rr], sig);
  for (int t = a.L - 1; t >= 0; --t) {
    const bool act = s + t < e;
    const int64_t k = act ? s + t : s;
    double tk[B], tki[B], ratio[B];
    LM::taus(a.grid, a.first, k, tk, tki);
#pragma unroll
    for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tni[i];
    const Rw<D> E = ld_row<D>(elems.e, k, rr, true);
    const Rw<D> cfk = ld_row<D>(cf, k, rr, true);
    const Rw<D> lk = smooth_factor<D, d>(g, ln, ratio, E, cfk, q);
    const Rw<D> lsn = sqrt_sum_lt(g, mm(g, E, ls), lk);
    ls = sel(act, lsn, ls);
    write_node<D, d>(g, okc && act, o, k, tk, ls, eta_out[k * D + rr], sig);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      tn[i] = act ? tk[i] : tn[i];
      tni[i] = act ? tki[i] : tni[i];
    }
  }
}

// eta (node-major + node-N slot) <- mu0 at every node.
template <int D>
__global__ void k_eta_fill_rows(const double* mu0, int64_t nodes, double* base) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < (nodes + 1) * D) base[i] = mu0[i % D];
}

}  // namespace grp
}  // namespace pode
