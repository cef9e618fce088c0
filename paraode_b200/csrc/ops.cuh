// Scan elements and their associative operators on a group of D lanes.
//
// Restates, in the row-per-lane layout of group.cuh:
//   kf_predict / kf_update            proj/src/sequential.cpp:30-67
//   make_filtering_element            proj/src/parallel.cpp:5-65
//   combine_filtering (⊗_f)           proj/src/parallel.cpp:67-100
//   make_smoothing_element / terminal proj/src/parallel.cpp:112-144
//   combine_smoothing (⊗_s)           proj/src/parallel.cpp:146-156
// Observations carry up to M rows; a step with m < M rows is padded with
// unit-noise dummy rows (H = 0, offset = 0, R = e_r), which leave the
// posterior unchanged exactly and keep every pivot well defined, so groups of
// one warp never diverge on m.
#pragma once

#include "group.cuh"

namespace pode {

// Error codes of the device error word (mapped to the reference's exception
// types by the C ABI; proj/include/paraode/errors.hpp).
enum DevErr : int { kErrNone = 0, kErrInvalid = 1, kErrSingular = 3, kErrLinearization = 4 };

// First failing index wins: key = (index << 8) | code, atomicMin.
struct DevError {
  unsigned long long key;
};

__device__ __forceinline__ void raise_error(DevError* err, long long index, int code) {
  if (err == nullptr) return;
  const unsigned long long key =
      (static_cast<unsigned long long>(index < 0 ? 0 : index) << 8) | static_cast<unsigned>(code);
  atomicMin(&err->key, key);
}

template <int D>
struct FEl {  // FilteringElement (parallel.hpp:20-26): row r / entry r
  Rw<D> a;
  double b;
  Rw<D> c;
  double eta;
  Rw<D> j;
};

template <int D>
struct SEl {  // SmoothingElement (parallel.hpp:32-36)
  Rw<D> e;
  double g;
  Rw<D> l;
};

template <int D>
struct Gauss {  // GaussianSqrt (statespace.hpp:13-16)
  double m;
  Rw<D> c;
};

// One observation, up to M rows, on lanes 0..M-1 (zero on lanes >= M).
template <int D, int M>
struct Obs {
  Rw<D> h;
  double off;
  Rw<M> r;  // row of R^1/2 (M columns)
  int m;    // real rows
};

template <int D>
__device__ __forceinline__ FEl<D> filtering_identity(const Grp<D>& g) {
  FEl<D> e;
#pragma unroll
  for (int k = 0; k < D; ++k) e.a[k] = (k == g.r) ? 1.0 : 0.0;
  e.b = 0.0;
  e.c = zeros<D>();
  e.eta = 0.0;
  e.j = zeros<D>();
  return e;
}

// --------------------------------------------------------------- Kalman ---
// kf_predict: m' = phi m, P'^1/2 = tria([phi P^1/2, Q^1/2])  (sequential.cpp:30-39)
template <int D>
__device__ __forceinline__ Gauss<D> kf_predict(const Grp<D>& g, const Gauss<D>& s, const Rw<D>& phi,
                                               const Rw<D>& q) {
  Gauss<D> p;
  p.m = matvec(g, phi, s.m);
  p.c = sqrt_sum(g, mm(g, phi, s.c), q);
  return p;
}

// kf_update (sequential.cpp:41-67): Psi = tria([[H P^1/2, R^1/2], [P^1/2, 0]]).
// Returns false (and leaves pred) if S^1/2 is singular.
template <int D, int M>
__device__ __forceinline__ bool kf_update(const Grp<D>& g, Gauss<D>& st, const Obs<D, M>& o) {
  constexpr int K = D + M;
  Rw<K> top, bot;
  const Rw<D> hp = mm(g, o.h, st.c);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    top[j] = hp[j];
    bot[j] = st.c[j];
  }
#pragma unroll
  for (int j = 0; j < M; ++j) {
    top[D + j] = (g.r < M) ? o.r[j] : 0.0;
    bot[D + j] = 0.0;
  }
  lq<D, M, D, K>(g, top, bot);
  const bool sing = singular_diag(g, pick(top, g.r < M ? g.r : K), o.m);
  // K = Psi21 S^-1 (x S = Psi21 row)
  Rw<D> srow = zeros<D>();
#pragma unroll
  for (int j = 0; j < M; ++j) srow[j] = (g.r < M) ? top[j] : 0.0;
  publish_factor<D, D>(g, srow);
  Rw<M> p21;
#pragma unroll
  for (int j = 0; j < M; ++j) p21[j] = bot[j];
  const Rw<M> kg = solve_xl<D, M>(g, p21);
  Rw<D> kpad = zeros<D>();
#pragma unroll
  for (int j = 0; j < M; ++j) kpad[j] = kg[j];
  const double z = matvec(g, o.h, st.m) - o.off;  // zero on padded rows
  st.m = st.m - matvec(g, kpad, z);
#pragma unroll
  for (int j = 0; j < D; ++j) st.c[j] = bot[M + j];
  return !sing;
}

// ------------------------------------------------------ filtering element ---
// make_filtering_element, interior step (parallel.cpp:38-64).
template <int D, int M>
__device__ __forceinline__ bool filtering_element(const Grp<D>& g, const Rw<D>& phi, const Rw<D>& q,
                                                  const Obs<D, M>& o, FEl<D>& el) {
  constexpr int K = D + M;
  Rw<K> top, bot;
  const Rw<D> hq = mm(g, o.h, q);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    top[j] = hq[j];
    bot[j] = q[j];
  }
#pragma unroll
  for (int j = 0; j < M; ++j) {
    top[D + j] = (g.r < M) ? o.r[j] : 0.0;
    bot[D + j] = 0.0;
  }
  lq<D, M, D, K>(g, top, bot);
  const bool sing = singular_diag(g, pick(top, g.r < M ? g.r : K), o.m);
  // H phi, and column r of it for the J factor.
  const Rw<D> hphi = mm(g, o.h, phi);
  publish<D, D>(g, hphi);
  Rw<M> hcol;
#pragma unroll
  for (int k = 0; k < M; ++k) hcol[k] = g.sc[k * D + g.r];
  // Publish S^1/2 (M x M lower, padded) as the factor.
  Rw<D> srow = zeros<D>();
#pragma unroll
  for (int j = 0; j < M; ++j) srow[j] = (g.r < M) ? top[j] : 0.0;
  publish_factor<D, D>(g, srow);
  Rw<M> p21;
#pragma unroll
  for (int j = 0; j < M; ++j) p21[j] = bot[j];
  const Rw<M> kg = solve_xl<D, M>(g, p21);  // K row r
  // J^1/2 row r = (S^-1/2 (H phi))[:, r]  (forward substitution, lane-local)
  Rw<M> jr;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    double acc = hcol[i];
#pragma unroll
    for (int k = 0; k < i; ++k) acc = fma(-g.sc[i * D + k], jr[k], acc);
    jr[i] = acc * g.vs[i];
  }
  // w = S^-1/2 offset (redundant on every lane)
  wsync();
  g.vs[2 * D + g.r] = o.off;
  wsync();
  Rw<M> w;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    double acc = g.vs[2 * D + i];
#pragma unroll
    for (int k = 0; k < i; ++k) acc = fma(-g.sc[i * D + k], w[k], acc);
    w[i] = acc * g.vs[i];
  }
  Rw<D> kpad = zeros<D>();
#pragma unroll
  for (int j = 0; j < M; ++j) kpad[j] = kg[j];
  // A = phi - K (H phi); b = K offset
  const Rw<D> khp = mm(g, kpad, hphi);
#pragma unroll
  for (int j = 0; j < D; ++j) el.a[j] = phi[j] - khp[j];
  el.b = matvec(g, kpad, o.off);
#pragma unroll
  for (int j = 0; j < D; ++j) el.c[j] = bot[M + j];
  el.j = zeros<D>();
  double eta = 0.0;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    el.j[k] = jr[k];
    eta = fma(jr[k], w[k], eta);
  }
  el.eta = eta;
  return !sing;
}

// First element: absorbs the initial distribution (parallel.cpp:13-24).
template <int D, int M>
__device__ __forceinline__ bool first_filtering_element(const Grp<D>& g, const Gauss<D>& init,
                                                        const Rw<D>& phi, const Rw<D>& q,
                                                        const Obs<D, M>& o, FEl<D>& el) {
  Gauss<D> s = kf_predict(g, init, phi, q);
  const bool ok = kf_update<D, M>(g, s, o);
  el.a = zeros<D>();
  el.b = s.m;
  el.c = s.c;
  el.eta = 0.0;
  el.j = zeros<D>();
  return ok;
}

// ⊗_f (parallel.cpp:67-100).
template <int D, bool kTri = false>
__device__ __forceinline__ bool combine_filtering(const Grp<D>& g, const FEl<D>& li, const FEl<D>& rj,
                                                  FEl<D>& out) {
  constexpr int K = 2 * D;
  Rw<K> top, bot;
  const Rw<D> x = mm_tn(g, li.c, rj.j);  // C_i^T J_j
#pragma unroll
  for (int j = 0; j < D; ++j) {
    top[j] = x[j];
    top[D + j] = (j == g.r) ? 1.0 : 0.0;
    bot[j] = rj.j[j];
    bot[D + j] = 0.0;
  }
  // Only the first D pivots are needed: they give Xi11 and Xi21, and the
  // remaining bottom block R satisfies R R^T = Xi22 Xi22^T (any factor of
  // Xi22 serves, since it only enters J through another tria).
  lq<D, D, 0, K, D>(g, top, bot);  // right block [I; 0]: lower triangular
  const bool sing = singular_diag(g, pick(top, g.r), D);
  Rw<D> xi11, xi21, xi22;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    xi11[j] = top[j];
    xi21[j] = bot[j];
    xi22[j] = bot[D + j];
  }
  publish_factor<D, D>(g, xi11);
  const Rw<D> w = solve_xlt<D, D>(g, li.c);  // W = C_i Xi11^-T
  Rw<D> gm = mm_nt(g, w, xi21);               // W Xi21^T
#pragma unroll
  for (int j = 0; j < D; ++j) gm[j] = ((j == g.r) ? 1.0 : 0.0) - gm[j];
  const Rw<D> ag = mm(g, rj.a, gm);  // A_j G
  out.a = mm(g, ag, li.a);           // A_j G A_i
  // b = A_j G (b_i + C_i (C_i^T eta_j)) + b_j
  const double t1 = matvec_t(g, li.c, rj.eta);
  const double t2 = matvec(g, li.c, t1);
  out.b = matvec(g, ag, li.b + t2) + rj.b;
  // eta = A_i^T G^T (eta_j - J_j (J_j^T b_i)) + eta_i = (G A_i)^T (...) + eta_i
  const double u1 = matvec_t(g, rj.j, li.b);
  const double u2 = matvec(g, rj.j, u1);
  const Rw<D> ga = mm(g, gm, li.a);
  out.eta = matvec_t(g, ga, rj.eta - u2) + li.eta;
  // C = tria([A_j W, C_j]) and J = tria([A_i^T Xi22, J_i]) in one sweep.
  const Rw<D> aw = mm(g, rj.a, w);
  const Rw<D> ax = mm_tn(g, li.a, xi22);
  Rw<2 * D> sc_c, sc_j;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    sc_c[j] = aw[j];
    sc_c[D + j] = rj.c[j];
    sc_j[j] = ax[j];
    sc_j[D + j] = li.j[j];
  }
  // right blocks C_j, J_i: lower triangular only when the elements come from
  // this library's own trias (kTri); reference-format elements carry a
  // general J (parallel.hpp:20-26)
  lq_pair<D, 2 * D, kTri ? D : 2 * D>(g, sc_c, sc_j);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    out.c[j] = sc_c[j];
    out.j[j] = sc_j[j];
  }
  return !sing;
}

// Gaussian-carry ⊗_f: (0, b_i, C_i, 0, 0) ⊗ rj -> (0, b, C, 0, 0).  Every
// prefix of a sequence whose first element absorbed the initial
// distribution has this form (parallel.cpp:13-24, 92-98), so the down-sweep
// of the IEKS aggregate scan only needs b and C: A, eta and J (and the
// J-side triangularisation) are skipped.
template <int D>
__device__ __forceinline__ bool combine_gauss(const Grp<D>& g, double bi, const Rw<D>& ci, const FEl<D>& rj,
                                              double& bo, Rw<D>& co) {
  constexpr int K = 2 * D;
  Rw<K> top, bot;
  const Rw<D> x = mm_tn(g, ci, rj.j);  // C_i^T J_j
#pragma unroll
  for (int j = 0; j < D; ++j) {
    top[j] = x[j];
    top[D + j] = (j == g.r) ? 1.0 : 0.0;
    bot[j] = rj.j[j];
    bot[D + j] = 0.0;
  }
  lq<D, D, 0, K, D>(g, top, bot);  // right block [I; 0]: lower triangular
  const bool sing = singular_diag(g, pick(top, g.r), D);
  Rw<D> xi11, xi21;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    xi11[j] = top[j];
    xi21[j] = bot[j];
  }
  publish_factor<D, D>(g, xi11);
  const Rw<D> w = solve_xlt<D, D>(g, ci);  // W = C_i Xi11^-T
  Rw<D> gm = mm_nt(g, w, xi21);
#pragma unroll
  for (int j = 0; j < D; ++j) gm[j] = ((j == g.r) ? 1.0 : 0.0) - gm[j];
  const Rw<D> ag = mm(g, rj.a, gm);
  const double t1 = matvec_t(g, ci, rj.eta);
  const double t2 = matvec(g, ci, t1);
  bo = matvec(g, ag, bi + t2) + rj.b;
  co = sqrt_sum_lt(g, mm(g, rj.a, w), rj.c);  // C_j: a tria output (IEKS aggregates)
  return !sing;
}

// ------------------------------------------------------ smoothing element ---
// make_smoothing_element (parallel.cpp:112-135).
template <int D>
__device__ __forceinline__ bool smoothing_element(const Grp<D>& g, const Gauss<D>& f, const Rw<D>& phi,
                                                  const Rw<D>& q, SEl<D>& el) {
  constexpr int K = 2 * D;
  Rw<K> top, bot;
  const Rw<D> pc = mm(g, phi, f.c);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    top[j] = pc[j];
    top[D + j] = q[j];
    bot[j] = f.c[j];
    bot[D + j] = 0.0;
  }
  lq<D, D, D, K>(g, top, bot);
  const bool sing = singular_diag(g, pick(top, g.r), D);
  Rw<D> p11, p21;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    p11[j] = top[j];
    p21[j] = bot[j];
    el.l[j] = bot[D + j];
  }
  publish_factor<D, D>(g, p11);
  el.e = solve_xl<D, D>(g, p21);  // E = Pi21 Pi11^-1
  const double pm = matvec(g, phi, f.m);
  el.g = f.m - matvec(g, el.e, pm);
  return !sing;
}

template <int D>
__device__ __forceinline__ SEl<D> terminal_smoothing_element(const Gauss<D>& f) {
  SEl<D> el;
  el.e = zeros<D>();
  el.g = f.m;
  el.l = f.c;
  return el;
}

// ⊗_s (parallel.cpp:146-156): E = E_i E_j, g = E_i g_j + g_i, L = tria([E_i L_j, L_i]).
template <int D>
__device__ __forceinline__ bool combine_smoothing(const Grp<D>& g, const SEl<D>& li, const SEl<D>& rj,
                                                  SEl<D>& out) {
  out.e = mm(g, li.e, rj.e);
  out.g = matvec(g, li.e, rj.g) + li.g;
  out.l = sqrt_sum(g, mm(g, li.e, rj.l), li.l);
  return true;
}

}  // namespace pode
