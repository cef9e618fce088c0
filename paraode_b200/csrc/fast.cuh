// The fused IEKS iteration for an ODE information operator (the headline hot
// path), templated on the state dimension D and
// the ODE dimension d (D = d (q+1)).
//
// One Gauss-Newton iteration = five kernels over chunks of L time steps, one
// group of D lanes per chunk, nothing materialised per step except what the
// backward pass needs:
//   A  k_fast_fwd_reduce : per chunk, EK1-linearise each step on the fly
//                          (statespace.cpp:65-88 at eta[n+1], rescaled by
//                          T(h), ieks.cpp:160-164) and fold the chunk's
//                          filtering elements into one aggregate (A,b,C,eta,J)
//                          with a square-root Kalman recursion conditioned on
//                          the chunk's predecessor state — the same element
//                          algebra as make_filtering_element + ⊗_f
//                          (parallel.cpp:5-100) at a third of the flops.
//   B  scan of the chunk aggregates under ⊗_f (engine.cuh chunked scan).
//   C  k_fast_fwd_down   : from the chunk's incoming filtered marginal, run the
//                          square-root Kalman filter through the chunk; at
//                          every node form the smoothing element (E, g)
//                          (parallel.cpp:112-135, from the same Householder
//                          sweep as the prediction) and fold them into the
//                          chunk's backward aggregate.
//   D  reverse scan of the chunk backward aggregates (affine maps).
//   E  k_fast_bwd_down   : from the chunk's incoming smoothed mean, run the
//                          backward mean recursion, write the new trajectory
//                          in original coordinates and reduce the objective
//                          (ieks.cpp:49-60) and the stopping maxima
//                          (ieks.cpp:62-77) per chunk.
// Covariances, the innovation statistics and the calibration are formed
// once, after convergence (ieks.cpp:190-208), by the element/scan engine.
#pragma once

#include "engine.cuh"
#include "field.cuh"

namespace pode {

template <int D>
struct FastConst {
  double q[D * D];      // sigma * Q_bar^1/2 (rescaled process-noise factor)
  double qunit[D * D];  // Q_bar^1/2 (unit diffusion, objective metric)
  double qunit_rdiag[D];
  double m0[D];         // T_0^-1 mu_0
};

struct FastArgs {
  const double* grid;   // N+1 nodes
  const double* eta;    // linearisation points (original coordinates): (N+1) x D row-major for the
                        // group passes; chunk-interleaved (lane::eta_at) for the lane passes
  const double* eta_term;  // lane layout: node N
  int64_t N;
  int L;
  int64_t nchunks;
  int ek0;
  DevProblem prob;
  DevError* err;
};

__device__ __forceinline__ double ipow(double h, int k) {
  if (k == 0) return 1.0;
  if (k == 1) return h;
  if (k == 2) return h * h;
  return pow(h, double(k));
}

template <int D, int d>
struct Fast {
  static constexpr int B = D / d;  // q + 1
  static constexpr int q = B - 1;
  static_assert(B * d == D && B >= 2, "D must be d (q + 1) with q >= 1");

  // Node scale T(h_n) per derivative order (prior.cpp:79-97; node n uses its
  // incoming step, node 0 the first, ieks.cpp:28-33).
  __device__ static void taus(const double* grid, int64_t n, double (&t)[B], double (&ti)[B]) {
    const double h = (n == 0) ? grid[1] - grid[0] : grid[n] - grid[n - 1];
    const double rh = sqrt(h);
    double fact = 1.0;
#pragma unroll
    for (int i = q; i >= 0; --i) {
      const int k = q - i;
      if (k > 0) fact *= k;
      t[i] = rh * ipow(h, k) / fact;
      ti[i] = 1.0 / t[i];
    }
  }

  // This lane's row of the binomial block (prior.cpp:99-107): coef[i] for
  // columns base + i of its block.
  struct PhiRow {
    int base;
    double coef[B];
  };
  __device__ static PhiRow phi_row(int r) {
    PhiRow p;
    const int a = r % B;
    p.base = r - a;
#pragma unroll
    for (int i = 0; i < B; ++i) {
      double c = 0.0;
      if (i >= a) {  // binomial(q - a, i - a)
        const int n = q - a, k = i - a;
        double num = 1.0, den = 1.0;
        for (int t = 0; t < k; ++t) {
          num *= double(n - t);
          den *= double(t + 1);
        }
        c = num / den;
      }
      p.coef[i] = c;
    }
    return p;
  }

  // Rows of phi_n X: phi_n = phi_bar diag(T_n ⊙ T_{n+1}^-1) (ieks.cpp:37-45);
  // X published in the group tile (stride K).
  template <int K>
  __device__ static Rw<K> phi_rows(const Grp<D>& g, const PhiRow& pr, const double (&ratio)[B], const Rw<K>& x) {
    publish<D, K>(g, x);
    Rw<K> o = zeros<K>();
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const double c = pr.coef[i] * ratio[i];
      const double* row = g.sc + (pr.base + i) * K;
#pragma unroll
      for (int j = 0; j < K; ++j) o[j] = fma(c, row[j], o[j]);
    }
    return o;
  }

  __device__ static double phi_vec(const Grp<D>& g, const PhiRow& pr, const double (&ratio)[B], double x) {
    const int lane0 = (threadIdx.x & 31) - g.r;
    double o = 0.0;
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const double xi = __shfl_sync(0xffffffffu, x, lane0 + pr.base + i);
      o = fma(pr.coef[i] * ratio[i], xi, o);
    }
    return o;
  }

  // EK1 / EK0 linearisation at node n (statespace.cpp:65-103): every lane
  // evaluates f and F_y redundantly; lanes i < d own observation row i.
  struct Lin {
    double off;      // offset_i on lane i < d, 0 elsewhere
    double jac[d * d];
    bool finite;
  };
  __device__ static Lin linearize(const FastArgs& a, int64_t n, int r, bool ok) {
    Lin l;
    double y[d], f[d];
#pragma unroll
    for (int j = 0; j < d; ++j) y[j] = ok ? a.eta[n * D + j * B] : 0.0;
    eval_field<d>(a.prob, y, f, l.jac);
    bool fin = true;
#pragma unroll
    for (int j = 0; j < d; ++j) fin &= isfinite(f[j]);
    if (!a.ek0) {
#pragma unroll
      for (int k = 0; k < d * d; ++k) fin &= isfinite(l.jac[k]);
    } else {
#pragma unroll
      for (int k = 0; k < d * d; ++k) l.jac[k] = 0.0;
    }
    l.finite = fin;
    double off = 0.0;
#pragma unroll
    for (int i = 0; i < d; ++i) {
      double jy = 0.0;
#pragma unroll
      for (int j = 0; j < d; ++j) jy += l.jac[i * d + j] * y[j];
      const double oi = a.ek0 ? f[i] : f[i] - jy;
      off = (r == i) ? oi : off;
    }
    l.off = off;
    return l;
  }

  // Rows of H_bar X for H_bar = (E_1 - F_y E_0) diag(T_{n}) (lanes i < d;
  // zero rows elsewhere), X published in the tile (stride K).
  template <int K>
  __device__ static Rw<K> h_rows(const Grp<D>& g, const Lin& l, const double (&t)[B], const Rw<K>& x) {
    publish<D, K>(g, x);
    Rw<K> o = zeros<K>();
    const int i = g.r < d ? g.r : 0;
    const double* r1 = g.sc + (i * B + 1) * K;
    const double s1 = (g.r < d) ? 1.0 * t[1] : 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) o[j] = s1 * r1[j];
#pragma unroll
    for (int c = 0; c < d; ++c) {
      double jic = 0.0;
#pragma unroll
      for (int ii = 0; ii < d; ++ii) jic = (ii == i) ? l.jac[ii * d + c] : jic;
      const double coef = (g.r < d) ? (-jic) * t[0] : 0.0;
      const double* rc = g.sc + (c * B) * K;
#pragma unroll
      for (int j = 0; j < K; ++j) o[j] = fma(coef, rc[j], o[j]);
    }
    return o;
  }

  __device__ static double h_vec(const Grp<D>& g, const Lin& l, const double (&t)[B], double x) {
    const int lane0 = (threadIdx.x & 31) - g.r;
    const int i = g.r < d ? g.r : 0;
    double o = (g.r < d ? 1.0 * t[1] : 0.0) * __shfl_sync(0xffffffffu, x, lane0 + i * B + 1);
#pragma unroll
    for (int c = 0; c < d; ++c) {
      double jic = 0.0;
#pragma unroll
      for (int ii = 0; ii < d; ++ii) jic = (ii == i) ? l.jac[ii * d + c] : jic;
      const double xc = __shfl_sync(0xffffffffu, x, lane0 + c * B);
      o = fma((g.r < d) ? (-jic) * t[0] : 0.0, xc, o);
    }
    return o;
  }

  // Square-root measurement update against the noiseless d-row observation:
  // Psi = tria([[H C], [C]]) (sequential.cpp:41-67 with R = 0).  Returns the
  // gain row K[r, 0..d), S^1/2 (d x d, on every lane) and C+.
  struct Upd {
    double k[d];
    double s[d][d];
    double sinv[d];
    Rw<D> cplus;
    bool singular;
  };
  __device__ static Upd update(const Grp<D>& g, const Lin& l, const double (&t)[B], const Rw<D>& cpred) {
    Upd u;
    Rw<D> top = h_rows<D>(g, l, t, cpred);
    Rw<D> bot = cpred;
    lq<D, d, D, D>(g, top, bot);
    u.singular = singular_diag(g, pick(top, g.r < d ? g.r : D), d);
    const int lane0 = (threadIdx.x & 31) - g.r;
#pragma unroll
    for (int i = 0; i < d; ++i) {
#pragma unroll
      for (int j = 0; j < d; ++j) {
        const double v = __shfl_sync(0xffffffffu, top[j], lane0 + i);
        u.s[i][j] = (j <= i) ? v : 0.0;
      }
      u.sinv[i] = rcp_nr(u.s[i][i]);
    }
    // K = Psi21 S^-1 (row r: x S = Psi21[r, :], back substitution)
#pragma unroll
    for (int i = d - 1; i >= 0; --i) {
      double acc = bot[i];
#pragma unroll
      for (int k = i + 1; k < d; ++k) acc = fma(-u.k[k], u.s[k][i], acc);
      u.k[i] = acc * u.sinv[i];
    }
#pragma unroll
    for (int j = 0; j < D; ++j) u.cplus[j] = (j < D - d) ? bot[d + j] : 0.0;
    return u;
  }

  // w = S^-1 v (forward substitution, every lane, registers only).
  __device__ static void s_solve(const Upd& u, const double (&v)[d], double (&w)[d]) {
#pragma unroll
    for (int i = 0; i < d; ++i) {
      double acc = v[i];
#pragma unroll
      for (int k = 0; k < i; ++k) acc = fma(-u.s[i][k], w[k], acc);
      w[i] = acc * u.sinv[i];
    }
  }

  // Entries i < d of a vector held on lanes 0..d-1, on every lane.
  __device__ static void gather_d(const Grp<D>& g, double x, double (&v)[d]) {
    const int lane0 = (threadIdx.x & 31) - g.r;
#pragma unroll
    for (int i = 0; i < d; ++i) v[i] = __shfl_sync(0xffffffffu, x, lane0 + i);
  }
};

// ------------------------------------------------------------- pass A ---
template <int D, int d>
__global__ void __launch_bounds__(kThreads) k_fast_fwd_reduce(FastArgs a, FastConst<D> cst, FEd agg) {
  using F = Fast<D, d>;
  constexpr int B = F::B;
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t c = group_index<D>(g);
  const bool okc = g.real() && c < a.nchunks;
  const int64_t s = c * a.L;
  const typename F::PhiRow pr = F::phi_row(g.r);
  Rw<D> qrow;
#pragma unroll
  for (int j = 0; j < D; ++j) qrow[j] = cst.q[g.r * D + j];
  // chunk 0 starts from the (known) initial distribution; every other chunk
  // from its unknown predecessor x_{s-1}: (A, b, C) = (I, 0, 0).
  Rw<D> A, C = zeros<D>(), J = zeros<D>();
  double b = (c == 0) ? cst.m0[g.r] : 0.0, eta = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) A[j] = (c != 0 && j == g.r) ? 1.0 : 0.0;
  double tk[B], tki[B], tn[B], tni[B];
  F::taus(a.grid, okc ? s : 0, tk, tki);
  bool bad_sing = false, bad_lin = false;
  int64_t bad_at = 0;
  for (int t = 0; t < a.L; ++t) {
    const int64_t k = s + t;  // step k: node k -> node k+1
    const bool ok = okc && k < a.N;
    F::taus(a.grid, ok ? k + 1 : 1, tn, tni);
    double ratio[B];
#pragma unroll
    for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tni[i];
    // predict: A- = phi A, b- = phi b, C- = tria([phi C, Q])
    const Rw<D> am = F::template phi_rows<D>(g, pr, ratio, A);
    const double bm = F::phi_vec(g, pr, ratio, b);
    const Rw<D> pc = F::template phi_rows<D>(g, pr, ratio, C);
    Rw<2 * D> st;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      st[j] = pc[j];
      st[D + j] = qrow[j];
    }
    const Rw<D> cm = tria<D, 2 * D>(g, st);
    // update against the linearised ODE information operator at node k+1
    const typename F::Lin lin = F::linearize(a, ok ? k + 1 : 0, g.r, ok);
    const typename F::Upd u = F::update(g, lin, tn, cm);
    // U = H A-, u = H b- - offset; A+ = A- - K U, b+ = b- - K u
    const Rw<D> U = F::template h_rows<D>(g, lin, tn, am);  // rows i < d
    const double uu = F::h_vec(g, lin, tn, bm) - lin.off;
    publish<D, D>(g, U);
    double uv[d], ucol[d], wcol[d], ubar[d];
    F::gather_d(g, uu, uv);
#pragma unroll
    for (int i = 0; i < d; ++i) ucol[i] = g.sc[i * D + g.r];
    Rw<D> an;
    double bn = bm;
#pragma unroll
    for (int j = 0; j < D; ++j) an[j] = am[j];
#pragma unroll
    for (int i = 0; i < d; ++i) {
#pragma unroll
      for (int j = 0; j < D; ++j) an[j] = fma(-u.k[i], g.sc[i * D + j], an[j]);
      bn = fma(-u.k[i], uv[i], bn);
    }
    // likelihood of the step's observation given x_{s-1}:
    //   Ubar = S^-1 U, ubar = S^-1 u; J += Ubar^T Ubar, eta -= Ubar^T ubar
    F::s_solve(u, ucol, wcol);
    F::s_solve(u, uv, ubar);
    Rw<D + d> jr;
#pragma unroll
    for (int j = 0; j < D; ++j) jr[j] = J[j];
    double de = 0.0;
#pragma unroll
    for (int i = 0; i < d; ++i) {
      jr[D + i] = wcol[i];
      de = fma(wcol[i], ubar[i], de);
    }
    Rw<D + d> none = zeros<D + d>();
    lq<D, 0, D, D + d>(g, none, jr);
    // commit (masked for padded steps)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      A[j] = ok ? an[j] : A[j];
      C[j] = ok ? u.cplus[j] : C[j];
      J[j] = ok ? jr[j] : J[j];
    }
    b = ok ? bn : b;
    eta = ok ? eta - de : eta;
    bad_sing |= ok && u.singular;
    if (ok && !lin.finite && !bad_lin) {
      bad_lin = true;
      bad_at = k + 1;
    }
#pragma unroll
    for (int i = 0; i < B; ++i) {
      tk[i] = tn[i];
      tki[i] = tni[i];
    }
  }
  if (okc && g.r == 0) {
    if (bad_lin) raise_error(a.err, bad_at, kErrLinearization);
    if (bad_sing) raise_error(a.err, s, kErrSingular);
  }
  FEl<D> e{A, b, C, eta, J};
  FOps<D>::store(agg, c, g.r, okc, e);
}

// ------------------------------------------------------------- pass C ---
// prefix: inclusive ⊗_f scan of the pass-A aggregates (prefix[c-1] = the
// filtered marginal at the first node of chunk c).  Writes the smoothing
// elements (E_n, g_n) of nodes 0..N and the chunk's backward aggregate.
template <int D, int d>
__global__ void __launch_bounds__(kThreads) k_fast_fwd_down(FastArgs a, FastConst<D> cst, FEd prefix,
                                                            SEd elems, SEd bagg) {
  using F = Fast<D, d>;
  constexpr int B = F::B;
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t c = group_index<D>(g);
  const bool okc = g.real() && c < a.nchunks;
  const int64_t s = c * a.L;
  const typename F::PhiRow pr = F::phi_row(g.r);
  Rw<D> qrow;
#pragma unroll
  for (int j = 0; j < D; ++j) qrow[j] = cst.q[g.r * D + j];
  const bool from_init = c == 0;
  double m = from_init ? cst.m0[g.r] : ld_ent<D>(prefix.b, c - 1, g.r, okc && !from_init);
  Rw<D> C = ld_row<D>(prefix.c, c - 1, g.r, okc && !from_init);
  Rw<D> eagg = zeros<D>();
  double gagg = 0.0;
  bool have = false, bad_sing = false, bad_lin = false;
  int64_t bad_at = 0;
  double tk[B], tki[B], tn[B], tni[B];
  F::taus(a.grid, okc ? s : 0, tk, tki);
  for (int t = 0; t < a.L; ++t) {
    const int64_t k = s + t;
    const bool ok = okc && k < a.N;
    F::taus(a.grid, ok ? k + 1 : 1, tn, tni);
    double ratio[B];
#pragma unroll
    for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tni[i];
    // Pi = tria([[phi C, Q], [C, 0]]), first D pivots: Pi11 = C- (the
    // prediction factor), Pi21 -> E = Pi21 Pi11^-1 (parallel.cpp:112-135).
    const Rw<D> pc = F::template phi_rows<D>(g, pr, ratio, C);
    Rw<2 * D> top, bot;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      top[j] = pc[j];
      top[D + j] = qrow[j];
      bot[j] = C[j];
      bot[D + j] = 0.0;
    }
    lq<D, D, 0, 2 * D>(g, top, bot);
    Rw<D> cm, p21;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      cm[j] = top[j];
      p21[j] = bot[j];
    }
    const bool sing_pred = singular_diag(g, pick(top, g.r), D);
    publish_factor<D, D>(g, cm);
    const Rw<D> E = solve_xl<D, D>(g, p21);
    const double mm_ = F::phi_vec(g, pr, ratio, m);
    const double gk = m - matvec(g, E, mm_);
    st_row<D>(elems.e, k, g.r, ok, E);
    st_ent<D>(elems.g, k, g.r, ok, gk);
    // fold into the chunk's backward aggregate (time order, ⊗_s on (E, g))
    const Rw<D> ef = mm(g, eagg, E);
    const double gf = matvec(g, eagg, gk) + gagg;
#pragma unroll
    for (int j = 0; j < D; ++j) eagg[j] = ok ? (have ? ef[j] : E[j]) : eagg[j];
    gagg = ok ? (have ? gf : gk) : gagg;
    have = have || ok;
    // measurement update at node k+1
    const typename F::Lin lin = F::linearize(a, ok ? k + 1 : 0, g.r, ok);
    const typename F::Upd u = F::update(g, lin, tn, cm);
    const double z = F::h_vec(g, lin, tn, mm_) - lin.off;
    double zv[d];
    F::gather_d(g, z, zv);
    double mp = mm_;
#pragma unroll
    for (int i = 0; i < d; ++i) mp = fma(-u.k[i], zv[i], mp);
    m = ok ? mp : m;
#pragma unroll
    for (int j = 0; j < D; ++j) C[j] = ok ? u.cplus[j] : C[j];
    bad_sing |= ok && (u.singular || sing_pred);
    if (ok && !lin.finite && !bad_lin) {
      bad_lin = true;
      bad_at = k + 1;
    }
#pragma unroll
    for (int i = 0; i < B; ++i) {
      tk[i] = tn[i];
      tki[i] = tni[i];
    }
  }
  // terminal node N (parallel.cpp:137-144): E = 0, g = m_f(N)
  const bool last = okc && s + a.L >= a.N;
  st_row<D>(elems.e, a.N, g.r, last, zeros<D>());
  st_ent<D>(elems.g, a.N, g.r, last, m);
  const double gt = matvec(g, eagg, m) + gagg;
  if (last) {
    eagg = zeros<D>();
    gagg = gt;
  }
  if (okc && g.r == 0) {
    if (bad_lin) raise_error(a.err, bad_at, kErrLinearization);
    if (bad_sing) raise_error(a.err, s, kErrSingular);
  }
  st_row<D>(bagg.e, c, g.r, okc, eagg);
  st_ent<D>(bagg.g, c, g.r, okc, gagg);
}

// ------------------------------------------------------------- pass E ---
// suffix: reverse inclusive scan of the pass-C aggregates (suffix[c+1].g =
// the smoothed mean at the last node of chunk c).  kInitial evaluates the
// objective of eta_old itself (the constant start, ieks.cpp:147-148).
// part[c] = (sum of whitened increments, max |d eta|, max |eta|).
template <int D, int d, bool kInitial>
__global__ void __launch_bounds__(kThreads) k_fast_bwd_down(FastArgs a, FastConst<D> cst, SEd elems,
                                                            SEd suffix, const double* eta_old,
                                                            double* eta_new, double* part) {
  using F = Fast<D, d>;
  constexpr int B = F::B;
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t c = group_index<D>(g);
  const bool okc = g.real() && c < a.nchunks;
  const int64_t s = c * a.L;
  const int64_t e = min(a.N, s + a.L);  // last node of the chunk
  const typename F::PhiRow pr = F::phi_row(g.r);
  const bool last = c == a.nchunks - 1;
  // smoothed mean at node e
  double mu;
  if (kInitial) {
    mu = 0.0;
  } else {
    mu = last ? ld_ent<D>(elems.g, a.N, g.r, okc) : ld_ent<D>(suffix.g, c + 1, g.r, okc && !last);
  }
  double te[B], tei[B];
  F::taus(a.grid, okc ? e : 0, te, tei);
  const int br = g.r % B;
  double eta_e = kInitial ? (okc ? eta_old[e * D + g.r] : 0.0) : te[br] * mu;
  double dmax = 0.0, emax = 0.0;
  if (last && okc) {  // node N belongs to the last chunk
    if (!kInitial) eta_new[a.N * D + g.r] = eta_e;
    dmax = fabs(eta_e - eta_old[a.N * D + g.r]);
    emax = fabs(eta_e);
  }
  double bar_next = tei[br] * eta_e;  // rescaled state at node k+1
  Rw<D> qu;
#pragma unroll
  for (int j = 0; j < D; ++j) qu[j] = cst.qunit[g.r * D + j];
  double obj = 0.0;
  double tn[B], tni[B];
#pragma unroll
  for (int i = 0; i < B; ++i) {
    tn[i] = te[i];
    tni[i] = tei[i];
  }
  for (int t = 0; t < a.L; ++t) {
    const int64_t k = s + (a.L - 1 - t);
    const bool ok = okc && k < a.N;
    double tk[B], tki[B];
    F::taus(a.grid, ok ? k : 0, tk, tki);
    double eta_k;
    if (kInitial) {
      eta_k = ok ? eta_old[k * D + g.r] : 0.0;
    } else {
      const Rw<D> E = ld_row<D>(elems.e, k, g.r, ok);
      const double gk = ld_ent<D>(elems.g, k, g.r, ok);
      const double mk = gk + matvec(g, E, mu);
      mu = ok ? mk : mu;
      eta_k = tk[br] * mk;
      if (ok) eta_new[k * D + g.r] = eta_k;
    }
    const double old = ok ? eta_old[k * D + g.r] : 0.0;
    if (ok) {
      dmax = fmax(dmax, fabs(eta_k - old));
      emax = fmax(emax, fabs(eta_k));
    }
    // objective term of step k: || Qunit^-1/2 (bar_{k+1} - phi_k bar_k) ||^2
    const double bar_k = tki[br] * eta_k;
    double ratio[B];
#pragma unroll
    for (int i = 0; i < B; ++i) ratio[i] = tk[i] * tni[i];
    const double inc = bar_next - F::phi_vec(g, pr, ratio, bar_k);
    const Rw<D> iv = gather_vec(g, inc);
    double w[D], acc2 = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double acc = iv[i];
#pragma unroll
      for (int k2 = 0; k2 < i; ++k2) acc = fma(-cst.qunit[i * D + k2], w[k2], acc);
      w[i] = acc * cst.qunit_rdiag[i];
      acc2 = fma(w[i], w[i], acc2);
    }
    obj += ok ? acc2 : 0.0;
    bar_next = ok ? bar_k : bar_next;
#pragma unroll
    for (int i = 0; i < B; ++i) {
      tn[i] = ok ? tk[i] : tn[i];
      tni[i] = ok ? tki[i] : tni[i];
    }
  }
  (void)qu;
  const double dm = group_max(g, dmax);
  const double em = group_max(g, emax);
  if (okc && g.r == 0) {
    part[c * 3 + 0] = obj;
    part[c * 3 + 1] = dm;
    part[c * 3 + 2] = em;
  }
}

}  // namespace pode
