// Wide groups: ⊗_f on 2D lanes per element, for the latency-bound upper
// levels of the IEKS aggregate scan (engine.cuh k_bscan_loc_w).
//
// Why: a group-of-D-lanes combine (ops.cuh) is a dependent chain of ~3000
// instructions per lane, and its latency grows like D^2 (measured per
// Sklansky step at the scan's top levels: 2.2 / 3.9 / 4.5 / 8.7 / 13.5 /
// 18.2 us at D = 2 / 3 / 4 / 6 / 8 / 9), i.e. it is the per-lane work, not
// the pivot chain, that sets it.  The top levels only have a few dozen
// combines in flight, so spreading each combine over twice the lanes cuts
// their latency where the group layout leaves the GPU idle.
//
// Layout: lane w = h D + r of a wide group owns row r (0..D-1) in half h.
//  - The 2D-row stacked matrix of Xi = tria([[C_i^T J_j, I], [J_j, 0]])
//    (parallel.cpp:75-79) has one row per lane: top rows on half 0, bottom
//    rows on half 1, so each Householder reflector updates ONE row per lane.
//  - After Xi, the two output trias C = tria([A_j W, C_j]) and
//    J = tria([A_i^T Xi22, J_i]) (parallel.cpp:92-98) run side by side: half
//    0 the C sweep, half 1 the J sweep, in the same instruction stream.
//  - The D x D products are split the same way (A_j G | G A_i, then A_j W |
//    A_i^T Xi22), with operands picked per half from the group's tiles.
// Both halves hold every input row (loaded twice); the result rows are
// exchanged by shuffles at the end, so each lane again holds a whole FEl row.
// The algebra and the Householder convention are ops.cuh's combine_filtering
// (kTri: C and J are tria outputs).
#pragma once

#include "ops.cuh"

namespace pode {

template <int D>
struct GrpW {
  static constexpr int W = 2 * D;                              // lanes per element
  static constexpr int kPerWarp = 32 / W;                      // real groups per warp
  static constexpr int kSlots = kPerWarp + ((32 % W) ? 1 : 0);  // + phantom
  // tiles: T0, T2 (2D x D), T1 (2D x 2D); vectors: 2D (+ 2D spare)
  static constexpr int kT0 = 0, kT1 = 2 * D * D, kT2 = 6 * D * D, kV = 8 * D * D;
  static constexpr int kRaw = 8 * D * D + 4 * D;
  static constexpr int kDoubles = kRaw + (18 - kRaw % 16) % 16;  // 2 (mod 16): distinct bank slots per group
  int w, r, h, gw, base;
  double* s;  // group scratch
  __device__ __forceinline__ static GrpW make(double* warp_scratch) {
    GrpW g;
    const int lane = threadIdx.x & 31;
    g.gw = lane / W;
    g.w = lane - g.gw * W;
    g.h = g.w >= D ? 1 : 0;
    g.r = g.w - g.h * D;
    g.base = g.gw * W;
    g.s = warp_scratch + g.gw * kDoubles;
    return g;
  }
  __device__ __forceinline__ bool real() const { return gw < kPerWarp; }
};

// Every lane's row (K entries) into row w of the tile at `off` (row stride K).
template <int D, int K>
__device__ __forceinline__ void publish_w(const GrpW<D>& g, int off, const Rw<K>& row) {
  wsync();
  st_tile_row<K>(g.s + off + g.w * K, row);
  wsync();
}

// y = x . M with M (D rows, stride `stride`) at `m`: y_j = sum_k x_k M[k][j].
template <int D>
__device__ __forceinline__ Rw<D> row_times(const Rw<D>& x, const double* m, int stride) {
  Rw<D> y = zeros<D>();
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double xk = x[k];
#pragma unroll
    for (int j = 0; j < D; ++j) y[j] = fma(xk, m[k * stride + j], y[j]);
  }
  return y;
}

// Householder LQ of the group's 2D x K row set (one row per lane), pivots
// 0..P-1; pivot p's row lives on lane base + (pivot_half D) + p, so the two
// halves can run two independent D-row sweeps (pivot_half = h) or one
// 2D-row sweep whose pivots are the top rows (pivot_half = 0).
template <int D, int K, int P, int S = K>
__device__ __forceinline__ void lq_w(const GrpW<D>& g, int pivot_half, Rw<K>& row) {
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int src = g.base + pivot_half * D + p;
    Rw<K> x;
#pragma unroll
    for (int j = 0; j < K; ++j)
      x[j] = (j >= p && live_col(j, p, S)) ? __shfl_sync(0xffffffffu, row[j], src) : 0.0;
    const Reflector<K> hr = make_reflector<K, S>(x, p);
    apply_reflector<K, S>(hr, p, row);
    if (g.w == pivot_half * D + p) {
      row[p] = hr.beta;
#pragma unroll
      for (int j = p + 1; j < K; ++j) row[j] = 0.0;
    }
  }
}

// ⊗_f of IEKS aggregates (lower-triangular C and J), parallel.cpp:67-100.
template <int D>
__device__ __forceinline__ bool combine_filtering_w(const GrpW<D>& g, const FEl<D>& li, const FEl<D>& rj,
                                                    FEl<D>& out) {
  constexpr int K = 2 * D;
  const bool h1 = g.h != 0;
  double* const t0 = g.s + GrpW<D>::kT0;
  double* const t1 = g.s + GrpW<D>::kT1;
  double* const t2 = g.s + GrpW<D>::kT2;
  double* const v = g.s + GrpW<D>::kV;
  // 1. C_i (half 0) and J_j (half 1) rows into T0; eta_j (half 0) and b_i
  //    (half 1) entries into v
  {
    Rw<D> pub;
#pragma unroll
    for (int j = 0; j < D; ++j) pub[j] = h1 ? rj.j[j] : li.c[j];
    wsync();
    st_tile_row<D>(t0 + g.w * D, pub);
    v[g.w] = h1 ? li.b : rj.eta;
    wsync();
  }
  // X = C_i^T J_j (row r), t1 = C_i^T eta_j, u1 = J_j^T b_i (entry r)
  Rw<D> x = zeros<D>();
  double t1r = 0.0, u1r = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double ckr = t0[k * D + g.r];
    const double jkr = t0[(D + k) * D + g.r];
    const Rw<D> jk = ld_tile_row<D>(t0 + (D + k) * D);
#pragma unroll
    for (int j = 0; j < D; ++j) x[j] = fma(ckr, jk[j], x[j]);
    t1r = fma(ckr, v[k], t1r);
    u1r = fma(jkr, v[D + k], u1r);
  }
  // t2 = C_i t1, u2 = J_j u1 (row r): gather t1 (half 0) / u1 (half 1)
  wsync();
  v[2 * D + g.w] = h1 ? u1r : t1r;
  wsync();
  double t2r = 0.0, u2r = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    t2r = fma(li.c[k], v[2 * D + k], t2r);
    u2r = fma(rj.j[k], v[3 * D + k], u2r);
  }
  // 2. Xi: top rows [X | I] on half 0, bottom rows [J_j | 0] on half 1;
  //    D pivots on the top rows; right block [I; 0] lower triangular
  Rw<K> row;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    row[j] = h1 ? rj.j[j] : x[j];
    row[D + j] = (!h1 && j == g.r) ? 1.0 : 0.0;
  }
  lq_w<D, K, D, D>(g, 0, row);
  // singular Xi11 (the reference's test on its diagonal, linalg.cpp:54-62)
  bool sing;
  {
    const double a = h1 ? 0.0 : fabs(pick(row, g.r));
    wsync();
    v[g.w] = a;
    wsync();
    double mx = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) mx = fmax(mx, v[k]);
    bool s = false;
#pragma unroll
    for (int k = 0; k < D; ++k) s |= v[k] <= 1e-13 * mx;
    sing = s;
  }
  // 3. Xi rows into T1 (stride 2D); 1 / Xi11 diagonal
  wsync();
  st_tile_row<K>(t1 + g.w * K, row);
  if (!h1) v[2 * D + g.r] = 1.0 / row[g.r];
  wsync();
  // W = C_i Xi11^-T (row r; forward substitution), G = I - W Xi21^T
  Rw<D> wr;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double acc = li.c[i];
#pragma unroll
    for (int k = 0; k < i; ++k) acc = fma(-t1[i * K + k], wr[k], acc);
    wr[i] = acc * v[2 * D + i];
  }
  Rw<D> gr;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const Rw<D> xi21 = ld_tile_row<D>(t1 + (D + j) * K);
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) acc = fma(wr[k], xi21[k], acc);
    gr[j] = ((j == g.r) ? 1.0 : 0.0) - acc;
  }
  // 4. round A: half 0 ag = A_j G, half 1 ga = G A_i (T0: G rows | A_i rows)
  {
    Rw<D> pub;
#pragma unroll
    for (int j = 0; j < D; ++j) pub[j] = h1 ? li.a[j] : gr[j];
    publish_w<D, D>(g, GrpW<D>::kT0, pub);
  }
  Rw<D> left;
#pragma unroll
  for (int j = 0; j < D; ++j) left[j] = h1 ? gr[j] : rj.a[j];
  const Rw<D> pa = row_times<D>(left, t0 + (h1 ? D * D : 0), D);  // ag (h0) | ga (h1)
  // round B: half 0 aw = A_j W, half 1 ax = A_i^T Xi22 (T2: W rows | ga rows)
  {
    Rw<D> pub;
#pragma unroll
    for (int j = 0; j < D; ++j) pub[j] = h1 ? pa[j] : wr[j];
    publish_w<D, D>(g, GrpW<D>::kT2, pub);
  }
#pragma unroll
  for (int j = 0; j < D; ++j) left[j] = h1 ? t0[(D + j) * D + g.r] : rj.a[j];  // A_j row | A_i column
  const Rw<D> pb = row_times<D>(left, h1 ? t1 + D * K + D : t2, h1 ? K : D);  // aw (h0) | ax (h1)
  // A = A_j (G A_i) (every lane), eta = (G A_i)^T (eta_j - J_j J_j^T b_i) + eta_i
  out.a = row_times<D>(rj.a, t2 + D * D, D);
  const double vb = li.b + t2r;   // b_i + C_i C_i^T eta_j   (entry r)
  const double ve = rj.eta - u2r;  // eta_j - J_j J_j^T b_i  (entry r)
  wsync();
  v[g.w] = h1 ? ve : vb;
  wsync();
  double eo = li.eta, bo = rj.b;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    eo = fma(t2[(D + k) * D + g.r], v[D + k], eo);
    bo = fma(pa[k], v[k], bo);  // half 0: ag row r . vb
  }
  out.eta = eo;
  // 5. the two output trias side by side: half 0 [A_j W | C_j], half 1
  //    [A_i^T Xi22 | J_i] (right blocks lower triangular)
#pragma unroll
  for (int j = 0; j < D; ++j) {
    row[j] = pb[j];
    row[D + j] = h1 ? li.j[j] : rj.c[j];
  }
  lq_w<D, K, D, D>(g, g.h, row);
  // 6. exchange: each lane keeps its half's factor row and takes the other's
  const int partner = g.base + (h1 ? g.r : D + g.r);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double o = __shfl_sync(0xffffffffu, row[j], partner);
    out.c[j] = h1 ? o : row[j];
    out.j[j] = h1 ? row[j] : o;
  }
  const double bp = __shfl_sync(0xffffffffu, bo, partner);
  out.b = h1 ? bp : bo;
  return !sing;
}

template <int D>
struct FWOps : FOps<D> {
  __device__ static bool combine(const GrpW<D>& g, const FEl<D>& l, const FEl<D>& rr, FEl<D>& out) {
    return combine_filtering_w<D>(g, l, rr, out);
  }
};

}  // namespace pode

namespace pode {

// Block Sklansky scan of G = kBWarps * (32 / 2D) aggregates on wide groups:
// the contract of k_bscan_loc<D, FTOps<D>, false> (engine.cuh) — block-local
// inclusive prefixes in loc, the block aggregate in agg[blockIdx.x].
constexpr int kBWarpsW = 8;
template <int D>
constexpr int bscan_groups_w() {
  return kBWarpsW * GrpW<D>::kPerWarp;
}
template <int D>
constexpr size_t bscan_smem_w() {
  return sizeof(double) * (size_t(kBWarpsW) * GrpW<D>::kSlots * GrpW<D>::kDoubles +
                           size_t(bscan_groups_w<D>()) * FOps<D>::kDoubles);
}

template <int D>
__global__ void __launch_bounds__(kBWarpsW * 32, 1) k_bscan_loc_w(FEd x, int64_t n, FEd loc, FEd agg, DevError* err) {
  extern __shared__ double smem[];
  constexpr int G = bscan_groups_w<D>();
  const int warp = threadIdx.x >> 5;
  const GrpW<D> g = GrpW<D>::make(smem + warp * GrpW<D>::kSlots * GrpW<D>::kDoubles);
  const FEd sb = FOps<D>::smem_arr(smem + kBWarpsW * GrpW<D>::kSlots * GrpW<D>::kDoubles, G);
  // warp index in the low position bits (as k_bscan_loc)
  const int p = g.gw * kBWarpsW + warp;
  const bool real = g.real();
  const int64_t lo = int64_t(blockIdx.x) * G;
  const int64_t hi = min(n, lo + G);
  const int cnt = int(hi - lo);
  const bool ok = real && p < cnt;
  const int64_t k = lo + p;
  const bool writer = g.h == 0;  // both halves hold every row; half 0 stores
  FEl<D> acc = FOps<D>::load(x, k, g.r, ok);
  bool bad = false;
#pragma unroll 1
  for (int h = 1; h < cnt; h <<= 1) {  // cnt is block-uniform
    if (real && writer && (p & (2 * h - 1)) == h - 1) FOps<D>::store(sb, p, g.r, true, acc);
    __syncthreads();
    const bool rd = real && (p & h);
    if (h >= kBWarpsW || (warp & h)) {  // warp-uniform
      const int j = (p & ~(2 * h - 1)) + h - 1;
      const FEl<D> left = FOps<D>::load(sb, rd ? j : 0, g.r, rd);
      FEl<D> tmp;
      const bool good = combine_filtering_w<D>(g, left, acc, tmp);
      bad |= rd && ok && !good;
      acc = FOps<D>::select(rd, tmp, acc);
    }
  }
  FOps<D>::store(loc, k, g.r, ok && writer, acc);
  if (ok && writer && p == cnt - 1) FOps<D>::store(agg, blockIdx.x, g.r, true, acc);
  if (ok && g.w == 0 && bad) raise_error(err, k, kErrSingular);
}

}  // namespace pode
