// Per-state-dimension engine: element kernels, the chunked associative scans
// and the smoother built from them.  Instantiated once per D in inst_*.cu.
//
// Scan design (replaces associative_scan / scan_in_place,
// proj/include/paraode/parallel.hpp:86-149): a reduce-then-scan over chunks.
// Each group of D lanes folds one chunk of L consecutive elements in time
// order (reduce), the chunk aggregates are scanned recursively with the same
// kernels, and each group re-folds its chunk from its exclusive carry
// (downsweep).  The combination tree depends only on (n, L), so results are
// bitwise reproducible run to run; work is <= 2n combines.
#pragma once

#include <functional>

#include <algorithm>
#include <mutex>
#include <cstdlib>
#include <vector>

#include "context.hpp"
#include "ops.cuh"

namespace pode {

constexpr int kWarpsPerBlock = 4;

// Runs a function-attribute setup once per device, thread-safe (several
// host threads may drive their own contexts concurrently).
struct OncePerDevice {
  std::mutex m;
  unsigned long long done = 0;
  template <class F>
  void operator()(F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(m);
    if ((done >> dev) & 1ull) return;
    f();
    done |= 1ull << dev;
  }
};
constexpr int kThreads = 32 * kWarpsPerBlock;

struct FEd {  // device filtering-element arrays
  double *a, *b, *c, *eta, *j;
};
struct SEd {
  double *e, *g, *l;
};

struct DevChain {  // device view of pode_chain
  int D, M;
  int64_t N;
  const double* init_mean;
  const double* init_cov;
  const double* phi;
  const double* q;
  int phi_shared, q_shared;
  const int32_t* obs_rows;
  const double* h;
  const double* off;
  const double* r;
};

struct ScanTally {
  int64_t combines = 0;
  int64_t depth = 0;
};

template <int D>
constexpr size_t smem_bytes() {
  return sizeof(double) * kWarpsPerBlock * Grp<D>::kSlots * Scratch<D>::kDoubles;
}

template <int D>
__device__ __forceinline__ Grp<D> make_group(double* smem) {
  const int warp = threadIdx.x >> 5;
  return Grp<D>::make(smem + warp * Grp<D>::kSlots * Scratch<D>::kDoubles);
}

// Global group index of this lane's group.
template <int D>
__device__ __forceinline__ int64_t group_index(const Grp<D>& g) {
  const int warp = threadIdx.x >> 5;
  return (static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + warp) * Grp<D>::kPerWarp + g.gw;
}

template <int D>
inline unsigned blocks_for(int64_t groups) {
  const int64_t per_block = int64_t(kWarpsPerBlock) * Grp<D>::kPerWarp;
  return static_cast<unsigned>((groups + per_block - 1) / per_block);
}

// ------------------------------------------------------------ load/store ---
template <int D>
__device__ __forceinline__ Rw<D> ld_row(const double* base, int64_t i, int r, bool ok) {
  Rw<D> o;
  const double* p = base + (i * D + r) * D;
#pragma unroll
  for (int j = 0; j < D; ++j) o[j] = ok ? p[j] : 0.0;
  return o;
}
template <int D>
__device__ __forceinline__ void st_row(double* base, int64_t i, int r, bool ok, const Rw<D>& x) {
  if (!ok) return;
  double* p = base + (i * D + r) * D;
#pragma unroll
  for (int j = 0; j < D; ++j) p[j] = x[j];
}
template <int D>
__device__ __forceinline__ double ld_ent(const double* base, int64_t i, int r, bool ok) {
  return ok ? base[i * D + r] : 0.0;
}
template <int D>
__device__ __forceinline__ void st_ent(double* base, int64_t i, int r, bool ok, double x) {
  if (ok) base[i * D + r] = x;
}

template <int D>
struct FOps {
  using El = FEl<D>;
  using Arr = FEd;
  static constexpr const char* kReduce = "scan_f_reduce";
  static constexpr const char* kDown = "scan_f_down";
  __device__ static El load(const Arr& x, int64_t i, int r, bool ok) {
    El e;
    e.a = ld_row<D>(x.a, i, r, ok);
    e.b = ld_ent<D>(x.b, i, r, ok);
    e.c = ld_row<D>(x.c, i, r, ok);
    e.eta = ld_ent<D>(x.eta, i, r, ok);
    e.j = ld_row<D>(x.j, i, r, ok);
    return e;
  }
  __device__ static void store(const Arr& x, int64_t i, int r, bool ok, const El& e) {
    st_row<D>(x.a, i, r, ok, e.a);
    st_ent<D>(x.b, i, r, ok, e.b);
    st_row<D>(x.c, i, r, ok, e.c);
    st_ent<D>(x.eta, i, r, ok, e.eta);
    st_row<D>(x.j, i, r, ok, e.j);
  }
  __device__ static bool combine(const Grp<D>& g, const El& l, const El& rr, El& out) {
    return combine_filtering<D>(g, l, rr, out);
  }
  static constexpr int kDoubles = 3 * D * D + 2 * D;  // one element
  __device__ static Arr smem_arr(double* buf, int n) {
    return Arr{buf, buf + 3 * n * D * D, buf + n * D * D, buf + 3 * n * D * D + n * D, buf + 2 * n * D * D};
  }
  __device__ static El select(bool take_a, const El& a, const El& b) {
    El o;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      o.a[j] = take_a ? a.a[j] : b.a[j];
      o.c[j] = take_a ? a.c[j] : b.c[j];
      o.j[j] = take_a ? a.j[j] : b.j[j];
    }
    o.b = take_a ? a.b : b.b;
    o.eta = take_a ? a.eta : b.eta;
    return o;
  }
};

template <int D>
struct SOps {
  using El = SEl<D>;
  using Arr = SEd;
  static constexpr const char* kReduce = "scan_s_reduce";
  static constexpr const char* kDown = "scan_s_down";
  __device__ static El load(const Arr& x, int64_t i, int r, bool ok) {
    El e;
    e.e = ld_row<D>(x.e, i, r, ok);
    e.g = ld_ent<D>(x.g, i, r, ok);
    e.l = ld_row<D>(x.l, i, r, ok);
    return e;
  }
  __device__ static void store(const Arr& x, int64_t i, int r, bool ok, const El& e) {
    st_row<D>(x.e, i, r, ok, e.e);
    st_ent<D>(x.g, i, r, ok, e.g);
    st_row<D>(x.l, i, r, ok, e.l);
  }
  __device__ static bool combine(const Grp<D>& g, const El& l, const El& rr, El& out) {
    return combine_smoothing<D>(g, l, rr, out);
  }
  __device__ static El select(bool take_a, const El& a, const El& b) {
    El o;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      o.e[j] = take_a ? a.e[j] : b.e[j];
      o.l[j] = take_a ? a.l[j] : b.l[j];
    }
    o.g = take_a ? a.g : b.g;
    return o;
  }
};

// Mean-only smoothing elements (E, g): the IEKS iterations need smoothed
// means only; covariances are formed once after convergence.
template <int D>
struct MOps {
  struct El {
    Rw<D> e;
    double g;
  };
  using Arr = SEd;  // l unused
  static constexpr const char* kReduce = "scan_m_reduce";
  static constexpr const char* kDown = "scan_m_down";
  __device__ static El load(const Arr& x, int64_t i, int r, bool ok) {
    El e;
    e.e = ld_row<D>(x.e, i, r, ok);
    e.g = ld_ent<D>(x.g, i, r, ok);
    return e;
  }
  __device__ static void store(const Arr& x, int64_t i, int r, bool ok, const El& e) {
    st_row<D>(x.e, i, r, ok, e.e);
    st_ent<D>(x.g, i, r, ok, e.g);
  }
  __device__ static bool combine(const Grp<D>& g, const El& l, const El& rr, El& out) {
    out.e = mm(g, l.e, rr.e);
    out.g = matvec(g, l.e, rr.g) + l.g;
    return true;
  }
  static constexpr int kDoubles = D * D + D;
  __device__ static Arr smem_arr(double* buf, int n) { return Arr{buf, buf + n * D * D, nullptr}; }
  __device__ static El select(bool take_a, const El& a, const El& b) {
    El o;
#pragma unroll
    for (int j = 0; j < D; ++j) o.e[j] = take_a ? a.e[j] : b.e[j];
    o.g = take_a ? a.g : b.g;
    return o;
  }
};

// ------------------------------------------------------ batched combines ---
template <int D, class Op>
__global__ void __launch_bounds__(kThreads) k_combine(int64_t count, typename Op::Arr lhs,
                                                      typename Op::Arr rhs, typename Op::Arr out,
                                                      DevError* err) {
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t i = group_index<D>(g);
  const bool ok = g.real() && i < count;
  const auto l = Op::load(lhs, i, g.r, ok);
  const auto rr = Op::load(rhs, i, g.r, ok);
  typename Op::El o;
  const bool good = Op::combine(g, l, rr, o);
  if (ok && g.r == 0 && !good) raise_error(err, i, kErrSingular);
  Op::store(out, i, g.r, ok, o);
}

// ------------------------------------------------------------- observation ---
template <int D>
__device__ __forceinline__ Obs<D, D> load_obs(const DevChain& ch, int64_t i, int r, bool ok) {
  Obs<D, D> o;
  const int m = ok ? ch.obs_rows[i] : 0;
  o.m = m;
  const int M = ch.M;
  const bool real_row = ok && r < m;
#pragma unroll
  for (int j = 0; j < D; ++j) o.h[j] = real_row ? ch.h[(i * M + r) * D + j] : 0.0;
  o.off = real_row ? ch.off[i * M + r] : 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (real_row)
      o.r[j] = (j < m) ? ch.r[(i * M + r) * M + j] : 0.0;
    else
      o.r[j] = (j == r) ? 1.0 : 0.0;  // unit-noise dummy row
  }
  return o;
}

template <int D>
__device__ __forceinline__ Rw<D> chain_phi(const DevChain& ch, int64_t i, int r, bool ok) {
  return ld_row<D>(ch.phi, ch.phi_shared ? 0 : i, r, ok);
}
template <int D>
__device__ __forceinline__ Rw<D> chain_q(const DevChain& ch, int64_t i, int r, bool ok) {
  return ld_row<D>(ch.q, ch.q_shared ? 0 : i, r, ok);
}

// make_filtering_element for every step (parallel.cpp:5-65).
template <int D>
__global__ void __launch_bounds__(kThreads) k_make_filtering(DevChain ch, int absorb_init, FEd out,
                                                             DevError* err) {
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t i = group_index<D>(g);
  const bool ok = g.real() && i < ch.N;
  const Rw<D> phi = chain_phi<D>(ch, i, g.r, ok);
  const Rw<D> q = chain_q<D>(ch, i, g.r, ok);
  const Obs<D, D> o = load_obs<D>(ch, i, g.r, ok);
  FEl<D> el;
  bool good;
  // Warp-uniform: every group evaluates both forms, the first step keeps
  // the init-absorbing one.
  FEl<D> e_first;
  Gauss<D> init;
  init.m = ok ? ch.init_mean[g.r] : 0.0;
  init.c = ld_row<D>(ch.init_cov, 0, g.r, ok);
  const bool good_first = first_filtering_element<D, D>(g, init, phi, q, o, e_first);
  const bool good_int = filtering_element<D, D>(g, phi, q, o, el);
  const bool first = absorb_init && i == 0;
  el = FOps<D>::select(first, e_first, el);
  good = first ? good_first : good_int;
  if (ok && g.r == 0 && !good) raise_error(err, i, kErrSingular);
  FOps<D>::store(out, i, g.r, ok, el);
}

// Smoothing elements for nodes 0..N (parallel.cpp:112-144).
template <int D>
__global__ void __launch_bounds__(kThreads) k_make_smoothing(DevChain ch, const double* fm,
                                                             const double* fc, SEd out, DevError* err) {
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t i = group_index<D>(g);
  const bool ok = g.real() && i <= ch.N;
  const bool terminal = i == ch.N;
  const bool ok_t = ok && !terminal;
  Gauss<D> f;
  f.m = ld_ent<D>(fm, i, g.r, ok);
  f.c = ld_row<D>(fc, i, g.r, ok);
  const Rw<D> phi = chain_phi<D>(ch, i, g.r, ok_t);
  const Rw<D> q = chain_q<D>(ch, i, g.r, ok_t);
  SEl<D> el;
  const bool good = smoothing_element<D>(g, f, phi, q, el);
  el = SOps<D>::select(terminal, terminal_smoothing_element<D>(f), el);
  if (ok_t && g.r == 0 && !good) raise_error(err, i, kErrSingular);
  SOps<D>::store(out, i, g.r, ok, el);
}

// ------------------------------------------------------------------ scans ---
// Reduce: agg[c] = x[cL] ⊗ .. ⊗ x[min(n, (c+1)L) - 1].
template <int D, class Op>
__global__ void __launch_bounds__(kThreads) k_scan_reduce(typename Op::Arr x, int64_t n, int L,
                                                          typename Op::Arr agg, DevError* err) {
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t c = group_index<D>(g);
  const int64_t lo = c * L;
  const int64_t hi = min(n, lo + L);
  const bool okc = g.real() && lo < n;
  auto acc = Op::load(x, lo, g.r, okc);
  bool bad = false;
  for (int t = 1; t < L; ++t) {
    const int64_t k = lo + t;
    const bool ok = okc && k < hi;
    const auto e = Op::load(x, k, g.r, ok);
    typename Op::El tmp;
    const bool good = Op::combine(g, acc, e, tmp);
    bad |= ok && !good;
    acc = Op::select(ok, tmp, acc);
  }
  if (okc && g.r == 0 && bad) raise_error(err, lo, kErrSingular);
  Op::store(agg, c, g.r, okc, acc);
}

// Downsweep: out[k] = carry ⊗ x[lo] ⊗ .. ⊗ x[k] (forward) or
// x[k] ⊗ .. ⊗ x[hi-1] ⊗ carry (reverse); carry from the scanned aggregates.
template <int D, class Op, bool kReverse>
__global__ void __launch_bounds__(kThreads) k_scan_down(typename Op::Arr x, int64_t n, int L,
                                                        typename Op::Arr aggs, int64_t nchunks,
                                                        typename Op::Arr out, DevError* err) {
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t c = group_index<D>(g);
  const int64_t lo = c * L;
  const int64_t hi = min(n, lo + L);
  const bool okc = g.real() && lo < n;
  const int64_t carry_idx = kReverse ? c + 1 : c - 1;
  bool have = okc && carry_idx >= 0 && carry_idx < nchunks;
  auto acc = Op::load(aggs, carry_idx, g.r, have);
  bool bad = false;
  for (int t = 0; t < L; ++t) {
    const int64_t k = kReverse ? lo + (L - 1 - t) : lo + t;
    const bool ok = okc && k < hi;
    const auto e = Op::load(x, k, g.r, ok);
    typename Op::El tmp;
    const bool good = kReverse ? Op::combine(g, e, acc, tmp) : Op::combine(g, acc, e, tmp);
    bad |= ok && have && !good;
    acc = Op::select(ok, Op::select(have, tmp, e), acc);
    have = have || ok;
    Op::store(out, k, g.r, ok, acc);
  }
  if (okc && g.r == 0 && bad) raise_error(err, lo, kErrSingular);
}

// The aggregate-scan kernels are latency-bound per group: cap them at 168
// registers (3 blocks of 4 warps per SM; measured 1 / 3 / 4: 3 is best, 4
// spills the block scan).
#ifndef PODE_GROUP_MIN_BLOCKS
#define PODE_GROUP_MIN_BLOCKS 3
#endif
constexpr int kGroupMinBlocks = PODE_GROUP_MIN_BLOCKS;

// --------------------------------------------- Gaussian-carry ⊗_f scan ---
// Reduce that also keeps every chunk-local inclusive prefix (loc), so the
// down-sweep is ONE combine deep: out[k] = carry ⊗ loc[k], independent k.
template <int D>
__global__ void __launch_bounds__(kThreads, kGroupMinBlocks) k_scan_reduce_loc(FEd x, int64_t n, int L, FEd loc, FEd agg,
                                                              DevError* err) {
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t c = group_index<D>(g);
  const int64_t lo = c * L;
  const int64_t hi = min(n, lo + L);
  const bool okc = g.real() && lo < n;
  FEl<D> acc = FOps<D>::load(x, lo, g.r, okc);
  FOps<D>::store(loc, lo, g.r, okc, acc);
  bool bad = false;
  for (int t = 1; t < L; ++t) {
    const int64_t k = lo + t;
    const bool ok = okc && k < hi;
    const FEl<D> e = FOps<D>::load(x, k, g.r, ok);
    FEl<D> tmp;
    // IEKS aggregates carry lower-triangular C and J (tria outputs)
    const bool good = combine_filtering<D, true>(g, acc, e, tmp);
    bad |= ok && !good;
    acc = FOps<D>::select(ok, tmp, acc);
    FOps<D>::store(loc, k, g.r, ok, acc);
  }
  if (okc && g.r == 0 && bad) raise_error(err, lo, kErrSingular);
  FOps<D>::store(agg, c, g.r, okc, acc);
}

// out[k] (b, C only) = carry[k / L - 1] ⊗ loc[k]; chunk 0 copies loc, or
// (fc: a time-axis shard's incoming Gaussian, b then C) is fc ⊗ loc[k].
template <int D>
__global__ void __launch_bounds__(kThreads, kGroupMinBlocks) k_scan_down_gauss(FEd loc, int64_t n, int L, FEd carry, FEd out,
                                                              DevError* err, const double* fc = nullptr) {
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t k = group_index<D>(g);
  const bool ok = g.real() && k < n;
  const int64_t c = k / L;
  const bool first = c == 0;
  const bool copy = first && fc == nullptr;  // block-uniform
  const FEl<D> e = FOps<D>::load(loc, k, g.r, ok);
  double bi;
  Rw<D> ci;
  if (first) {
    bi = (ok && fc) ? fc[g.r] : 0.0;
    ci = ld_row<D>(fc ? fc + D : nullptr, 0, g.r, ok && fc);
  } else {
    bi = ld_ent<D>(carry.b, c - 1, g.r, ok);
    ci = ld_row<D>(carry.c, c - 1, g.r, ok);
  }
  double bo;
  Rw<D> co;
  const bool good = combine_gauss<D>(g, bi, ci, e, bo, co);
  if (ok && !copy && g.r == 0 && !good) raise_error(err, k, kErrSingular);
  st_ent<D>(out.b, k, g.r, ok, copy ? e.b : bo);
  st_row<D>(out.c, k, g.r, ok, copy ? e.c : co);
}

// ------------------------------------- reverse mean-only scan (E = 0 tail) ---
// Chunk-local suffixes loc[k] = e_k ⊗ .. ⊗ e_{hi-1} (⊗_s on (E, g)) and the
// chunk aggregate; the sequence ends in the terminal element (E = 0), so
// every global suffix is a Gaussian mean and the down-sweep is one matvec.
template <int D>
__global__ void __launch_bounds__(kThreads) k_mscan_reduce_loc(SEd x, int64_t n, int L, SEd loc, SEd agg) {
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t c = group_index<D>(g);
  const int64_t lo = c * L;
  const int64_t hi = min(n, lo + L);
  const bool okc = g.real() && lo < n;
  typename MOps<D>::El acc = MOps<D>::load(x, hi - 1, g.r, okc);
  MOps<D>::store(loc, hi - 1, g.r, okc, acc);
  for (int t = 1; t < L; ++t) {
    const int64_t k = hi - 1 - t;
    const bool ok = okc && k >= lo;
    const typename MOps<D>::El e = MOps<D>::load(x, k, g.r, ok);
    typename MOps<D>::El tmp;
    MOps<D>::combine(g, e, acc, tmp);
    acc = MOps<D>::select(ok, tmp, acc);
    MOps<D>::store(loc, k, g.r, ok, acc);
  }
  MOps<D>::store(agg, c, g.r, okc, acc);
}

// out.g[k] = loc[k] ⊗ (0, g_carry) = E_loc g_carry + g_loc, carry = the
// suffix of the next chunk (the last chunk copies loc).
// rc (a time-axis shard's smoothed mean at its right halo node): the last
// chunk is E_loc rc + g_loc instead of a copy.
template <int D>
__global__ void __launch_bounds__(kThreads) k_mscan_down(SEd loc, int64_t n, int L, int64_t nchunks, SEd carry,
                                                         SEd out, const double* rc = nullptr) {
  extern __shared__ double smem[];
  const Grp<D> g = make_group<D>(smem);
  const int64_t k = group_index<D>(g);
  const bool ok = g.real() && k < n;
  const int64_t c = k / L;
  const bool last = c >= nchunks - 1;
  const typename MOps<D>::El e = MOps<D>::load(loc, k, g.r, ok);
  const double gc = last ? ((ok && rc) ? rc[g.r] : 0.0) : ld_ent<D>(carry.g, c + 1, g.r, ok);
  const double go = matvec(g, e.e, gc) + e.g;
  st_ent<D>(out.g, k, g.r, ok, (last && rc == nullptr) ? e.g : go);
}

// IEKS chunk aggregates: C and J are tria outputs (lower triangular).
template <int D>
struct FTOps : FOps<D> {
  __device__ static bool combine(const Grp<D>& g, const FEl<D>& l, const FEl<D>& rr, FEl<D>& out) {
    return combine_filtering<D, true>(g, l, rr, out);
  }
};

}  // namespace pode
#include "wide.cuh"  // wide groups (2D lanes per element) for the latency-bound upper scan levels
namespace pode {

// ---------------------------------------- block (Sklansky) local scans ---
// The upper levels of the aggregate scans are latency-bound chains of
// combines.  Here one CTA of kBWarps warps scans G = kBWarps * (32 / D)
// consecutive elements with the Sklansky tree: log2(G) combine steps (every
// group of a warp steps together, so the shuffles inside the combine stay
// warp-uniform), elements exchanged through shared memory.  Produces the
// block-local inclusive prefixes (suffixes when kRev) in loc and the block
// aggregate in agg[blockIdx.x] — the same contract as k_scan_reduce_loc with
// chunk length G, so the one-combine-deep down-sweeps are unchanged.
constexpr int kBWarps = 8;
static_assert((kBWarps & (kBWarps - 1)) == 0, "k_bscan_loc puts the warp index in the low position bits");

template <int D>
constexpr int bscan_groups() {
  return kBWarps * Grp<D>::kPerWarp;
}
template <int D, class Op>
constexpr size_t bscan_smem() {
  return sizeof(double) *
         (size_t(kBWarps) * Grp<D>::kSlots * Scratch<D>::kDoubles + size_t(bscan_groups<D>()) * Op::kDoubles);
}

template <int D, class Op, bool kRev>
__global__ void __launch_bounds__(kBWarps * 32, kGroupMinBlocks / 2) k_bscan_loc(typename Op::Arr x, int64_t n, typename Op::Arr loc,
                                                            typename Op::Arr agg, DevError* err) {
  extern __shared__ double smem[];
  constexpr int G = bscan_groups<D>();
  const Grp<D> g = make_group<D>(smem);
  const typename Op::Arr sb = Op::smem_arr(smem + kBWarps * Grp<D>::kSlots * Scratch<D>::kDoubles, G);
  // position in the block, warp index in the low bits: the Sklansky steps
  // h < kBWarps then split readers / idle groups along whole warps, and an
  // idle warp skips its combine
  const int warp = threadIdx.x >> 5;
  const int p = g.gw * kBWarps + warp;
  const bool real = g.real();
  const int64_t lo = int64_t(blockIdx.x) * G;
  const int64_t hi = min(n, lo + G);
  const int cnt = int(hi - lo);
  const bool ok = real && p < cnt;
  const int64_t k = kRev ? hi - 1 - p : lo + p;
  auto acc = Op::load(x, k, g.r, ok);
  bool bad = false;
#pragma unroll 1
  for (int h = 1; h < cnt; h <<= 1) {  // cnt is block-uniform
    // slot j is written once: at the step h = 2^(trailing ones of j)
    if (real && (p & (2 * h - 1)) == h - 1) Op::store(sb, p, g.r, true, acc);
    __syncthreads();
    const bool rd = real && (p & h);
    if (h >= kBWarps || (warp & h)) {  // warp-uniform
      const int j = (p & ~(2 * h - 1)) + h - 1;
      const auto left = Op::load(sb, rd ? j : 0, g.r, rd);
      typename Op::El tmp;
      const bool good = kRev ? Op::combine(g, acc, left, tmp) : Op::combine(g, left, acc, tmp);
      bad |= rd && ok && !good;
      acc = Op::select(rd, tmp, acc);
    }
  }
  Op::store(loc, k, g.r, ok, acc);
  if (ok && p == cnt - 1) Op::store(agg, blockIdx.x, g.r, true, acc);
  if (ok && g.r == 0 && bad) raise_error(err, k, kErrSingular);
}

// The block scan needs its tiles and G elements in shared memory (<= 227 KB
// per CTA): large D (e.g. 15) keeps the fan-in levels throughout.
template <int D, class Op>
constexpr bool bscan_fits() {
  return bscan_smem<D, Op>() <= size_t(227) * 1024;
}

// Scan levels above 0 with at most this many elements use the block kernel
// (latency-bound: Sklansky depth); larger levels keep the work-efficient
// sequential fan-in (throughput-bound).  PODE_BSCAN=0 disables, =n sets it.
// Upper ⊗_f scan levels on wide groups (wide.cuh) when PODE_WIDE=1.  Off by
// default: per iteration at N = 2^20 (tools/prof_events.py, block-scan time)
// it is neutral at D = 2 / 6 (-1 / -3 %), slower at D = 8 (+8 %) and faster
// only where the scan is a small share of the iteration (D = 4: -15 %,
// D = 9: -17 %, D = 12: -40 %; whole iterations within 0.6 %).  The per-pivot
// broadcast of the 2D-wide pivot row and its redundant reflector — not the
// row updates that the wide layout halves — set the combine's latency.
inline bool bscan_wide() {
  const char* env = std::getenv("PODE_WIDE");
  return env != nullptr && *env != '\0' && std::atoi(env) == 1;
}

inline int64_t bscan_max() {
  const char* env = std::getenv("PODE_BSCAN");
  if (env == nullptr || *env == '\0') return 16384;  // tools/knob_sweep.py (ms per iteration)
  const long long v = std::atoll(env);
  return v == 1 ? (int64_t(1) << 62) : int64_t(v);
}

// ------------------------------------------------------------- engine ---
template <int D>
struct Engine {
  // Chunk length per recursion level: level 0 fills the GPU; upper levels are
  // latency-bound (each group runs L dependent combines), so they use short
  // chunks and more levels.
  static int chunk_len(pode_context* ctx, int64_t n, int level) {
    const int64_t target = int64_t(ctx->sm_count) * 16 * Grp<D>::kPerWarp;
    int64_t L = (n + target - 1) / target;
    const int lmin = level == 0 ? 4 : 4;
    L = std::max<int64_t>(L, lmin);
    return static_cast<int>(std::min<int64_t>(L, 256));
  }

  template <class Op>
  static typename Op::Arr alloc(pode_context* ctx, const std::string& tag, int64_t n);

  template <class Op, bool kReverse>
  static void scan_rec(pode_context* ctx, typename Op::Arr in, typename Op::Arr out, int64_t n, int level,
                       ScanTally& t) {
    const int L = chunk_len(ctx, n, level);
    DevError* err = reinterpret_cast<DevError*>(ctx->d_err);
    if (n <= L) {
      k_scan_down<D, Op, kReverse><<<1, kThreads, smem_bytes<D>(), ctx->stream>>>(in, n, static_cast<int>(n),
                                                                                   in, 0, out, err);
      note_launch(ctx, Op::kDown);
      t.combines += n - 1;
      t.depth += n - 1;
      return;
    }
    const int64_t nc = (n + L - 1) / L;
    typename Op::Arr agg = alloc<Op>(ctx, "scan_agg_" + std::to_string(level), nc);
    k_scan_reduce<D, Op><<<blocks_for<D>(nc), kThreads, smem_bytes<D>(), ctx->stream>>>(in, n, L, agg, err);
    note_launch(ctx, Op::kReduce);
    t.combines += n - nc;
    t.depth += L - 1;
    scan_rec<Op, kReverse>(ctx, agg, agg, nc, level + 1, t);
    k_scan_down<D, Op, kReverse><<<blocks_for<D>(nc), kThreads, smem_bytes<D>(), ctx->stream>>>(in, n, L, agg,
                                                                                                nc, out, err);
    note_launch(ctx, Op::kDown);
    t.combines += n - 1;
    t.depth += L;
  }

  static void set_smem() {
    static OncePerDevice once;
    once([] { set_smem_now(); });
  }
  static void set_smem_now() {
    const int bytes = static_cast<int>(smem_bytes<D>());
    cudaFuncSetAttribute(k_combine<D, FOps<D>>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_combine<D, SOps<D>>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_make_filtering<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_make_smoothing<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_scan_reduce<D, FOps<D>>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_scan_reduce<D, SOps<D>>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_scan_down<D, FOps<D>, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_scan_down<D, FOps<D>, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_scan_down<D, SOps<D>, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_scan_down<D, SOps<D>, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_scan_reduce<D, MOps<D>>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_scan_down<D, MOps<D>, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_combine<D, MOps<D>>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  }

  // In-order total x[0] ⊗ .. ⊗ x[n-1] (fan-in-4 reduce tree, any Op); the
  // result is element 0 of the returned array.
  template <class Op>
  static typename Op::Arr reduce_total(pode_context* ctx, typename Op::Arr x, int64_t n, const std::string& tag) {
    set_smem();
    DevError* err = reinterpret_cast<DevError*>(ctx->d_err);
    int level = 0;
    while (n > 1) {
      const int L = 4;
      const int64_t nb = (n + L - 1) / L;
      typename Op::Arr agg = alloc<Op>(ctx, tag + std::to_string(level++), nb);
      k_scan_reduce<D, Op><<<blocks_for<D>(nb), kThreads, smem_bytes<D>(), ctx->stream>>>(x, n, L, agg, err);
      note_launch(ctx, Op::kReduce);
      x = agg;
      n = nb;
    }
    return x;
  }

  // out[0] = l[0] ⊗ r[0] (one element).
  template <class Op>
  static void combine_one(pode_context* ctx, typename Op::Arr l, typename Op::Arr r, typename Op::Arr o) {
    set_smem();
    k_combine<D, Op><<<1, kThreads, smem_bytes<D>(), ctx->stream>>>(1, l, r, o,
                                                                    reinterpret_cast<DevError*>(ctx->d_err));
    note_launch(ctx, "combine");
  }

  // Inclusive ⊗_f scan of a sequence whose first element is Gaussian
  // (A = eta = J = 0): every prefix is Gaussian, so only its (b, C) are
  // produced (into out.b / out.c).  k-ary tree with local prefixes: depth
  // (L-1) full combines per level up, ONE Gaussian-carry combine per level
  // down.
  // top(full, n): called once at the top level with its n full inclusive
  // prefixes (a time-axis shard reads its local total there and sets the
  // incoming carry fc before the down-sweeps run).
  using TopHook = std::function<void(FEd full, int64_t n)>;
  static void scan_gauss_rec(pode_context* ctx, FEd in, FEd out, int64_t n, int level, int L, ScanTally& t,
                             const TopHook* hook = nullptr, const double* fc = nullptr) {
    DevError* err = reinterpret_cast<DevError*>(ctx->d_err);
    size_t sm = smem_bytes<D>();
    FEd loc = alloc<FOps<D>>(ctx, "gscan_loc_" + std::to_string(level), n);
    if constexpr (2 * D <= 32 && bscan_smem_w<D>() <= size_t(227) * 1024) {
      if (level >= 1 && n <= bscan_max() && bscan_wide()) {  // block Sklansky levels, wide groups
        constexpr int G = bscan_groups_w<D>();
        sm = bscan_smem_w<D>();
        static OncePerDevice once;
        once([&] {
          cuda_check(cudaFuncSetAttribute(k_bscan_loc_w<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)),
                     "bscan smem");
        });
        const int64_t nb = (n + G - 1) / G;
        FEd agg = alloc<FOps<D>>(ctx, "gscan_agg_" + std::to_string(level), nb);
        k_bscan_loc_w<D><<<unsigned(nb), kBWarpsW * 32, sm, ctx->stream>>>(in, n, nb == 1 ? out : loc, agg, err);
        note_launch(ctx, "bscan_g");
        int depth = 0;
        while ((1 << depth) < std::min<int64_t>(n, G)) ++depth;
        t.depth += depth;
        t.combines += n * depth;
        if (nb == 1) {
          top_fix(ctx, out, out, n, hook, fc);
          return;
        }
        scan_gauss_rec(ctx, agg, agg, nb, level + 1, L, t, hook, fc);
        k_scan_down_gauss<D><<<blocks_for<D>(n), kThreads, smem_bytes<D>(), ctx->stream>>>(loc, n, G, agg, out, err,
                                                                                            fc);
        note_launch(ctx, "scan_g_down");
        t.combines += n - std::min<int64_t>(n, G);
        t.depth += 1;
        return;
      }
    }
    if (level >= 1 && n <= bscan_max() && bscan_fits<D, FOps<D>>()) {  // block Sklansky levels
      constexpr int G = bscan_groups<D>();
      sm = bscan_smem<D, FOps<D>>();
      static OncePerDevice once;
      once([&] {
        cuda_check(cudaFuncSetAttribute(k_bscan_loc<D, FTOps<D>, false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)),
                   "bscan smem");
      });
      const int64_t nb = (n + G - 1) / G;
      FEd agg = alloc<FOps<D>>(ctx, "gscan_agg_" + std::to_string(level), nb);
      k_bscan_loc<D, FTOps<D>, false><<<unsigned(nb), kBWarps * 32, sm, ctx->stream>>>(in, n, nb == 1 ? out : loc,
                                                                                     agg, err);
      note_launch(ctx, "bscan_g");
      int depth = 0;
      while ((1 << depth) < std::min<int64_t>(n, G)) ++depth;
      t.depth += depth;
      t.combines += n * depth;
      if (nb == 1) {
        top_fix(ctx, out, out, n, hook, fc);
        return;
      }
      scan_gauss_rec(ctx, agg, agg, nb, level + 1, L, t, hook, fc);
      k_scan_down_gauss<D><<<blocks_for<D>(n), kThreads, smem_bytes<D>(), ctx->stream>>>(loc, n, G, agg, out, err,
                                                                                          fc);
      note_launch(ctx, "scan_g_down");
      t.combines += n - std::min<int64_t>(n, G);
      t.depth += 1;
      return;
    }
    if (n <= L) {
      // the single chunk's aggregate goes to a scratch slot: loc[0] must stay
      // the first element's own prefix
      FEd top = alloc<FOps<D>>(ctx, "gscan_top", 1);
      k_scan_reduce_loc<D><<<1, kThreads, sm, ctx->stream>>>(in, n, static_cast<int>(n), loc, top, err);
      note_launch(ctx, "scan_g_reduce");
      t.combines += n - 1;
      t.depth += n - 1;
      if (hook != nullptr) {
        top_fix(ctx, loc, out, n, hook, fc);
        return;
      }
      cuda_check(cudaMemcpyAsync(out.b, loc.b, sizeof(double) * D * n, cudaMemcpyDeviceToDevice, ctx->stream),
                 "gscan copy");
      cuda_check(cudaMemcpyAsync(out.c, loc.c, sizeof(double) * D * D * n, cudaMemcpyDeviceToDevice, ctx->stream),
                 "gscan copy");
      return;
    }
    const int64_t nc = (n + L - 1) / L;
    FEd agg = alloc<FOps<D>>(ctx, "gscan_agg_" + std::to_string(level), nc);
    k_scan_reduce_loc<D><<<blocks_for<D>(nc), kThreads, sm, ctx->stream>>>(in, n, L, loc, agg, err);
    note_launch(ctx, "scan_g_reduce");
    t.combines += n - nc;
    t.depth += L - 1;
    scan_gauss_rec(ctx, agg, agg, nc, level + 1, L, t, hook, fc);
    k_scan_down_gauss<D><<<blocks_for<D>(n), kThreads, sm, ctx->stream>>>(loc, n, L, agg, out, err, fc);
    note_launch(ctx, "scan_g_down");
    t.combines += n - std::min<int64_t>(n, L);
    t.depth += 1;
  }

  // Top of a hooked scan: the hook sees the full prefixes, then (shard
  // carry fc) every top prefix becomes fc ⊗ prefix (b, C into out).
  static void top_fix(pode_context* ctx, FEd full, FEd out, int64_t n, const TopHook* top, const double* fc) {
    if (top == nullptr) return;
    (*top)(full, n);
    if (fc == nullptr && full.b == out.b) return;
    k_scan_down_gauss<D><<<blocks_for<D>(n), kThreads, smem_bytes<D>(), ctx->stream>>>(
        full, n, static_cast<int>(n), full, out, reinterpret_cast<DevError*>(ctx->d_err), fc);
    note_launch(ctx, "scan_g_top");
  }

  // The Gaussian-carry scan of a time-axis shard whose first element is not
  // Gaussian: the up-sweep's top total goes to `top` (the exchange), which
  // writes the incoming carry to fc (b then C; nullptr on the first shard:
  // its first element absorbed the prior); the down-sweeps then apply fc to
  // the first block of every level.  Same depth as the single-device scan,
  // no separate reduction of the aggregates.
  static ScanTally scan_filtering_gauss_shard(pode_context* ctx, int64_t n, FEd io, int L, const TopHook& top,
                                              const double* fc) {
    set_gauss_attrs();
    ScanTally t;
    if (n >= 1) scan_gauss_rec(ctx, io, io, n, 0, L, t, &top, fc);
    return t;
  }

  static void set_gauss_attrs() {
    set_smem();
    static OncePerDevice once;
    once([&] {
      const int bytes = static_cast<int>(smem_bytes<D>());
      cudaFuncSetAttribute(k_scan_reduce_loc<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      cudaFuncSetAttribute(k_scan_down_gauss<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    });
  }

  static ScanTally scan_filtering_gauss(pode_context* ctx, int64_t n, FEd in, FEd out, int L) {
    set_gauss_attrs();
    ScanTally t;
    if (n >= 1) scan_gauss_rec(ctx, in, out, n, 0, L, t);
    return t;
  }

  // Reverse inclusive scan of mean-only elements ending in the terminal
  // element (E = 0): only the suffix means (out.g) are produced.
  // hook(full, n): called at the top level with its n full suffixes (a
  // time-axis shard reads its local total, element 0, and writes its right
  // carry rc before the down-sweeps run).
  using MTopHook = std::function<void(SEd full, int64_t n)>;
  static void mscan_top_fix(pode_context* ctx, SEd full, SEd out, int64_t n, const MTopHook* hook, const double* rc) {
    if (hook == nullptr) return;
    (*hook)(full, n);
    if (rc == nullptr && full.g == out.g) return;
    k_mscan_down<D><<<blocks_for<D>(n), kThreads, smem_bytes<D>(), ctx->stream>>>(full, n, static_cast<int>(n), 1,
                                                                                  full, out, rc);
    note_launch(ctx, "scan_m_top");
  }
  static void mscan_rec(pode_context* ctx, SEd in, SEd out, int64_t n, int level, int L, ScanTally& t,
                        const MTopHook* hook = nullptr, const double* rc = nullptr) {
    size_t sm = smem_bytes<D>();
    SEd loc = alloc<SOps<D>>(ctx, "mscan_loc_" + std::to_string(level), n);
    if (level >= 1 && n <= bscan_max() && bscan_fits<D, MOps<D>>()) {  // block Sklansky levels
      constexpr int G = bscan_groups<D>();
      sm = bscan_smem<D, MOps<D>>();
      static OncePerDevice once;
      once([&] {
        cuda_check(cudaFuncSetAttribute(k_bscan_loc<D, MOps<D>, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(sm)),
                   "bscan smem");
      });
      const int64_t nb = (n + G - 1) / G;
      SEd agg = alloc<SOps<D>>(ctx, "mscan_agg_" + std::to_string(level), nb);
      k_bscan_loc<D, MOps<D>, true><<<unsigned(nb), kBWarps * 32, sm, ctx->stream>>>(in, n, nb == 1 ? out : loc,
                                                                                    agg, nullptr);
      note_launch(ctx, "bscan_m");
      int depth = 0;
      while ((1 << depth) < std::min<int64_t>(n, G)) ++depth;
      t.depth += depth;
      t.combines += n * depth;
      if (nb == 1) {
        mscan_top_fix(ctx, out, out, n, hook, rc);
        return;
      }
      mscan_rec(ctx, agg, agg, nb, level + 1, L, t, hook, rc);
      k_mscan_down<D><<<blocks_for<D>(n), kThreads, smem_bytes<D>(), ctx->stream>>>(loc, n, G, nb, agg, out, rc);
      note_launch(ctx, "scan_m_down");
      t.combines += n - std::min<int64_t>(n, G);
      t.depth += 1;
      return;
    }
    if (n <= L) {
      k_mscan_reduce_loc<D><<<1, kThreads, sm, ctx->stream>>>(in, n, static_cast<int>(n), loc, loc);
      note_launch(ctx, "scan_m_reduce");
      t.combines += n - 1;
      t.depth += n - 1;
      if (hook != nullptr) {
        mscan_top_fix(ctx, loc, out, n, hook, rc);
        return;
      }
      cuda_check(cudaMemcpyAsync(out.g, loc.g, sizeof(double) * D * n, cudaMemcpyDeviceToDevice, ctx->stream),
                 "mscan copy");
      return;
    }
    const int64_t nc = (n + L - 1) / L;
    SEd agg = alloc<SOps<D>>(ctx, "mscan_agg_" + std::to_string(level), nc);
    k_mscan_reduce_loc<D><<<blocks_for<D>(nc), kThreads, sm, ctx->stream>>>(in, n, L, loc, agg);
    note_launch(ctx, "scan_m_reduce");
    t.combines += n - nc;
    t.depth += L - 1;
    mscan_rec(ctx, agg, agg, nc, level + 1, L, t, hook, rc);
    k_mscan_down<D><<<blocks_for<D>(n), kThreads, sm, ctx->stream>>>(loc, n, L, nc, agg, out, rc);
    note_launch(ctx, "scan_m_down");
    t.combines += n - std::min<int64_t>(n, L);
    t.depth += 1;
  }

  static void set_mscan_attrs() {
    static OncePerDevice once;
    once([&] {
      const int bytes = static_cast<int>(smem_bytes<D>());
      cudaFuncSetAttribute(k_mscan_reduce_loc<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      cudaFuncSetAttribute(k_mscan_down<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    });
  }
  static ScanTally scan_means_terminal(pode_context* ctx, int64_t n, SEd io, int L) {
    set_mscan_attrs();
    ScanTally t;
    if (n >= 1) mscan_rec(ctx, io, io, n, 0, L, t);
    return t;
  }
  // A time-axis shard's mean scan: its last chunk does not hold the terminal
  // element; `hook` gets the local total at the top (the exchange) and writes
  // the right carry rc (nullptr on the last shard), which the down-sweeps
  // apply to the last block of every level.
  static ScanTally scan_means_terminal_shard(pode_context* ctx, int64_t n, SEd io, int L, const MTopHook& hook,
                                             const double* rc) {
    set_mscan_attrs();
    ScanTally t;
    if (n >= 1) mscan_rec(ctx, io, io, n, 0, L, t, &hook, rc);
    return t;
  }

  // Reverse inclusive scan of mean-only smoothing elements.
  static ScanTally scan_means_reverse(pode_context* ctx, int64_t n, SEd io) {
    set_smem();
    ScanTally t;
    if (n >= 1) scan_rec<MOps<D>, true>(ctx, io, io, n, 0, t);
    return t;
  }

  static void combine_filtering(pode_context* ctx, int64_t count, FEd l, FEd r, FEd o) {
    set_smem();
    k_combine<D, FOps<D>><<<blocks_for<D>(count), kThreads, smem_bytes<D>(), ctx->stream>>>(
        count, l, r, o, reinterpret_cast<DevError*>(ctx->d_err));
    note_launch(ctx, "combine_filtering");
  }
  static void combine_smoothing(pode_context* ctx, int64_t count, SEd l, SEd r, SEd o) {
    set_smem();
    k_combine<D, SOps<D>><<<blocks_for<D>(count), kThreads, smem_bytes<D>(), ctx->stream>>>(
        count, l, r, o, reinterpret_cast<DevError*>(ctx->d_err));
    note_launch(ctx, "combine_smoothing");
  }
  static void make_filtering(pode_context* ctx, const DevChain& ch, int absorb, FEd out) {
    set_smem();
    k_make_filtering<D><<<blocks_for<D>(ch.N), kThreads, smem_bytes<D>(), ctx->stream>>>(
        ch, absorb, out, reinterpret_cast<DevError*>(ctx->d_err));
    note_launch(ctx, "make_filtering");
  }
  static void make_smoothing(pode_context* ctx, const DevChain& ch, const double* fm, const double* fc,
                             SEd out) {
    set_smem();
    k_make_smoothing<D><<<blocks_for<D>(ch.N + 1), kThreads, smem_bytes<D>(), ctx->stream>>>(
        ch, fm, fc, out, reinterpret_cast<DevError*>(ctx->d_err));
    note_launch(ctx, "make_smoothing");
  }
  static ScanTally scan_filtering(pode_context* ctx, int64_t n, FEd in, FEd out, bool reverse) {
    set_smem();
    ScanTally t;
    if (n < 1) return t;
    if (reverse)
      scan_rec<FOps<D>, true>(ctx, in, out, n, 0, t);
    else
      scan_rec<FOps<D>, false>(ctx, in, out, n, 0, t);
    return t;
  }
  static ScanTally scan_smoothing(pode_context* ctx, int64_t n, SEd in, SEd out, bool reverse) {
    set_smem();
    ScanTally t;
    if (n < 1) return t;
    if (reverse)
      scan_rec<SOps<D>, true>(ctx, in, out, n, 0, t);
    else
      scan_rec<SOps<D>, false>(ctx, in, out, n, 0, t);
    return t;
  }

  // para_rts (parallel.cpp:166-209) on device buffers.
  static ScanTally rts(pode_context* ctx, const DevChain& ch, double* fmean, double* fcov, double* smean,
                       double* scov) {
    const int64_t N = ch.N;
    FEd fe = alloc<FOps<D>>(ctx, "rts_fe", N);
    make_filtering(ctx, ch, 1, fe);
    ScanTally tf = scan_filtering(ctx, N, fe, fe, false);
    // filtered[0] = init, filtered[n+1] = (b_n, C_n)
    cuda_check(cudaMemcpyAsync(fmean, ch.init_mean, sizeof(double) * D, cudaMemcpyDeviceToDevice, ctx->stream),
               "copy init");
    cuda_check(cudaMemcpyAsync(fcov, ch.init_cov, sizeof(double) * D * D, cudaMemcpyDeviceToDevice, ctx->stream),
               "copy init");
    cuda_check(cudaMemcpyAsync(fmean + D, fe.b, sizeof(double) * D * N, cudaMemcpyDeviceToDevice, ctx->stream),
               "copy filtered");
    cuda_check(cudaMemcpyAsync(fcov + D * D, fe.c, sizeof(double) * D * D * N, cudaMemcpyDeviceToDevice,
                               ctx->stream),
               "copy filtered");
    SEd se = alloc<SOps<D>>(ctx, "rts_se", N + 1);
    make_smoothing(ctx, ch, fmean, fcov, se);
    ScanTally ts = scan_smoothing(ctx, N + 1, se, se, true);
    if (smean)
      cuda_check(cudaMemcpyAsync(smean, se.g, sizeof(double) * D * (N + 1), cudaMemcpyDeviceToDevice,
                                 ctx->stream),
                 "copy smoothed");
    if (scov)
      cuda_check(cudaMemcpyAsync(scov, se.l, sizeof(double) * D * D * (N + 1), cudaMemcpyDeviceToDevice,
                                 ctx->stream),
                 "copy smoothed");
    ScanTally out;
    out.combines = std::max(tf.combines, ts.combines);
    out.depth = std::max(tf.depth, ts.depth);
    return out;
  }
};

template <int D>
template <class Op>
typename Op::Arr Engine<D>::alloc(pode_context* ctx, const std::string& tag, int64_t n) {
  if constexpr (std::is_same_v<Op, FOps<D>>) {
    FEd e;
    double* base = ctx->ws.arr<double>(tag, size_t(n) * (3 * D * D + 2 * D));
    e.a = base;
    e.c = e.a + n * D * D;
    e.j = e.c + n * D * D;
    e.b = e.j + n * D * D;
    e.eta = e.b + n * D;
    return e;
  } else {
    SEd e;
    double* base = ctx->ws.arr<double>(tag, size_t(n) * (2 * D * D + D));
    e.e = base;
    e.l = e.e + n * D * D;
    e.g = e.l + n * D * D;
    return e;
  }
}

}  // namespace pode
