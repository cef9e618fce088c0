// Shared argument blocks of the fused IEKS iteration (lane.cuh kernels,
// fast_driver.cuh host loop) for an ODE information operator, D = d (q+1).
//
// One Gauss-Newton iteration:
//   A  fold each chunk's filtering elements into one aggregate (A,b,C,eta,J),
//      EK1-linearising every step on the fly (statespace.cpp:65-88 at
//      eta[n+1], rescaled by T(h), ieks.cpp:160-164) — the element algebra of
//      make_filtering_element + ⊗_f (parallel.cpp:5-100);
//   B  scan of the chunk aggregates under ⊗_f (engine.cuh);
//   C  the square-root filter through each chunk from its incoming marginal,
//      forming the smoothing elements (E, g) (parallel.cpp:112-135);
//   C2/D  backward chunk aggregates and their reverse scan;
//   E  the backward mean recursion, the new trajectory, the objective
//      (ieks.cpp:49-60) and the stopping maxima (ieks.cpp:62-77).
// Covariances, innovation statistics and calibration are formed once after
// convergence (ieks.cpp:190-208, lane.cuh finalize kernels).
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
  // Graph-loop mode (it_dev != nullptr): the linearisation point is
  // pair[*it_dev & 1] (its node-N slot at + term_off), the new trajectory
  // goes to the other buffer, so one captured iteration serves every
  // iteration of the device-side loop.
  const int* it_dev;
  double* pair0;
  double* pair1;
  int64_t term_off;
  // Time-axis shard: local node 0 is global node g0 (grid
  // points at the global grid + g0).  first: this shard starts at global
  // node 0 (chunk 0 absorbs the initial distribution); otherwise chunk 0
  // starts from `carry` = the filtered (b, C) at local node 0 folded from the
  // preceding shards.  last: this shard ends at global node N (terminal
  // element, node N counted in the stopping maxima and written out).
  int first = 1;
  int last = 1;
  const double* carry = nullptr;  // D + D*D doubles
  // Batch of independent IVPs (pode_ieks_batch, the kBatch kernels): IVP b
  // owns chunks [b seg_chunks, (b+1) seg_chunks) of the chunk axis, the first
  // seg_real of them real (N steps each, a shared grid), the rest padding up
  // to whole lane blocks (identity aggregates, no output).  Every IVP's chunk
  // 0 absorbs its own initial distribution, so the unsegmented aggregate
  // scans restart at each IVP (a Gaussian element, A = 0, ignores its left
  // operand; the terminal backward element, E = 0, its right operand).
  int64_t seg_chunks = 0;
  int64_t seg_real = 0;
  const DevProblem* probs = nullptr;  // per IVP
  const double* m0s = nullptr;        // per IVP: T_0^-1 mu_0 (D)
  const int* active = nullptr;        // per IVP: still iterating (converged IVPs keep their buffers)
  const int* seg_it = nullptr;        // finalize: per-IVP iteration count (its buffer parity)
};

// Position of chunk c on its IVP (kBatch) or on the single time axis.
struct SegPos {
  int64_t seg;    // IVP
  int64_t cl;     // chunk index within the IVP
  int64_t nreal;  // real chunks of the IVP
};
template <bool kBatch>
__device__ __forceinline__ SegPos seg_pos(const FastArgs& a, int64_t c) {
  if constexpr (kBatch) {
    const int64_t b = c / a.seg_chunks;
    return SegPos{b, c - b * a.seg_chunks, a.seg_real};
  } else {
    return SegPos{0, c, a.nchunks};
  }
}

// The linearisation point of this iteration (its node-N slot in `term`).
// Kernels keep their FastArgs parameter unmodified, so it stays in the
// constant parameter bank (a written copy would be spilled to the stack).
struct LinPoint {
  const double* eta;
  const double* term;
};
__device__ __forceinline__ LinPoint lin_point(const FastArgs& a) {
  if (a.it_dev != nullptr) {  // graph-loop mode
    const double* b = (*a.it_dev & 1) ? a.pair1 : a.pair0;
    return LinPoint{b, b + a.term_off};
  }
  return LinPoint{a.eta, a.eta_term};
}
// Batch: IVP seg's linearisation point (its node-N slot: term + seg D).  After
// the loop (seg_it set) each IVP's own final point, pair[(it_b + 1) & 1].
template <int D, bool kBatch>
__device__ __forceinline__ LinPoint lin_point_seg(const FastArgs& a, int64_t seg) {
  if constexpr (!kBatch) {
    return lin_point(a);
  } else {
    int par;
    if (a.seg_it != nullptr)
      par = (a.seg_it[seg] + 1) & 1;
    else
      par = *a.it_dev & 1;
    const double* b = par ? a.pair1 : a.pair0;
    return LinPoint{b, b + a.term_off + seg * D};
  }
}

__device__ __forceinline__ double ipow(double h, int k) {
  if (k == 0) return 1.0;
  if (k == 1) return h;
  if (k == 2) return h * h;
  return pow(h, double(k));
}


// Node times for a backward loop over steps k = e-1 down to s: step(k)
// returns h_k = t_k - t_{k-1} (node 0 of the time axis, origin: t_1 - t_0)
// and issues the load of t_{k-2} one step ahead.  A shard's grid pointer is
// offset into the global grid, so t_{-1} is its left neighbour's node.
struct BwdGrid {
  const double* g;
  int origin;
  double tk, tkm;
  __device__ BwdGrid(const double* grid, int org, int64_t k) : g(grid), origin(org) {
    tk = grid[k];
    tkm = (k >= 1 || !org) ? grid[k - 1] : 0.0;
  }
  __device__ double step(int64_t k) {
    const double h = (k == 0 && origin) ? g[1] - g[0] : tk - tkm;
    tk = tkm;
    tkm = (k >= 2 || (k == 1 && !origin)) ? g[k - 2] : 0.0;
    return h;
  }
};

}  // namespace pode
