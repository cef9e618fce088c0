// Host driver of the fused IEKS iteration (lane.cuh passes + engine.cuh
// aggregate scans): per Gauss-Newton iteration five lane passes, two
// aggregate scans and one 3-scalar device->host read for the stopping rule
// (ieks.cpp:157-187).
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "fast.cuh"
#include "ieks.cuh"
#include "lane.cuh"
#include "lane_scan.cuh"

namespace pode {

namespace lane {

// eta (N+1 nodes, chunk-interleaved + node-N slot) <- mu0 at every node.
template <int D>
__global__ void k_eta_fill(const double* mu0, int64_t nc, int L, double* base) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t total = nc * L * D;
  if (i < total) base[i] = mu0[(i / nc) % D];
  if (i < D) base[total + i] = mu0[i];
}

// chunk-interleaved eta -> (N+1) x D row-major
template <int D>
__global__ void k_eta_rows(const double* base, const double* term, int64_t N, int L, int64_t nc, double* rows) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= (N + 1) * D) return;
  const int64_t k = i / D;
  const int r = int(i - k * D);
  rows[i] = eta_at<D>(base, term, k, r, N, L, nc);
}

}  // namespace lane

template <int D, int d>
struct FastEngine {
  // Chunk-aggregate scans: the group engine by default (its ⊗_f has the
  // shorter critical path); PODE_SCAN_MODE=lane selects the lane-serial one.
  static bool lane_scans() {
    const char* env = std::getenv("PODE_SCAN_MODE");
    return env != nullptr && std::string(env) == "lane";
  }
  static int scan_fanin() {
    const char* env = std::getenv("PODE_SCAN_FANIN");
    const int v = env ? std::atoi(env) : 4;
    return v >= 2 ? v : 4;
  }

  // One chunk per thread, ~256 resident threads per SM.
  static int chunk_len(pode_context* ctx, int64_t N) {
    const char* env = std::getenv("PODE_CHUNK");
    if (env) return std::max(2, std::atoi(env));
    const int64_t target = int64_t(ctx->sm_count) * 256;
    const int64_t L = (N + target - 1) / target;
    return static_cast<int>(std::max<int64_t>(8, std::min<int64_t>(L, 4096)));
  }

  static IeksResult run(pode_context* ctx, const host::Problem& p, const pode_prior& prior, const double* grid_h,
                        int64_t n1, const pode_ieks_config& cfg, double* means, double* cov, double* sol_m,
                        double* sol_c) {
    using IE = IeksEngine<D>;
    IeksSetup<D> s;
    IE::setup(ctx, p, prior, grid_h, n1, s);
    cudaStream_t st = ctx->stream;
    Workspace& ws = ctx->ws;
    const int64_t N = s.N;
    const int L = chunk_len(ctx, N);
    const int64_t nc = (N + L - 1) / L;
    FastConst<D> cst;
    std::memcpy(cst.q, s.h_q.data(), sizeof(cst.q));
    std::memcpy(cst.qunit, s.h_qunit.data(), sizeof(cst.qunit));
    std::memcpy(cst.qunit_rdiag, s.h_qinv.data(), sizeof(cst.qunit_rdiag));
    std::memcpy(cst.m0, s.h_m0.data(), sizeof(cst.m0));

    const size_t padded = size_t(nc) * L;
    const size_t eta_len = padded * D + D;
    double* eta_a = ws.arr<double>("lane_eta_a", eta_len);
    double* eta_b = ws.arr<double>("lane_eta_b", eta_len);
    FEd agg = Engine<D>::template alloc<FOps<D>>(ctx, "fast_agg", nc);
    lane::ElemSoA soa;
    {
      double* base = ws.arr<double>("fast_elems", padded * (D * D + D) + D);
      soa = lane::ElemSoA{base, base + padded * D * D, base + padded * (D * D + D), nc, L};
    }
    SEd bagg;
    {
      double* base = ws.arr<double>("fast_bagg", size_t(nc) * (D * D + D));
      bagg = SEd{base, base + size_t(nc) * D * D, nullptr};
    }
    const unsigned lblocks = static_cast<unsigned>((nc + lane::kLaneThreads - 1) / lane::kLaneThreads);
    const int64_t nparts = int64_t(lblocks);
    double* part = ws.arr<double>("fast_part", nparts * 3 + 3);
    double* red = part + nparts * 3;
    const unsigned th = lane::kLaneThreads;
    auto term = [&](double* base) { return base + padded * D; };
    FastArgs a{s.grid, eta_a, term(eta_a), N, L, nc, cfg.linearization, s.prob,
               reinterpret_cast<DevError*>(ctx->d_err)};

    lane::k_eta_fill<D><<<grid1(int64_t(padded) * D + D), kRedThreads, 0, st>>>(s.mu0, nc, L, eta_a);
    note_launch(ctx, "fill");
    auto finish = [&]() {
      k_finish3<<<1, kRedThreads, 0, st>>>(part, nparts, red);
      note_launch(ctx, "finish3");
      cuda_check(cudaMemcpyAsync(ctx->h_scalars, red, sizeof(double) * 3, cudaMemcpyDeviceToHost, st), "red");
    };
    // objective of the constant start (ieks.cpp:147-148)
    lane::k_lane_bwd_down<D, d, true><<<lblocks, th, 0, st>>>(a, cst, soa, bagg, eta_a, term(eta_a), eta_b,
                                                               term(eta_b), part);
    note_launch(ctx, "fast_objective");
    finish();
    cuda_check(cudaStreamSynchronize(st), "sync");
    prof_mark(ctx);
    double v_prev = 0.5 * ctx->h_scalars[0];

    IeksResult res;
    int it = 0;
    while (it < cfg.max_iterations) {
      ++it;
      reset_error(ctx);
      a.eta = eta_a;
      a.eta_term = term(eta_a);
      lane::k_lane_fwd_reduce<D, d><<<lblocks, th, 0, st>>>(a, cst, agg);
      note_launch(ctx, "fast_fwd_reduce");
      ScanTally tf, tr;
      if (lane_scans())
        lane::LaneScan<D, lane::LFOps<D>, false>::run(ctx, agg, agg, nc, 0, scan_fanin(), tf);
      else
        tf = Engine<D>::scan_filtering_gauss(ctx, nc, agg, agg, scan_fanin());
      lane::k_lane_fwd_down<D, d><<<lblocks, th, 0, st>>>(a, cst, agg, soa);
      note_launch(ctx, "fast_fwd_down");
      lane::k_lane_bfold<D><<<lblocks, th, 0, st>>>(soa, N, L, nc, bagg);
      note_launch(ctx, "fast_bwd_fold");
      if (lane_scans())
        lane::LaneScan<D, lane::LMOps<D>, true>::run(ctx, bagg, bagg, nc, 0, scan_fanin(), tr);
      else
        tr = Engine<D>::scan_means_terminal(ctx, nc, bagg, scan_fanin());
      lane::k_lane_bwd_down<D, d, false><<<lblocks, th, 0, st>>>(a, cst, soa, bagg, eta_a, term(eta_a), eta_b,
                                                                  term(eta_b), part);
      note_launch(ctx, "fast_bwd_down");
      finish();
      IE::check_linearization(ctx, s, it);  // syncs the stream
      // scan tally of the whole time axis: chunk folds + aggregate scans
      res.stats.combines = std::max(res.stats.combines, (N - nc) + tf.combines + N);
      res.stats.depth = std::max(res.stats.depth, int64_t(L) + tf.depth + int64_t(L) + tr.depth);
      const double v = 0.5 * ctx->h_scalars[0];
      const double dmax = ctx->h_scalars[1], emax = ctx->h_scalars[2];
      res.trace.push_back(v);
      const bool conv = (dmax <= cfg.traj_rtol * emax) ||
                        (std::fabs(v - v_prev) <= cfg.obj_atol + cfg.obj_rtol * std::fabs(v));
      std::swap(eta_a, eta_b);
      v_prev = v;
      if (conv) {
        res.converged = true;
        break;
      }
    }
    res.iterations = it;
    // row-major copies of the final linearisation point and trajectory
    double* lin_rows = ws.arr<double>("lane_lin_rows", size_t(n1) * D);
    double* out_rows = ws.arr<double>("lane_out_rows", size_t(n1) * D);
    lane::k_eta_rows<D><<<grid1(n1 * D), kRedThreads, 0, st>>>(eta_b, term(eta_b), N, L, nc, lin_rows);
    note_launch(ctx, "eta_rows");
    lane::k_eta_rows<D><<<grid1(n1 * D), kRedThreads, 0, st>>>(eta_a, term(eta_a), N, L, nc, out_rows);
    note_launch(ctx, "eta_rows");
    IE::finalize(ctx, s, lin_rows, out_rows, cfg.linearization, it, prior.sigma, means, cov, sol_m, sol_c, res);
    return res;
  }
};

}  // namespace pode
