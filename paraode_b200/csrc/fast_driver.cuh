// Host driver of the fused IEKS iteration (fast.cuh): five launches per
// Gauss-Newton iteration and one 3-scalar device->host read for the stopping
// rule (ieks.cpp:157-187).
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

template <int D, int d>
struct FastEngine {
  static void set_smem() {
    static bool done = false;
    if (done) return;
    done = true;
    const int bytes = static_cast<int>(smem_bytes<D>());
    cudaFuncSetAttribute(k_fast_fwd_reduce<D, d>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_fast_fwd_down<D, d>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_fast_bwd_down<D, d, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_fast_bwd_down<D, d, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  }

  static bool lane_mode() {
    const char* env = std::getenv("PODE_FAST_MODE");
    return !(env != nullptr && std::string(env) == "group");
  }
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

  // Chunk length: enough chunks to fill every SM with resident groups.
  static int chunk_len(pode_context* ctx, int64_t N) {
    if (lane_mode()) {  // one chunk per thread, ~256 resident threads per SM
      const int64_t target = int64_t(ctx->sm_count) * 256;
      const int64_t L = (N + target - 1) / target;
      return static_cast<int>(std::max<int64_t>(8, std::min<int64_t>(L, 4096)));
    }
    const int64_t target = int64_t(ctx->sm_count) * 16 * Grp<D>::kPerWarp;
    const int64_t L = (N + target - 1) / target;
    return static_cast<int>(std::max<int64_t>(4, std::min<int64_t>(L, 4096)));
  }

  static IeksResult run(pode_context* ctx, const host::Problem& p, const pode_prior& prior, const double* grid_h,
                        int64_t n1, const pode_ieks_config& cfg, double* means, double* cov, double* sol_m,
                        double* sol_c) {
    set_smem();
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
    FastArgs a{s.grid, nullptr, N, L, nc, cfg.linearization, s.prob, reinterpret_cast<DevError*>(ctx->d_err)};

    double* eta_a = ws.arr<double>("ieks_eta_a", n1 * D);
    double* eta_b = ws.arr<double>("ieks_eta_b", n1 * D);
    FEd agg = Engine<D>::template alloc<FOps<D>>(ctx, "fast_agg", nc);
    SEd elems;  // element-major (group passes)
    lane::ElemSoA soa;  // chunk-interleaved (lane passes)
    {
      const size_t padded = size_t(nc) * L;
      const size_t n_el = std::max<size_t>(size_t(n1), padded + 1);
      double* base = ws.arr<double>("fast_elems", n_el * (D * D + D) + D);
      elems = SEd{base, base + n_el * D * D, nullptr};
      soa = lane::ElemSoA{base, base + padded * D * D, base + n_el * (D * D + D), nc, L};
    }
    SEd bagg;
    {
      double* base = ws.arr<double>("fast_bagg", size_t(nc) * (D * D + D));
      bagg = SEd{base, base + size_t(nc) * D * D, nullptr};
    }
    const bool lanes = lane_mode();
    const unsigned lblocks = static_cast<unsigned>((nc + lane::kLaneThreads - 1) / lane::kLaneThreads);
    const int64_t nparts = lanes ? int64_t(lblocks) : nc;
    double* part = ws.arr<double>("fast_part", nparts * 3 + 3);
    double* red = part + nparts * 3;
    const unsigned blocks = blocks_for<D>(nc);
    const size_t sm = smem_bytes<D>();

    k_fill_rows<<<grid1(n1 * D), kRedThreads, 0, st>>>(s.mu0, n1, D, eta_a);
    note_launch(ctx, "fill");
    auto finish = [&]() {
      k_finish3<<<1, kRedThreads, 0, st>>>(part, nparts, red);
      note_launch(ctx, "finish3");
      cuda_check(cudaMemcpyAsync(ctx->h_scalars, red, sizeof(double) * 3, cudaMemcpyDeviceToHost, st), "red");
    };
    // objective of the constant start (ieks.cpp:147-148)
    a.eta = eta_a;
    if (lanes)
      lane::k_lane_bwd_down<D, d, true><<<lblocks, lane::kLaneThreads, 0, st>>>(a, cst, soa, bagg, eta_a, eta_b,
                                                                               part);
    else
      k_fast_bwd_down<D, d, true><<<blocks, kThreads, sm, st>>>(a, cst, elems, bagg, eta_a, eta_b, part);
    note_launch(ctx, "fast_objective");
    finish();
    cuda_check(cudaStreamSynchronize(st), "sync");
    double v_prev = 0.5 * ctx->h_scalars[0];

    IeksResult res;
    int it = 0;
    while (it < cfg.max_iterations) {
      ++it;
      reset_error(ctx);
      a.eta = eta_a;
      if (lanes)
        lane::k_lane_fwd_reduce<D, d><<<lblocks, lane::kLaneThreads, 0, st>>>(a, cst, agg);
      else
        k_fast_fwd_reduce<D, d><<<blocks, kThreads, sm, st>>>(a, cst, agg);
      note_launch(ctx, "fast_fwd_reduce");
      ScanTally tf, tr;
      if (lane_scans())
        lane::LaneScan<D, lane::LFOps<D>, false>::run(ctx, agg, agg, nc, 0, scan_fanin(), tf);
      else
        tf = Engine<D>::scan_filtering_gauss(ctx, nc, agg, agg, scan_fanin());
      if (lanes) {
        lane::k_lane_fwd_down<D, d><<<lblocks, lane::kLaneThreads, 0, st>>>(a, cst, agg, soa);
        note_launch(ctx, "fast_fwd_down");
        lane::k_lane_bfold<D><<<lblocks, lane::kLaneThreads, 0, st>>>(soa, N, L, nc, bagg);
        note_launch(ctx, "fast_bwd_fold");
      } else {
        k_fast_fwd_down<D, d><<<blocks, kThreads, sm, st>>>(a, cst, agg, elems, bagg);
        note_launch(ctx, "fast_fwd_down");
      }
      if (lane_scans())
        lane::LaneScan<D, lane::LMOps<D>, true>::run(ctx, bagg, bagg, nc, 0, scan_fanin(), tr);
      else
        tr = Engine<D>::scan_means_terminal(ctx, nc, bagg, scan_fanin());
      if (lanes)
        lane::k_lane_bwd_down<D, d, false><<<lblocks, lane::kLaneThreads, 0, st>>>(a, cst, soa, bagg, eta_a,
                                                                                  eta_b, part);
      else
        k_fast_bwd_down<D, d, false><<<blocks, kThreads, sm, st>>>(a, cst, elems, bagg, eta_a, eta_b, part);
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
    IE::finalize(ctx, s, eta_b, eta_a, cfg.linearization, it, prior.sigma, means, cov, sol_m, sol_c, res);
    return res;
  }
};

}  // namespace pode
