// Host driver of the large-state fused IEKS engine (big.cuh): per
// Gauss-Newton iteration three chunk-parallel passes, two one-CTA chunk
// chains and the reference's stopping rule (ieks.cpp:157-187) on three
// reduced scalars; finalize once.
#pragma once

#include <algorithm>
#include <cstring>
#include <vector>

#include "big.cuh"
#include "grp_fused.cuh"
#include "ieks.cuh"

namespace pode {

template <int D, int d>
struct BigEngine {
  using S = big::Slots<D, d>;
  static constexpr int B = D / d;

  static void set_attrs() {
    static OncePerDevice once;
    once([] {
      const int sm = int(big::big_smem_bytes<D>(false)), smc = int(big::big_smem_bytes<D>(true));
      auto set = [](const void* f, int bytes) {
        cuda_check(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "big smem");
      };
      set(reinterpret_cast<const void*>(big::k_big_fwd_reduce<D, d>), sm);
      set(reinterpret_cast<const void*>(big::k_big_chain_fwd<D, d>), smc);
      set(reinterpret_cast<const void*>(big::k_big_fwd_down<D, d, false>), sm);
      set(reinterpret_cast<const void*>(big::k_big_fwd_down<D, d, true>), sm);
      set(reinterpret_cast<const void*>(big::k_big_fin_fold<D, d>), sm);
      set(reinterpret_cast<const void*>(big::k_big_chain_fin<D>), sm);
      set(reinterpret_cast<const void*>(big::k_big_fin_bwd<D, d>), sm);
    });
  }

  static IeksResult run(pode_context* ctx, const host::Problem& p, const pode_prior& prior, const double* grid_h,
                        int64_t n1, const pode_ieks_config& cfg, double* means, double* cov, double* sol_m,
                        double* sol_c) {
    set_attrs();
    const size_t sm = big::big_smem_bytes<D>(false), smc = big::big_smem_bytes<D>(true);
    IeksSetup<D> s;
    IeksEngine<D>::setup(ctx, p, prior, grid_h, n1, s, false);
    cudaStream_t st = ctx->stream;
    Workspace& ws = ctx->ws;
    const int64_t N = s.N;
    // one CTA per chunk, about one per SM (the chain passes are sequential
    // over chunks: more chunks would lengthen them)
    int64_t nc = std::min<int64_t>(N, ctx->opt_chunk > 0 ? (N + ctx->opt_chunk - 1) / ctx->opt_chunk
                                                          : int64_t(ctx->sm_count));
    nc = std::max<int64_t>(nc, 1);
    const int L = static_cast<int>((N + nc - 1) / nc);
    nc = (N + L - 1) / L;

    // constants: sigma^2 Q Q^T, the unit-diffusion block, T_0^-1 mu_0
    std::vector<double> qq(size_t(D) * D, 0.0), q1u(size_t(B) * B);
    for (int i = 0; i < D; ++i)
      for (int j = 0; j < D; ++j) {
        double acc = 0.0;
        for (int k = 0; k < D; ++k) acc += s.h_q[size_t(i) * D + k] * s.h_q[size_t(j) * D + k];
        qq[size_t(i) * D + j] = acc;
      }
    for (int i = 0; i < B; ++i)
      for (int j = 0; j < B; ++j) q1u[size_t(i) * B + j] = s.h_qunit[size_t(i) * D + j];
    double* cst = ws.arr<double>("big_consts", size_t(D) * D + B * B);
    cuda_check(cudaMemcpyAsync(cst, qq.data(), sizeof(double) * D * D, cudaMemcpyHostToDevice, st), "qq");
    cuda_check(cudaMemcpyAsync(cst + D * D, q1u.data(), sizeof(double) * B * B, cudaMemcpyHostToDevice, st), "q1");

    const size_t DD = size_t(D) * D;
    double* eta_a = ws.arr<double>("big_eta_a", size_t(n1) * D);
    double* eta_b = ws.arr<double>("big_eta_b", size_t(n1) * D);
    double* E = ws.arr<double>("big_E", size_t(N) * DD);
    double* g = ws.arr<double>("big_g", size_t(N) * D + D);
    double* g_term = g + size_t(N) * D;
    double* agg = ws.arr<double>("big_agg", size_t(nc) * (3 * DD + 2 * D));
    double* prefix = ws.arr<double>("big_prefix", size_t(nc) * (DD + D));
    double* bagg = ws.arr<double>("big_bagg", size_t(nc) * (DD + D));
    double* suffix = ws.arr<double>("big_suffix", size_t(nc) * D);
    double* chain = ws.arr<double>("big_chain", 4 * DD + size_t(D) * (D + 1) + 2 * D);
    double* part = ws.arr<double>("big_part", size_t(nc) * 3 + 3);
    double* red = part + nc * 3;
    double* wsp = ws.arr<double>("big_ws", size_t(nc) * S::kStride);

    big::BigArgs a{};
    a.grid = s.grid;
    a.N = N;
    a.L = L;
    a.nchunks = nc;
    a.ek0 = cfg.linearization;
    a.prob = s.prob;
    a.err = reinterpret_cast<DevError*>(ctx->d_err);
    a.qq = cst;
    a.q1u = cst + D * D;
    a.m0 = s.init_m;
    a.ws = wsp;
    a.ws_stride = S::kStride;
    const bool phases = std::getenv("PODE_BIG_PHASES") != nullptr;
    if (phases) {
      a.phases = ws.arr<long long>("big_phases", 16);
      cuda_check(cudaMemsetAsync(a.phases, 0, sizeof(long long) * 16, st), "phases");
    }
    const unsigned th = big::kBT;

    grp::k_eta_fill_rows<D><<<grid1(n1 * D), kRedThreads, 0, st>>>(s.mu0, N, eta_a);
    note_launch(ctx, "fill");
    auto finish = [&]() {
      k_finish3<<<1, kRedThreads, 0, st>>>(part, nc, red);
      note_launch(ctx, "finish3");
      cuda_check(cudaMemcpyAsync(ctx->h_scalars, red, sizeof(double) * 3, cudaMemcpyDeviceToHost, st), "red");
    };
    reset_error(ctx);
    a.eta = eta_a;
    big::k_big_bwd_down<D, d, true><<<unsigned(nc), th, 0, st>>>(a, E, g, g_term, suffix, eta_a, eta_b, part, 1);
    note_launch(ctx, "big_objective");
    finish();
    cuda_check(cudaStreamSynchronize(st), "sync");
    double v_prev = 0.5 * ctx->h_scalars[0];

    IeksResult res;
    int it = 0;
    while (it < cfg.max_iterations) {
      ++it;
      reset_error(ctx);
      a.eta = eta_a;
      NvtxRange nv("big_iteration");
      big::k_big_fwd_reduce<D, d><<<unsigned(nc), th, sm, st>>>(a, agg, 1);
      note_launch(ctx, "big_fwd_reduce");
      big::k_big_chain_fwd<D, d><<<1, th, smc, st>>>(a, agg, prefix, chain, 1, nullptr);
      note_launch(ctx, "big_chain_fwd");
      big::k_big_fwd_down<D, d, false><<<unsigned(nc), th, sm, st>>>(a, prefix, E, g, g_term, bagg, nullptr, nullptr,
                                                                    nullptr, 1, 1, nullptr);
      note_launch(ctx, "big_fwd_down");
      big::k_big_chain_bwd<D><<<1, th, 0, st>>>(nc, bagg, suffix, nullptr);
      note_launch(ctx, "big_chain_bwd");
      big::k_big_bwd_down<D, d, false><<<unsigned(nc), th, 0, st>>>(a, E, g, g_term, suffix, eta_a, eta_b, part, 1);
      note_launch(ctx, "big_bwd_down");
      finish();
      IeksEngine<D>::check_linearization(ctx, s, it);  // syncs
      const double v = 0.5 * ctx->h_scalars[0];
      const double dmax = ctx->h_scalars[1], emax = ctx->h_scalars[2];
      res.trace.push_back(v);
      res.stats.combines = std::max(res.stats.combines, 2 * N + 2 * nc);
      res.stats.depth = std::max(res.stats.depth, int64_t(2 * L + 2 * nc));
      std::swap(eta_a, eta_b);
      const bool conv = (dmax <= cfg.traj_rtol * emax) ||
                        (std::fabs(v - v_prev) <= cfg.obj_atol + cfg.obj_rtol * std::fabs(v));
      v_prev = v;
      if (conv) {
        res.converged = true;
        break;
      }
    }
    res.iterations = it;
    if (phases) {  // debug: pass-C phase split of CTA 0 (clock64 cycles, all iterations)
      long long h[16];
      cuda_check(cudaMemcpy(h, a.phases, sizeof(h), cudaMemcpyDeviceToHost), "phases");
      std::fprintf(stderr, "[pode] big pass C phases (Mcycles, CTA 0):");
      for (int i = 0; i < 11; ++i) std::fprintf(stderr, " %d:%.2f", i, h[i] * 1e-6);
      std::fprintf(stderr, "\n");
      a.phases = nullptr;
    }
    // finalize at the final linearisation point (eta_b) with the newest
    // trajectory (eta_a); the last pass-B prefixes are for that point
    double* pf = ws.arr<double>("big_pf", size_t(N) * DD + DD);
    double* pterm = pf + size_t(N) * DD;
    double* sagg = ws.arr<double>("big_sagg", size_t(nc) * 2 * DD);
    double* ps = ws.arr<double>("big_ps", size_t(nc) * DD);
    a.eta = eta_b;
    reset_error(ctx);
    big::k_big_fwd_down<D, d, true><<<unsigned(nc), th, sm, st>>>(a, prefix, E, g, g_term, nullptr, pf, pterm, part, 1,
                                                                 1, nullptr);
    note_launch(ctx, "big_fin_fwd");
    k_finish3<<<1, kRedThreads, 0, st>>>(part, nc, red);
    note_launch(ctx, "finish3");
    IeksEngine<D>::check_linearization(ctx, s, it);
    big::k_big_fin_fold<D, d><<<unsigned(nc), th, sm, st>>>(a, E, pf, pterm, sagg, 1);
    note_launch(ctx, "big_fin_fold");
    big::k_big_chain_fin<D><<<1, th, sm, st>>>(nc, sagg, ps, chain, nullptr);
    note_launch(ctx, "big_chain_fin");
    const double count = double(N) * s.dim;
    big::BigOut o{means, cov, sol_m, sol_c};
    big::k_big_fin_bwd<D, d><<<unsigned(nc), th, sm, st>>>(a, E, pf, pterm, ps, eta_a, red, count, o, 1);
    note_launch(ctx, "big_fin_bwd");
    cuda_check(cudaMemcpyAsync(ctx->h_scalars, red, sizeof(double), cudaMemcpyDeviceToHost, st), "innov");
    IeksEngine<D>::check_linearization(ctx, s, it);  // syncs
    res.sigma_hat = std::sqrt(ctx->h_scalars[0] / count) * prior.sigma;
    return res;
  }
};

}  // namespace pode
