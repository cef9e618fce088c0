// Batched fused IEKS: many independent IVPs (one field kind and dimension,
// one prior, one grid, one config — a parameter or initial-value sweep;
// SURVEY.md §8(f) item 4) solved in ONE pass sequence per Gauss–Newton
// iteration, so small-N solves fill the GPU together.
//
// Layout: IVP b owns chunks [b S, (b+1) S) of the chunk axis (S = seg_chunks,
// a whole number of lane blocks; the first seg_real chunks cover its N steps,
// the rest are identity padding).  The lane passes are the kBatch
// instantiations of the single-solve kernels (lane.cuh); the aggregate scans
// run unsegmented over all chunks: IVP b's chunk 0 absorbs its own initial
// distribution (A = 0: ⊗_f ignores everything to its left) and its last chunk
// absorbs its terminal element (E = 0: the reverse ⊗_s ignores everything to
// its right), so the prefixes of one IVP never see another's.
//
// Stopping: each IVP follows the reference's rule (ieks.cpp:157-187) on its
// own objective; a converged IVP is frozen (its passes skip, both trajectory
// buffers keep its last two iterates) while the others continue, so every
// IVP's report equals its own para_ieks.  The loop is the same device-side
// while-graph as the single solve.  After the loop one more pass A + B at
// every IVP's final linearisation point rebuilds the prefixes, and the
// finalize kernels form covariances, sigma-hat and outputs for all IVPs.
#pragma once

#include <vector>

#include "fast_driver.cuh"

namespace pode {

// Per-IVP stopping state, one CUDA block per IVP (fixed-order reduction of
// its lane blocks' pass-E partials, as k_finish3).  init: objective of the
// constant start (ieks.cpp:147-148).
static __global__ void k_finish_batch(const double* part, int64_t bps, int* active, int* it_b, int* conv_b,
                                      double* vprev, double* trace, int max_it, double traj_rtol, double obj_atol,
                                      double obj_rtol, int init) {
  const int b = blockIdx.x;
  if (!active[b]) return;  // uniform per block
  double r[3];
  finish3_block(part + size_t(b) * bps * 3, bps, r);
  if (threadIdx.x != 0) return;
  const double v = 0.5 * r[0];
  if (init) {
    vprev[b] = v;
    return;
  }
  const int it = it_b[b];
  trace[size_t(b) * max_it + it] = v;
  const bool conv = (r[1] <= traj_rtol * r[2]) || (fabs(v - vprev[b]) <= obj_atol + obj_rtol * fabs(v));
  vprev[b] = v;
  it_b[b] = it + 1;
  conv_b[b] = conv ? 1 : 0;
  if (conv || it + 1 >= max_it) active[b] = 0;
}

// End of a batch iteration: the global iteration counter (trajectory buffer
// parity) advances, and in graph mode the while node continues while any IVP
// is active and no device error was raised.
static __global__ void k_batch_cond(int* it_dev, const int* active, int nseg, const unsigned long long* err,
                                    cudaGraphConditionalHandle h, int set) {
  int any = 0;
  for (int b = threadIdx.x; b < nseg; b += blockDim.x) any |= active[b];
  any = __syncthreads_or(any);
  if (threadIdx.x != 0) return;
  *it_dev += 1;
  if (set) cudaGraphSetConditional(h, (any && *err == ~0ull) ? 1u : 0u);
}

// Per-IVP sums of the finalize's innovation partials (one block per IVP).
static __global__ void k_seg_sums(const double* part, int64_t bps, double* out) {
  double r[3];
  finish3_block(part + size_t(blockIdx.x) * bps * 3, bps, r);
  if (threadIdx.x == 0) out[blockIdx.x] = r[0];
}

namespace lane {
// eta of every IVP <- its mu0 at every node (chunk-interleaved; node-N slots
// after the nc L D body, one per IVP).
template <int D>
__global__ void k_eta_fill_batch(const double* mu0s, int64_t nc, int L, int64_t seg_chunks, int nseg, double* base) {
  const int row = blockIdx.y;  // t * D + r; row L D: the node-N slots
  if (row == L * D) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nseg * D; i += gridDim.x * blockDim.x)
      base[nc * L * D + i] = mu0s[i];
    return;
  }
  const int r = row % D;
  const unsigned sc = static_cast<unsigned>(seg_chunks);
  double* dst = base + int64_t(row) * nc;
  for (unsigned c = blockIdx.x * blockDim.x + threadIdx.x; c < unsigned(nc); c += gridDim.x * blockDim.x)
    dst[c] = mu0s[(c / sc) * D + r];
}
}  // namespace lane

template <int D, int d>
struct BatchEngine {
  using P = LanePasses<D, d>;
  using FE = FastEngine<D, d, P>;
  static constexpr unsigned kTh = lane::kLaneThreads;

  static unsigned blocks(int64_t nc) { return P::blocks(nc); }

  // Chunk length: the total chunk count targets the single solve's ~256
  // resident lane threads per SM.
  static int chunk_len(pode_context* ctx, int64_t N, int nb) {
    if (ctx->opt_chunk > 0) return static_cast<int>(std::max<int64_t>(2, std::min<int64_t>(ctx->opt_chunk, N)));
    const int64_t target = int64_t(ctx->sm_count) * 256;
    int64_t L = (N * nb + target - 1) / target;
    L = std::max<int64_t>(L, 8);
    // at most N / 128 steps per chunk, so an IVP spans whole lane blocks
    // instead of padding most of one
    L = std::min<int64_t>(L, std::max<int64_t>(2, N / kTh));
    return static_cast<int>(std::max<int64_t>(2, std::min<int64_t>(L, std::min<int64_t>(N, 4096))));
  }

  // T_0^-1 (k_node_scales' formula for node 0 from the first step, ieks.cpp:28-33).
  static std::vector<double> scale_inv0(const double* grid_h, int nu, int dim) {
    std::vector<double> si0(D);
    const double h = grid_h[1] - grid_h[0], root_h = std::sqrt(h);
    double fact = 1.0;
    for (int i = nu; i >= 0; --i) {
      const int k = nu - i;
      if (k > 0) fact *= k;
      const double tau = root_h * std::pow(h, double(k)) / fact;
      for (int r = 0; r < dim; ++r) si0[r * (nu + 1) + i] = 1.0 / tau;
    }
    return si0;
  }

  // outputs: (nb (N+1)) x ... stacked device arrays (any may be null).
  static std::vector<IeksResult> run(pode_context* ctx, const std::vector<host::Problem>& ps, const pode_prior& prior,
                                     const double* grid_h, int64_t n1, const pode_ieks_config& cfg, double* means,
                                     double* cov, double* sol_m, double* sol_c) {
    using IE = IeksEngine<D>;
    P::set_attrs();
    {
      static OncePerDevice once;
      once([] {
        cuda_check(cudaFuncSetAttribute(lane::k_lane_fwd_down<D, d, false, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(lane::fwd_down_smem<D>())),
                   "batch pass C smem");
      });
    }
    const int nb = static_cast<int>(ps.size());
    IeksSetup<D> s;
    IE::setup(ctx, ps[0], prior, grid_h, n1, s, false);  // grid, prior constants
    cudaStream_t st = ctx->stream;
    Workspace& ws = ctx->ws;
    const int64_t N = s.N;
    const int L = chunk_len(ctx, N, nb);
    const int64_t seg_real = (N + L - 1) / L;
    const int64_t seg_chunks = (seg_real + kTh - 1) / kTh * kTh;
    const int64_t nc = seg_chunks * nb;
    const int64_t bps = seg_chunks / kTh;  // lane blocks per IVP
    FastConst<D> cst;
    std::memcpy(cst.q, s.h_q.data(), sizeof(cst.q));
    std::memcpy(cst.qunit, s.h_qunit.data(), sizeof(cst.qunit));
    std::memcpy(cst.qunit_rdiag, s.h_qinv.data(), sizeof(cst.qunit_rdiag));
    std::memcpy(cst.m0, s.h_m0.data(), sizeof(cst.m0));

    // per-IVP constants: field parameters, mu0 (taylor_init) and T_0^-1 mu0
    const std::vector<double> si0 = scale_inv0(grid_h, s.nu, s.dim);
    std::vector<DevProblem> h_probs(nb);
    std::vector<double> h_mu0(size_t(nb) * D), h_m0(size_t(nb) * D);
    for (int b = 0; b < nb; ++b) {
      const host::Problem& p = ps[b];
      if (p.kind != ps[0].kind || p.dim != ps[0].dim)
        throw ApiError(PODE_ERR_INVALID_INPUT, "ieks_batch: every problem must have the same kind and dimension");
      if (p.params.size() > size_t(kMaxParams)) throw ApiError(PODE_ERR_UNSUPPORTED, "too many problem params");
      h_probs[b] = DevProblem{};
      h_probs[b].kind = p.kind;
      h_probs[b].dim = p.dim;
      for (size_t k = 0; k < p.params.size(); ++k) h_probs[b].params[k] = p.params[k];
      const std::vector<double> mu0 = host::taylor_init(p, s.nu);
      for (int k = 0; k < D; ++k) {
        h_mu0[size_t(b) * D + k] = mu0[k];
        h_m0[size_t(b) * D + k] = si0[k] * mu0[k];
      }
    }
    DevProblem* probs = ws.arr<DevProblem>("batch_probs", nb);
    double* mu0s = ws.arr<double>("batch_mu0", size_t(nb) * D);
    double* m0s = ws.arr<double>("batch_m0", size_t(nb) * D);
    int* ints = ws.arr<int>("batch_ints", size_t(nb) * 3 + 2);
    int* active = ints;
    int* it_b = ints + nb;
    int* conv_b = ints + 2 * nb;
    int* it_dev = ints + 3 * nb;
    double* vprev = ws.arr<double>("batch_vprev", nb);
    const int max_it = std::max(1, cfg.max_iterations);
    double* trace = ws.arr<double>("batch_trace", size_t(nb) * max_it);
    cuda_check(cudaMemcpyAsync(probs, h_probs.data(), sizeof(DevProblem) * nb, cudaMemcpyHostToDevice, st), "probs");
    cuda_check(cudaMemcpyAsync(mu0s, h_mu0.data(), sizeof(double) * h_mu0.size(), cudaMemcpyHostToDevice, st), "mu0");
    cuda_check(cudaMemcpyAsync(m0s, h_m0.data(), sizeof(double) * h_m0.size(), cudaMemcpyHostToDevice, st), "m0");
    {
      std::vector<int> h_ints(size_t(nb) * 3 + 2, 0);
      for (int b = 0; b < nb; ++b) h_ints[b] = 1;
      cuda_check(cudaMemcpyAsync(ints, h_ints.data(), sizeof(int) * h_ints.size(), cudaMemcpyHostToDevice, st), "ints");
    }

    const size_t padded = size_t(nc) * L;
    const size_t eta_len = padded * D + size_t(nb) * D;
    double* pair0 = ws.arr<double>("batch_eta_a", eta_len);
    double* pair1 = ws.arr<double>("batch_eta_b", eta_len);
    FEd agg = Engine<D>::template alloc<FOps<D>>(ctx, "batch_agg", nc);
    lane::ElemSoA soa;
    {
      double* base = ws.arr<double>("batch_elems", padded * (D * D + D) + size_t(nb) * D);
      soa = lane::ElemSoA{base, base + padded * D * D, base + padded * (D * D + D), nc, L};
    }
    SEd bagg;
    {
      double* base = ws.arr<double>("batch_bagg", size_t(nc) * (D * D + D));
      bagg = SEd{base, base + size_t(nc) * D * D, nullptr};
    }
    const int64_t nparts = int64_t(blocks(nc));
    double* part = ws.arr<double>("batch_part", size_t(nparts) * 3);

    FastArgs a{s.grid, nullptr, nullptr, N, L, nc, cfg.linearization, s.prob,
               reinterpret_cast<DevError*>(ctx->d_err)};
    a.it_dev = it_dev;
    a.pair0 = pair0;
    a.pair1 = pair1;
    a.term_off = int64_t(padded) * D;
    a.seg_chunks = seg_chunks;
    a.seg_real = seg_real;
    a.probs = probs;
    a.m0s = m0s;
    a.active = active;

    lane::k_eta_fill_batch<D><<<lane::eta_fill_grid(nc, L, D), 256, 0, st>>>(mu0s, nc, L, seg_chunks, nb, pair0);
    note_launch(ctx, "fill");
    reset_error(ctx);
    // objective of the constant start (pass E on pair0 = iteration parity 0)
    lane::k_lane_bwd_down<D, d, true, true><<<blocks(nc), kTh, 0, st>>>(a, cst, soa, bagg, nullptr, nullptr, nullptr,
                                                                         nullptr, part);
    note_launch(ctx, "fast_objective");
    k_finish_batch<<<nb, kRedThreads, 0, st>>>(part, bps, active, it_b, conv_b, vprev, trace, max_it, cfg.traj_rtol,
                                               cfg.obj_atol, cfg.obj_rtol, 1);
    note_launch(ctx, "finish_batch");

    ScanTally tf, tr;
    auto body = [&](bool graph, cudaGraphConditionalHandle h) {
      lane::k_lane_fwd_reduce<D, d, true><<<blocks(nc), kTh, lane::fwd_reduce_smem<D>(), st>>>(a, cst, agg);
      note_launch(ctx, "fast_fwd_reduce");
      tf = Engine<D>::scan_filtering_gauss(ctx, nc, agg, agg, FE::scan_fanin());
      lane::k_lane_fwd_down<D, d, false, true><<<blocks(nc), kTh, lane::fwd_down_smem<D>(), st>>>(
          a, cst, agg, soa, nullptr, nullptr, nullptr, bagg);
      note_launch(ctx, "fast_fwd_down");
      tr = Engine<D>::scan_means_terminal(ctx, nc, bagg, FE::scan_fanin());
      lane::k_lane_bwd_down<D, d, false, true><<<blocks(nc), kTh, 0, st>>>(a, cst, soa, bagg, nullptr, nullptr,
                                                                            nullptr, nullptr, part);
      note_launch(ctx, "fast_bwd_down");
      k_finish_batch<<<nb, kRedThreads, 0, st>>>(part, bps, active, it_b, conv_b, vprev, trace, max_it, cfg.traj_rtol,
                                                 cfg.obj_atol, cfg.obj_rtol, 0);
      note_launch(ctx, "finish_batch");
      k_batch_cond<<<1, kRedThreads, 0, st>>>(it_dev, active, nb, ctx->d_err, h, graph ? 1 : 0);
      note_launch(ctx, "batch_cond");
    };
    // iteration 1 eagerly (the scans' workspaces are allocated outside capture)
    body(false, cudaGraphConditionalHandle{});
    IE::check_linearization(ctx, s, 1);  // syncs
    std::vector<int> h_act(nb);
    cuda_check(cudaMemcpy(h_act.data(), active, sizeof(int) * nb, cudaMemcpyDeviceToHost), "active");
    bool any = false;
    for (int b = 0; b < nb; ++b) any |= h_act[b] != 0;
    if (any) {  // iterations 2.. in the device-side while loop
      pode_context::GraphSlot& slot = ctx->graphs["batch_" + std::to_string(D) + "_" + std::to_string(d)];
      typename FE::KeyWriter kw;
      kw << ctx->ws.generation << N << L << nc << nb << seg_chunks << cfg.linearization << cfg.max_iterations
         << cfg.traj_rtol << cfg.obj_atol << cfg.obj_rtol << FE::scan_fanin() << bscan_max() << a.grid << pair0
         << pair1 << agg.a << soa.e << bagg.e << part << ints << vprev << trace << probs << m0s << ctx->d_err;
      for (int k = 0; k < D * D; ++k) kw << cst.q[k] << cst.qunit[k];
      for (int k = 0; k < D; ++k) kw << cst.qunit_rdiag[k];
      if (slot.exec == nullptr || slot.key != kw.k) {
        if (slot.exec) cudaGraphExecDestroy(slot.exec);
        if (slot.graph) cudaGraphDestroy(slot.graph);
        slot = pode_context::GraphSlot{};
        cuda_check(cudaGraphCreate(&slot.graph, 0), "graph");
        cudaGraphConditionalHandle h;
        cuda_check(cudaGraphConditionalHandleCreate(&h, slot.graph, 1, cudaGraphCondAssignDefault), "cond handle");
        cudaGraphNodeParams np = {};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = h;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        cuda_check(cudaGraphAddNode(&node, slot.graph, nullptr, 0, &np), "while node");
        cudaGraph_t g_body = np.conditional.phGraph_out[0];
        const int64_t l0 = ctx->launches;
        cuda_check(cudaStreamBeginCaptureToGraph(st, g_body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed),
                   "capture");
        try {
          body(true, h);
          cuda_check(cudaStreamEndCapture(st, &g_body), "end capture");
          slot.per_iter = ctx->launches - l0;
          ctx->launches = l0;
          cuda_check(cudaGraphInstantiate(&slot.exec, slot.graph, 0), "instantiate");
        } catch (...) {
          cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
          if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
            cudaGraph_t dropped = nullptr;
            cudaStreamEndCapture(st, &dropped);
          }
          cudaGetLastError();
          if (slot.exec) cudaGraphExecDestroy(slot.exec);
          if (slot.graph) cudaGraphDestroy(slot.graph);
          slot = pode_context::GraphSlot{};
          ctx->launches = l0;
          throw;
        }
        slot.key = kw.k;
      }
      cuda_check(cudaGraphLaunch(slot.exec, st), "graph launch");
      int it_h = 0;
      cuda_check(cudaMemcpyAsync(&it_h, it_dev, sizeof(int), cudaMemcpyDeviceToHost, st), "it");
      const unsigned long long ekey = fetch_error(ctx);  // syncs
      ctx->launches += slot.per_iter * (it_h - 1);
      if (ekey != ~0ull) IE::check_linearization(ctx, s, it_h);  // throws
    }

    std::vector<int> h_it(nb), h_conv(nb);
    std::vector<double> h_trace(size_t(nb) * max_it);
    cuda_check(cudaMemcpy(h_it.data(), it_b, sizeof(int) * nb, cudaMemcpyDeviceToHost), "it_b");
    cuda_check(cudaMemcpy(h_conv.data(), conv_b, sizeof(int) * nb, cudaMemcpyDeviceToHost), "conv_b");
    cuda_check(cudaMemcpy(h_trace.data(), trace, sizeof(double) * h_trace.size(), cudaMemcpyDeviceToHost), "trace");

    // ---- finalize: every IVP at its own final linearisation point
    NvtxRange nv("batch_finalize");
    FastArgs f = a;
    f.it_dev = nullptr;
    f.active = nullptr;
    f.seg_it = it_b;
    lane::k_lane_fwd_reduce<D, d, true><<<blocks(nc), kTh, lane::fwd_reduce_smem<D>(), st>>>(f, cst, agg);
    note_launch(ctx, "fast_fwd_reduce");
    const ScanTally tfin = Engine<D>::scan_filtering_gauss(ctx, nc, agg, agg, FE::scan_fanin());
    double* cf = ws.arr<double>("batch_cf", padded * D * D + size_t(nb) * D * D);
    double* cterm = cf + padded * D * D;
    double* fpart = ws.arr<double>("batch_fpart", size_t(nparts) * 3);
    double* innov = ws.arr<double>("batch_innov", nb);
    lane::k_lane_fwd_down<D, d, true, true><<<blocks(nc), kTh, 0, st>>>(f, cst, agg, soa, cf, cterm, fpart);
    note_launch(ctx, "fin_fwd");
    k_seg_sums<<<nb, kRedThreads, 0, st>>>(fpart, bps, innov);
    note_launch(ctx, "seg_sums");
    IE::check_linearization(ctx, s, *std::max_element(h_it.begin(), h_it.end()));  // syncs
    SEd sagg = Engine<D>::template alloc<SOps<D>>(ctx, "batch_sagg", nc);
    lane::k_lane_fin_fold<D, d, true><<<blocks(nc), kTh, 0, st>>>(f, cst, soa, cf, cterm, sagg);
    note_launch(ctx, "fin_fold");
    const ScanTally ts = Engine<D>::scan_smoothing(ctx, nc, sagg, sagg, true);
    const double count = double(N) * s.dim;
    lane::k_lane_fin_bwd<D, d, true><<<blocks(nc), kTh, 0, st>>>(f, cst, soa, cf, cterm, sagg, nullptr, nullptr, innov,
                                                                  count, lane::FinOut{means, cov, sol_m, sol_c});
    note_launch(ctx, "fin_bwd");
    std::vector<double> h_innov(nb);
    cuda_check(cudaMemcpyAsync(h_innov.data(), innov, sizeof(double) * nb, cudaMemcpyDeviceToHost, st), "innov");
    IE::check_linearization(ctx, s, *std::max_element(h_it.begin(), h_it.end()));  // syncs

    std::vector<IeksResult> out(nb);
    for (int b = 0; b < nb; ++b) {
      IeksResult& r = out[b];
      r.iterations = h_it[b];
      r.converged = h_conv[b] != 0;
      r.trace.assign(h_trace.begin() + size_t(b) * max_it, h_trace.begin() + size_t(b) * max_it + h_it[b]);
      r.sigma_hat = std::sqrt(h_innov[b] / count) * prior.sigma;
      // this IVP's share of the scan tally (its chunk folds, 1 / nb of the
      // shared aggregate scans, the finalize's smoothing scan)
      r.stats.combines = (N - seg_real) + tf.combines / nb + N + (tfin.combines + ts.combines) / nb;
      r.stats.depth = int64_t(L) + tf.depth + int64_t(L) + tr.depth;
    }
    return out;
  }
};

}  // namespace pode
