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
#include "grp_fused.cuh"
#include "ieks.cuh"
#include "lane.cuh"
#include "nccl.hpp"

namespace pode {

namespace lane {

// eta (N+1 nodes, chunk-interleaved + node-N slot) <- mu0 at every node:
// row (t D + r) of the layout (blockIdx.y) holds mu0[r] for every chunk.
template <int D>
__global__ void k_eta_fill(const double* mu0, int64_t nc, int L, double* base) {
  const int row = blockIdx.y;  // t * D + r, t < L; row L D: the node-N slot
  const double v = mu0[row % D];
  if (row == L * D) {
    if (blockIdx.x == 0 && threadIdx.x < D) base[nc * L * D + threadIdx.x] = mu0[threadIdx.x];
    return;
  }
  double* dst = base + int64_t(row) * nc;
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < nc; c += int64_t(gridDim.x) * blockDim.x)
    dst[c] = v;
}
inline dim3 eta_fill_grid(int64_t nc, int L, int D) {
  return dim3(static_cast<unsigned>(std::min<int64_t>((nc + 255) / 256, 64)), static_cast<unsigned>(L * D + 1));
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

// Device-side loop state of the graph-captured IEKS iteration.
struct LoopState {
  int it;         // completed iterations
  int converged;
  int max_it;
  int pad;
  double v_prev;  // objective of the previous iterate
  double traj_rtol, obj_atol, obj_rtol;
};

// Per-iteration finish in graph-loop mode: the fixed-order reduction of the
// pass-E partials (as k_finish3), the objective trace, the reference's
// stopping rule (ieks.cpp:157-187) and the while-node condition; a device
// error (singular factor / non-finite field) also ends the loop.
static __global__ void k_finish_iter(const double* part, int64_t nparts, LoopState* ls, double* trace,
                                     const unsigned long long* err, cudaGraphConditionalHandle h) {
  double r[3];
  finish3_block(part, nparts, r);
  if (threadIdx.x != 0) return;
  const double v = 0.5 * r[0];
  trace[ls->it] = v;
  const bool conv =
      (r[1] <= ls->traj_rtol * r[2]) || (fabs(v - ls->v_prev) <= ls->obj_atol + ls->obj_rtol * fabs(v));
  ls->v_prev = v;
  ls->it += 1;
  ls->converged = conv ? 1 : 0;
  const bool failed = *err != ~0ull;
  cudaGraphSetConditional(h, (!conv && !failed && ls->it < ls->max_it) ? 1u : 0u);
}

// Packed device moves of up to five fields (one launch per element move of
// the shard exchanges) and a one-double store.
struct MoveSpec {
  const double* src[5];
  double* dst[5];
  int len[5];
  int nfields;
};
static __global__ void k_move_fields(MoveSpec m) {
  for (int f = 0; f < m.nfields; ++f)
    for (int i = threadIdx.x; i < m.len[f]; i += blockDim.x) m.dst[f][i] = m.src[f][i];
}
static __global__ void k_set_scalar(double* p, double v) { *p = v; }

// Launch policies of the fused iteration: the lane-serial passes (lane.cuh,
// one chunk per thread, chunk-interleaved HBM layout; D <= 9) and the
// group-of-D-lanes passes (grp_fused.cuh, one chunk per group, node-major
// layout; D = 10..16).  The driver below is shared.
template <int D, int d>
struct LanePasses {
  static constexpr bool kLane = true;
  static constexpr const char* kName = "lane";
  static int64_t target_chunks(pode_context* ctx) { return int64_t(ctx->sm_count) * 256; }
  static unsigned blocks(int64_t nc) { return static_cast<unsigned>((nc + lane::kLaneThreads - 1) / lane::kLaneThreads); }
  static void set_attrs() {
    static OncePerDevice once;
    once([] {
      cuda_check(cudaFuncSetAttribute(lane::k_lane_fwd_down<D, d, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(lane::fwd_down_smem<D>())),
                 "pass C smem");
      if constexpr (lane::fwd_reduce_smem<D>() > 0) {
        cuda_check(cudaFuncSetAttribute(lane::k_lane_fwd_reduce<D, d, false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(lane::fwd_reduce_smem<D>())),
                   "pass A smem");
        cuda_check(cudaFuncSetAttribute(lane::k_lane_fwd_reduce<D, d, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(lane::fwd_reduce_smem<D>())),
                   "pass A smem");
      }
    });
  }
  static void fill(cudaStream_t st, const double* mu0, int64_t nc, int L, double* eta) {
    lane::k_eta_fill<D><<<lane::eta_fill_grid(nc, L, D), 256, 0, st>>>(mu0, nc, L, eta);
  }
  static void rows(cudaStream_t st, const double* base, const double* term, int64_t N, int L, int64_t nc,
                   double* out) {
    lane::k_eta_rows<D><<<grid1((N + 1) * D), kRedThreads, 0, st>>>(base, term, N, L, nc, out);
  }
  static void fwd_reduce(cudaStream_t st, const FastArgs& a, const FastConst<D>& cst, const FEd& agg) {
    lane::k_lane_fwd_reduce<D, d><<<blocks(a.nchunks), lane::kLaneThreads, lane::fwd_reduce_smem<D>(), st>>>(a, cst, agg);
  }
  static void fwd_down(cudaStream_t st, const FastArgs& a, const FastConst<D>& cst, const FEd& agg,
                       const lane::ElemSoA& soa, const SEd& bagg) {
    lane::k_lane_fwd_down<D, d><<<blocks(a.nchunks), lane::kLaneThreads, lane::fwd_down_smem<D>(), st>>>(
        a, cst, agg, soa, nullptr, nullptr, nullptr, bagg);
  }
  template <bool kInit>
  static void bwd_down(cudaStream_t st, const FastArgs& a, const FastConst<D>& cst, const lane::ElemSoA& soa,
                       const SEd& bagg, const double* eo, const double* ot, double* en, double* nt, double* part) {
    lane::k_lane_bwd_down<D, d, kInit><<<blocks(a.nchunks), lane::kLaneThreads, 0, st>>>(a, cst, soa, bagg, eo, ot, en,
                                                                                         nt, part);
  }
  static void fin_fwd(cudaStream_t st, const FastArgs& a, const FastConst<D>& cst, const FEd& agg,
                      const lane::ElemSoA& soa, double* cf, double* cterm, double* part) {
    lane::k_lane_fwd_down<D, d, true><<<blocks(a.nchunks), lane::kLaneThreads, 0, st>>>(a, cst, agg, soa, cf, cterm,
                                                                                        part);
  }
  static void fin_fold(cudaStream_t st, const FastArgs& a, const FastConst<D>& cst, const lane::ElemSoA& soa,
                       const double* cf, const double* cterm, const SEd& sagg) {
    lane::k_lane_fin_fold<D, d><<<blocks(a.nchunks), lane::kLaneThreads, 0, st>>>(a, cst, soa, cf, cterm, sagg);
  }
  static void fin_bwd(cudaStream_t st, const FastArgs& a, const FastConst<D>& cst, const lane::ElemSoA& soa,
                      const double* cf, const double* cterm, const SEd& sagg, const double* eo, const double* eot,
                      const double* red, double count, const lane::FinOut& out) {
    lane::k_lane_fin_bwd<D, d><<<blocks(a.nchunks), lane::kLaneThreads, 0, st>>>(a, cst, soa, cf, cterm, sagg, eo, eot,
                                                                                red, count, out);
  }
};

template <int D, int d>
struct GroupPasses {
  static constexpr bool kLane = false;
  static constexpr const char* kName = "grp";
  // groups are latency-bound per step: ~32 chunks per SM
  // One resident wave of groups (the passes are latency-bound chains, and a
  // second wave only halves the chunk length while doubling the aggregate
  // scan: rigid body IWP(4) 2^20, 29.92 -> 29.49 ms per iteration).
  static int64_t target_chunks(pode_context* ctx) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, grp::k_grp_fwd_down<D, d, false>, kThreads,
                                                  smem_bytes<D>());
    cudaGetLastError();
    const int64_t groups = int64_t(std::max(per_sm, 1)) * kWarpsPerBlock * Grp<D>::kPerWarp;
    return int64_t(ctx->sm_count) * groups;
  }
  static unsigned blocks(int64_t nc) { return blocks_for<D>(nc); }
  static void set_attrs() {
    static OncePerDevice once;
    once([] {
      const int bytes = int(smem_bytes<D>());
      cudaFuncSetAttribute(grp::k_grp_fwd_reduce<D, d>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      cudaFuncSetAttribute(grp::k_grp_fwd_down<D, d, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      cudaFuncSetAttribute(grp::k_grp_fwd_down<D, d, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      cudaFuncSetAttribute(grp::k_grp_bwd_down<D, d, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      cudaFuncSetAttribute(grp::k_grp_bwd_down<D, d, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      cudaFuncSetAttribute(grp::k_grp_fin_fold<D, d>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      cudaFuncSetAttribute(grp::k_grp_fin_bwd<D, d>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    });
  }
  static void fill(cudaStream_t st, const double* mu0, int64_t nc, int L, double* eta) {
    grp::k_eta_fill_rows<D><<<grid1((nc * L + 1) * D), kRedThreads, 0, st>>>(mu0, nc * L, eta);
  }
  static void rows(cudaStream_t st, const double* base, const double* term, int64_t N, int, int64_t,
                   double* out) {
    cuda_check(cudaMemcpyAsync(out, base, sizeof(double) * N * D, cudaMemcpyDeviceToDevice, st), "eta rows");
    cuda_check(cudaMemcpyAsync(out + N * D, term, sizeof(double) * D, cudaMemcpyDeviceToDevice, st), "eta rows");
  }
  static void fwd_reduce(cudaStream_t st, const FastArgs& a, const FastConst<D>& cst, const FEd& agg) {
    grp::k_grp_fwd_reduce<D, d><<<blocks(a.nchunks), kThreads, smem_bytes<D>(), st>>>(a, cst, agg);
  }
  static void fwd_down(cudaStream_t st, const FastArgs& a, const FastConst<D>& cst, const FEd& agg,
                       const lane::ElemSoA& soa, const SEd& bagg) {
    grp::k_grp_fwd_down<D, d, false><<<blocks(a.nchunks), kThreads, smem_bytes<D>(), st>>>(a, cst, agg, soa, nullptr,
                                                                                         nullptr, nullptr, bagg);
  }
  template <bool kInit>
  static void bwd_down(cudaStream_t st, const FastArgs& a, const FastConst<D>& cst, const lane::ElemSoA& soa,
                       const SEd& bagg, const double* eo, const double* ot, double* en, double* nt, double* part) {
    grp::k_grp_bwd_down<D, d, kInit><<<blocks(a.nchunks), kThreads, smem_bytes<D>(), st>>>(a, cst, soa, bagg, eo, ot,
                                                                                          en, nt, part);
  }
  static void fin_fwd(cudaStream_t st, const FastArgs& a, const FastConst<D>& cst, const FEd& agg,
                      const lane::ElemSoA& soa, double* cf, double* cterm, double* part) {
    grp::k_grp_fwd_down<D, d, true><<<blocks(a.nchunks), kThreads, smem_bytes<D>(), st>>>(a, cst, agg, soa, cf, cterm,
                                                                                        part, SEd{});
  }
  static void fin_fold(cudaStream_t st, const FastArgs& a, const FastConst<D>& cst, const lane::ElemSoA& soa,
                       const double* cf, const double* cterm, const SEd& sagg) {
    grp::k_grp_fin_fold<D, d><<<blocks(a.nchunks), kThreads, smem_bytes<D>(), st>>>(a, cst, soa, cf, cterm, sagg);
  }
  static void fin_bwd(cudaStream_t st, const FastArgs& a, const FastConst<D>& cst, const lane::ElemSoA& soa,
                      const double* cf, const double* cterm, const SEd& sagg, const double* eo, const double* eot,
                      const double* red, double count, const lane::FinOut& out) {
    grp::k_grp_fin_bwd<D, d><<<blocks(a.nchunks), kThreads, smem_bytes<D>(), st>>>(a, cst, soa, cf, cterm, sagg, eo,
                                                                                   eot, red, count, out);
  }
};

template <int D, int d, class Pass = LanePasses<D, d>>
struct FastEngine {
  // Iterations 2.. run as one CUDA graph with a device-side while node (no
  // host round trip per iteration) unless profiling or PODE_GRAPH=0.
  static bool use_graph(pode_context* ctx, const pode_ieks_config& cfg) {
    const char* env = std::getenv("PODE_GRAPH");
    return !ctx->prof_on && cfg.max_iterations > 1 && !(env != nullptr && *env != '\0' && std::atoi(env) == 0);
  }

  template <class Body>
  // `key` serialises every argument the captured kernels see (plus the
  // workspace generation): an identical key reuses the instantiated graph of
  // an earlier solve on this context instead of capturing again.
  static void graph_loop(pode_context* ctx, const IeksSetup<D>& s, Body& body, LoopState* ls, double* trace_dev,
                         int& it, double& v_prev, const pode_ieks_config& cfg, IeksResult& res,
                         const std::string& key) {
    cudaStream_t st = ctx->stream;
    LoopState h0{it, 0, cfg.max_iterations, 0, v_prev, cfg.traj_rtol, cfg.obj_atol, cfg.obj_rtol};
    cuda_check(cudaMemcpyAsync(ls, &h0, sizeof(h0), cudaMemcpyHostToDevice, st), "loop state");
    reset_error(ctx);
    pode_context::GraphSlot& slot = ctx->graphs["ieks_" + std::to_string(D) + "_" + std::to_string(d)];
    if (slot.exec == nullptr || slot.key != key) {
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
        // leave the stream out of capture mode and drop the half-built graph,
        // so the context stays usable for the next solve
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
      slot.key = key;
    }
    cuda_check(cudaGraphLaunch(slot.exec, st), "graph launch");
    LoopState hs;
    cuda_check(cudaMemcpyAsync(&hs, ls, sizeof(hs), cudaMemcpyDeviceToHost, st), "loop state");
    const unsigned long long ekey = fetch_error(ctx);  // syncs
    ctx->launches += slot.per_iter * (hs.it - it);
    std::vector<double> tr(size_t(hs.it), 0.0);
    if (hs.it > it)
      cuda_check(cudaMemcpy(tr.data() + it, trace_dev + it, sizeof(double) * (hs.it - it), cudaMemcpyDeviceToHost),
                 "trace");
    for (int k = it; k < hs.it; ++k) res.trace.push_back(tr[k]);
    it = hs.it;
    v_prev = hs.v_prev;
    res.converged = hs.converged != 0;
    if (ekey != ~0ull) IeksEngine<D>::check_linearization(ctx, s, it);  // throws
  }

  // Byte key of the values a captured iteration depends on.
  struct KeyWriter {
    std::string k;
    template <class T>
    KeyWriter& operator<<(const T& v) {
      k.append(reinterpret_cast<const char*>(&v), sizeof(T));
      return *this;
    }
  };

  // Chunk-aggregate scans run on the group engine (engine.cuh): a lane-serial
  // ⊗_f needs ~250 live doubles per thread and spills.
  static int scan_fanin() {
    const char* env = std::getenv("PODE_SCAN_FANIN");
    const int v = (env && *env) ? std::atoi(env) : 8;  // tools/knob_sweep.py: 8 is fastest per iteration
    return v >= 2 ? v : 4;
  }

  static void set_attrs() { Pass::set_attrs(); }

  // Lane passes: one chunk per thread, ~256 resident threads per SM; group
  // passes: one chunk per group, ~32 per SM.
  static int chunk_len(pode_context* ctx, int64_t N) {
    if (ctx->opt_chunk > 0)  // pode_context_set_option(PODE_OPT_CHUNK_LEN)
      return static_cast<int>(std::max<int64_t>(2, std::min<int64_t>(ctx->opt_chunk, std::max<int64_t>(N, 2))));
    const char* env = std::getenv("PODE_CHUNK");  // developer override; unset or empty: the default below
    if (env && *env) return static_cast<int>(std::max<int64_t>(2, std::min<int64_t>(std::atoll(env), std::max<int64_t>(N, 2))));
    const int64_t target = Pass::target_chunks(ctx);
    const int64_t L = (N + target - 1) / target;
    // Floor of the chunk length: below one resident wave of chunks the lane
    // passes are latency chains of L steps, so small grids take short chunks
    // (FHN, ms per iteration, tools/small_n_chunks.py: N = 2^12 L = 2 0.219
    // vs L = 8 0.260; 2^14 0.251 vs 0.282; 2^16 L = 8 best).  Group passes
    // keep 8.
    const int64_t lmin = Pass::kLane ? std::max<int64_t>(2, std::min<int64_t>(8, N / 8192)) : 8;
    return static_cast<int>(std::max<int64_t>(lmin, std::min<int64_t>(L, 4096)));
  }

  static IeksResult run(pode_context* ctx, const host::Problem& p, const pode_prior& prior, const double* grid_h,
                        int64_t n1, const pode_ieks_config& cfg, double* means, double* cov, double* sol_m,
                        double* sol_c) {
    using IE = IeksEngine<D>;
    set_attrs();
    IeksSetup<D> s;
    const bool element_finalize = std::getenv("PODE_FINALIZE") && std::string(std::getenv("PODE_FINALIZE")) == "elements";
    IE::setup(ctx, p, prior, grid_h, n1, s, element_finalize);
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
    const int64_t nparts = int64_t(Pass::blocks(nc));
    double* part = ws.arr<double>("fast_part", nparts * 3 + 3);
    double* red = part + nparts * 3;
    auto term = [&](double* base) { return base + padded * D; };
    FastArgs a{s.grid, eta_a, term(eta_a), N, L, nc, cfg.linearization, s.prob,
               reinterpret_cast<DevError*>(ctx->d_err)};

    Pass::fill(st, s.mu0, nc, L, eta_a);
    note_launch(ctx, "fill");
    auto finish = [&]() {
      k_finish3<<<1, kRedThreads, 0, st>>>(part, nparts, red);
      note_launch(ctx, "finish3");
      cuda_check(cudaMemcpyAsync(ctx->h_scalars, red, sizeof(double) * 3, cudaMemcpyDeviceToHost, st), "red");
    };
    // objective of the constant start (ieks.cpp:147-148)
    Pass::template bwd_down<true>(st, a, cst, soa, bagg, eta_a, term(eta_a), eta_b, term(eta_b), part);
    note_launch(ctx, "fast_objective");
    finish();
    cuda_check(cudaStreamSynchronize(st), "sync");
    prof_mark(ctx);
    double v_prev = 0.5 * ctx->h_scalars[0];

    IeksResult res;
    int it = 0;
    double* const pair0 = eta_a;  // trajectory buffers: iteration i (0-based)
    double* const pair1 = eta_b;  // linearises at pair[i & 1]
    LoopState* ls = ws.arr<LoopState>("fast_loop", 1);
    double* trace_dev = ws.arr<double>("fast_trace", size_t(std::max(1, cfg.max_iterations)));
    // One iteration's launches.  graph: buffers by device iteration parity
    // and the stopping rule evaluated on the device (k_finish_iter).
    auto body = [&](bool graph, cudaGraphConditionalHandle h) {
      FastArgs ag = a;
      if (graph) {
        ag.it_dev = &ls->it;
        ag.pair0 = pair0;
        ag.pair1 = pair1;
        ag.term_off = int64_t(padded) * D;
      } else {
        ag.eta = eta_a;
        ag.eta_term = term(eta_a);
      }
      {
        NvtxRange r("pass_A_chunk_fold");
        Pass::fwd_reduce(st, ag, cst, agg);
        note_launch(ctx, "fast_fwd_reduce");
      }
      ScanTally tf, tr;
      {
        NvtxRange r("pass_B_aggregate_scan");
        tf = Engine<D>::scan_filtering_gauss(ctx, nc, agg, agg, scan_fanin());
      }
      {
        NvtxRange r("pass_C_filter_smoothing_elements");
        Pass::fwd_down(st, ag, cst, agg, soa, bagg);
        note_launch(ctx, "fast_fwd_down");
      }
      {
        NvtxRange r("pass_D_backward_scan");
        tr = Engine<D>::scan_means_terminal(ctx, nc, bagg, scan_fanin());
      }
      {
        NvtxRange r("pass_E_backward_means_objective");
        Pass::template bwd_down<false>(st, ag, cst, soa, bagg, eta_a, term(eta_a), eta_b, term(eta_b), part);
        note_launch(ctx, "fast_bwd_down");
      }
      if (graph) {
        k_finish_iter<<<1, kRedThreads, 0, st>>>(part, nparts, ls, trace_dev, ctx->d_err, h);
        note_launch(ctx, "finish_iter");
      } else {
        finish();
      }
      // scan tally of the whole time axis: chunk folds + aggregate scans
      res.stats.combines = std::max(res.stats.combines, (N - nc) + tf.combines + N);
      res.stats.depth = std::max(res.stats.depth, int64_t(L) + tf.depth + int64_t(L) + tr.depth);
    };
    while (it < cfg.max_iterations) {
      if (it == 1 && use_graph(ctx, cfg)) {  // workspaces exist after one eager iteration
        KeyWriter kw;
        kw << Pass::kName << ctx->ws.generation << N << L << nc << padded << cfg.linearization << scan_fanin() << bscan_max()
           << a.grid << a.err << a.prob.kind << a.prob.dim << pair0 << pair1 << agg.a << agg.b << agg.c << agg.eta
           << agg.j << soa.e << soa.g << soa.term << bagg.e << bagg.g << part << nparts << ls << trace_dev
           << ctx->d_err;
        for (int k = 0; k < kMaxParams; ++k) kw << a.prob.params[k];
        for (int k = 0; k < D * D; ++k) kw << cst.q[k] << cst.qunit[k];
        for (int k = 0; k < D; ++k) kw << cst.qunit_rdiag[k] << cst.m0[k];
        graph_loop(ctx, s, body, ls, trace_dev, it, v_prev, cfg, res, kw.k);
        if (res.converged || it >= cfg.max_iterations) break;
        continue;  // unreachable: the device loop runs to convergence or the budget
      }
      ++it;
      reset_error(ctx);
      body(false, cudaGraphConditionalHandle{});
      IE::check_linearization(ctx, s, it);  // syncs the stream
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
    // newest trajectory in eta_a, final linearisation point in eta_b
    eta_a = (it & 1) ? pair1 : pair0;
    eta_b = (it & 1) ? pair0 : pair1;
    res.iterations = it;
    if (element_finalize) {
      // row-major copies of the final linearisation point and trajectory
      double* lin_rows = ws.arr<double>("lane_lin_rows", size_t(n1) * D);
      double* out_rows = ws.arr<double>("lane_out_rows", size_t(n1) * D);
      Pass::rows(st, eta_b, term(eta_b), N, L, nc, lin_rows);
      note_launch(ctx, "eta_rows");
      Pass::rows(st, eta_a, term(eta_a), N, L, nc, out_rows);
      note_launch(ctx, "eta_rows");
      IE::finalize(ctx, s, lin_rows, out_rows, cfg.linearization, it, prior.sigma, means, cov, sol_m, sol_c, res);
      return res;
    }
    finalize(ctx, s, a, cst, agg, soa, eta_a, term(eta_a), eta_b, term(eta_b), prior.sigma, it,
             lane::FinOut{means, cov, sol_m, sol_c}, res);
    return res;
  }

  // ------------------------------------------------ time-axis shards ---
  static constexpr int kFel = 3 * D * D + 2 * D;  // one filtering element
  static constexpr int kSel = 2 * D * D + D;      // one smoothing element
  // element views of a contiguous per-element buffer
  static FEd fview(double* b) {
    FEd e;
    e.a = b;
    e.c = b + D * D;
    e.j = b + 2 * D * D;
    e.b = b + 3 * D * D;
    e.eta = b + 3 * D * D + D;
    return e;
  }
  static SEd sview(double* b) { return SEd{b, b + 2 * D * D, b + D * D}; }  // {e, g, l}
  static void d2d(pode_context* ctx, double* dst, const double* src, size_t n) {
    if (src == nullptr || dst == nullptr) return;
    cuda_check(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream), "shard copy");
  }
  // Element i of src -> element j of dst, every field in one launch.
  static void fel_move(pode_context* ctx, const FEd& src, int64_t i, const FEd& dst, int64_t j) {
    k_move_fields<<<1, 128, 0, ctx->stream>>>(
        MoveSpec{{src.a + i * D * D, src.c + i * D * D, src.j + i * D * D, src.b + i * D, src.eta + i * D},
                 {dst.a + j * D * D, dst.c + j * D * D, dst.j + j * D * D, dst.b + j * D, dst.eta + j * D},
                 {D * D, D * D, D * D, D, D}, 5});
    note_launch(ctx, "move");
  }
  static void sel_move(pode_context* ctx, const SEd& src, int64_t i, const SEd& dst, int64_t j, bool with_l) {
    k_move_fields<<<1, 128, 0, ctx->stream>>>(
        MoveSpec{{src.e + i * D * D, src.g + i * D, with_l ? src.l + i * D * D : nullptr, nullptr, nullptr},
                 {dst.e + j * D * D, dst.g + j * D, with_l ? dst.l + j * D * D : nullptr, nullptr, nullptr},
                 {D * D, D, with_l ? D * D : 0, 0, 0}, with_l ? 3 : 2});
    note_launch(ctx, "move");
  }

  // All-gather of one contiguous device element (count doubles) from every
  // shard; the R copies land contiguously in dev_all (rank order).  With an
  // NCCL communicator on the context (pode_context_nccl_init) the exchange
  // stays on the device (ncclAllGather on the context stream); otherwise it
  // goes through the caller's host all-gather callback.
  static void gather(pode_context* ctx, const pode_shard_comm& comm, const double* dev_own, int64_t count,
                     double* dev_all, std::vector<double>* host_all = nullptr) {
    if (ctx->nccl_comm) {
      double* recv = dev_all ? dev_all : ctx->ws.arr<double>("sh_recv", size_t(count) * comm.ranks);
      nccl::all_gather(ctx, dev_own, count, recv);
      if (host_all) {  // the stopping scalars: the decision is taken on the host
        host_all->resize(size_t(count) * comm.ranks);
        cuda_check(cudaMemcpyAsync(host_all->data(), recv, sizeof(double) * host_all->size(), cudaMemcpyDeviceToHost,
                                   ctx->stream),
                   "shard scalars");
        cuda_check(cudaStreamSynchronize(ctx->stream), "shard sync");
      }
      return;
    }
    std::vector<double> send(static_cast<size_t>(count)), recv(static_cast<size_t>(count) * comm.ranks);
    cuda_check(cudaMemcpyAsync(send.data(), dev_own, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream),
               "shard send");
    cuda_check(cudaStreamSynchronize(ctx->stream), "shard sync");
    if (comm.allgather == nullptr || comm.allgather(comm.user, send.data(), count, recv.data()) != 0)
      throw ApiError(PODE_ERR_INVALID_INPUT, "ieks_sharded: all-gather failed");
    if (dev_all)
      cuda_check(cudaMemcpyAsync(dev_all, recv.data(), sizeof(double) * recv.size(), cudaMemcpyHostToDevice,
                                 ctx->stream),
                 "shard recv");
    cuda_check(cudaStreamSynchronize(ctx->stream), "shard sync");
    if (host_all) *host_all = std::move(recv);
  }

  // Fixed-order fold of the gathered scalars (sum, max, max) of every shard.
  static void gather3(pode_context* ctx, const pode_shard_comm& comm, const double* dev3, double (&out)[3],
                      bool& any_failed, bool own_failed) {
    double* tmp = ctx->ws.arr<double>("sh_s3", 4);
    cuda_check(cudaMemcpyAsync(tmp, dev3, sizeof(double) * 3, cudaMemcpyDeviceToDevice, ctx->stream), "s3");
    k_set_scalar<<<1, 1, 0, ctx->stream>>>(tmp + 3, own_failed ? 1.0 : 0.0);
    note_launch(ctx, "flag");
    std::vector<double> all;
    gather(ctx, comm, tmp, 4, nullptr, &all);
    out[0] = 0.0;
    out[1] = 0.0;
    out[2] = 0.0;
    any_failed = false;
    for (int r = 0; r < comm.ranks; ++r) {
      out[0] += all[size_t(r) * 4 + 0];
      out[1] = std::max(out[1], all[size_t(r) * 4 + 1]);
      out[2] = std::max(out[2], all[size_t(r) * 4 + 2]);
      any_failed |= all[size_t(r) * 4 + 3] != 0.0;
    }
  }

  // para_ieks over the time-axis shard `comm.rank`: the same
  // passes on the local steps, plus three exchanges per iteration (forward
  // aggregate -> Gaussian carry, backward aggregate -> right mean carry,
  // stopping scalars).  Per-iteration host loop (the exchanges are host
  // collectives).
  static IeksResult run_sharded(pode_context* ctx, const host::Problem& p, const pode_prior& prior,
                                const double* grid_h, int64_t n1g, const pode_ieks_config& cfg,
                                const pode_shard_comm& comm, double* means, double* cov, double* sol_m,
                                double* sol_c) {
    using IE = IeksEngine<D>;
    set_attrs();
    const int R = comm.ranks, rank = comm.rank;
    IeksSetup<D> s;
    IE::setup(ctx, p, prior, grid_h, n1g, s, false);
    cudaStream_t st = ctx->stream;
    Workspace& ws = ctx->ws;
    const int64_t Ng = s.N;
    const int64_t g0 = shard_first_step(Ng, rank, R);
    const int64_t N = shard_first_step(Ng, rank + 1, R) - g0;  // local steps
    if (N < 1) throw ApiError(PODE_ERR_INVALID_INPUT, "ieks_sharded: fewer steps than shards");
    const int L = chunk_len(ctx, N);
    const int64_t nc = (N + L - 1) / L;
    FastConst<D> cst;
    std::memcpy(cst.q, s.h_q.data(), sizeof(cst.q));
    std::memcpy(cst.qunit, s.h_qunit.data(), sizeof(cst.qunit));
    std::memcpy(cst.qunit_rdiag, s.h_qinv.data(), sizeof(cst.qunit_rdiag));
    std::memcpy(cst.m0, s.h_m0.data(), sizeof(cst.m0));
    const size_t padded = size_t(nc) * L;
    double* eta_a = ws.arr<double>("lane_eta_a", padded * D + D);
    double* eta_b = ws.arr<double>("lane_eta_b", padded * D + D);
    FEd agg = Engine<D>::template alloc<FOps<D>>(ctx, "fast_agg", nc);
    lane::ElemSoA soa;
    {
      double* base = ws.arr<double>("fast_elems", padded * (D * D + D) + D);
      soa = lane::ElemSoA{base, base + padded * D * D, base + padded * (D * D + D), nc, L};
    }
    SEd bagg = Engine<D>::template alloc<MOps<D>>(ctx, "sh_bagg", nc);
    const unsigned lblocks = static_cast<unsigned>((nc + lane::kLaneThreads - 1) / lane::kLaneThreads);
    const int64_t nparts = int64_t(lblocks);
    double* part = ws.arr<double>("fast_part", nparts * 3 + 3);
    double* red = part + nparts * 3;
    const unsigned th = lane::kLaneThreads;
    auto term = [&](double* base) { return base + padded * D; };
    // exchange buffers: R gathered elements + own element + carry (b, C)
    double* xf = ws.arr<double>("sh_xf", size_t(R + 2) * kFel);
    double* xs = ws.arr<double>("sh_xs", size_t(R + 2) * kSel);
    double* carry = ws.arr<double>("sh_carry", D + D * D);
    FastArgs a{s.grid + g0, eta_a, term(eta_a), N, L, nc, cfg.linearization, s.prob,
               reinterpret_cast<DevError*>(ctx->d_err)};
    a.first = rank == 0 ? 1 : 0;
    a.last = rank == R - 1 ? 1 : 0;
    a.carry = carry;

    // forward exchange, at the top of the local aggregate scan's up-sweep:
    // the local total (the last top prefix) is all-gathered, shard r folds
    // t_0 ⊗ .. ⊗ t_{r-1} (Gaussian: t_0 absorbed the prior) into `carry`,
    // and the scan's down-sweeps apply it (Engine::scan_filtering_gauss_shard;
    // no separate reduction of the aggregates)
    const typename Engine<D>::TopHook forward_top = [&](FEd full, int64_t ntop) {
      double* own = xf + size_t(R) * kFel;
      fel_move(ctx, full, ntop - 1, fview(own), 0);
      gather(ctx, comm, own, kFel, xf);
      if (rank == 0) return;
      for (int i = 1; i < rank; ++i)
        Engine<D>::template combine_one<FOps<D>>(ctx, fview(xf), fview(xf + size_t(i) * kFel), fview(xf));
      d2d(ctx, carry, fview(xf).b, D);
      d2d(ctx, carry + D, fview(xf).c, D * D);
    };
    // backward exchange, at the top of the local mean scan's up-sweep: the
    // local (E, g) total is all-gathered, shard r folds t_{r+1} ⊗ .. ⊗
    // t_{R-1} from the right (E = 0: the last shard absorbed the terminal)
    // into the smoothed mean at its halo node (elems.term), which the scan's
    // down-sweeps apply to its last block at every level
    const typename Engine<D>::MTopHook backward_top = [&](SEd full, int64_t) {
      double* own = xs + size_t(R) * kSel;
      sel_move(ctx, full, 0, sview(own), 0, false);
      gather(ctx, comm, own, kSel, xs);
      if (rank == R - 1) return;
      double* acc = xs + size_t(R - 1) * kSel;
      for (int i = R - 2; i > rank; --i)
        Engine<D>::template combine_one<MOps<D>>(ctx, sview(xs + size_t(i) * kSel), sview(acc), sview(acc));
      d2d(ctx, soa.term, sview(acc).g, D);
    };

    lane::k_eta_fill<D><<<lane::eta_fill_grid(nc, L, D), 256, 0, st>>>(s.mu0, nc, L, eta_a);
    note_launch(ctx, "fill");
    reset_error(ctx);
    // objective of the constant start (ieks.cpp:147-148)
    lane::k_lane_bwd_down<D, d, true><<<lblocks, th, 0, st>>>(a, cst, soa, bagg, eta_a, term(eta_a), eta_b,
                                                               term(eta_b), part);
    note_launch(ctx, "fast_objective");
    k_finish3<<<1, kRedThreads, 0, st>>>(part, nparts, red);
    note_launch(ctx, "finish3");
    double r3[3];
    bool any_failed = false;
    gather3(ctx, comm, red, r3, any_failed, false);
    double v_prev = 0.5 * r3[0];

    IeksResult res;
    int it = 0;
    while (it < cfg.max_iterations) {
      ++it;
      reset_error(ctx);
      a.eta = eta_a;
      a.eta_term = term(eta_a);
      lane::k_lane_fwd_reduce<D, d><<<lblocks, th, lane::fwd_reduce_smem<D>(), st>>>(a, cst, agg);
      note_launch(ctx, "fast_fwd_reduce");
      const ScanTally tf = Engine<D>::scan_filtering_gauss_shard(ctx, nc, agg, scan_fanin(), forward_top,
                                                                 rank == 0 ? nullptr : carry);
      lane::k_lane_fwd_down<D, d><<<lblocks, th, lane::fwd_down_smem<D>(), st>>>(a, cst, agg, soa, nullptr, nullptr,
                                                                                nullptr, bagg);
      note_launch(ctx, "fast_fwd_down");
      const ScanTally tr = Engine<D>::scan_means_terminal_shard(ctx, nc, bagg, scan_fanin(), backward_top,
                                                                rank == R - 1 ? nullptr : soa.term);
      lane::k_lane_bwd_down<D, d, false><<<lblocks, th, 0, st>>>(a, cst, soa, bagg, eta_a, term(eta_a), eta_b,
                                                                  term(eta_b), part);
      note_launch(ctx, "fast_bwd_down");
      k_finish3<<<1, kRedThreads, 0, st>>>(part, nparts, red);
      note_launch(ctx, "finish3");
      const unsigned long long key = fetch_error(ctx);
      gather3(ctx, comm, red, r3, any_failed, key != ~0ull);
      if (key != ~0ull) IE::check_linearization(ctx, s, it, g0);  // throws this shard's error
      if (any_failed) throw ApiError(PODE_ERR_SINGULAR_FACTOR, "ieks_sharded: another shard failed", 0, 0.0, it);
      res.stats.combines = std::max(res.stats.combines, (Ng - nc * R) + tf.combines * R + Ng);
      res.stats.depth = std::max(res.stats.depth, int64_t(L) + tf.depth + int64_t(L) + tr.depth + 2 * R);
      const double v = 0.5 * r3[0];
      res.trace.push_back(v);
      const bool conv = (r3[1] <= cfg.traj_rtol * r3[2]) ||
                        (std::fabs(v - v_prev) <= cfg.obj_atol + cfg.obj_rtol * std::fabs(v));
      std::swap(eta_a, eta_b);
      v_prev = v;
      if (conv) {
        res.converged = true;
        break;
      }
    }
    res.iterations = it;

    // finalize on the shard (eta_a: newest trajectory, eta_b: linearisation point)
    a.eta = eta_b;
    a.eta_term = term(eta_b);
    double* cf = ws.arr<double>("fin_cf", padded * D * D + D * D);
    double* cterm = cf + padded * D * D;
    reset_error(ctx);
    lane::k_lane_fwd_down<D, d, true><<<lblocks, th, 0, st>>>(a, cst, agg, soa, cf, cterm, part);
    note_launch(ctx, "fin_fwd");
    k_finish3<<<1, kRedThreads, 0, st>>>(part, lblocks, red);
    note_launch(ctx, "finish3");
    {
      const unsigned long long key = fetch_error(ctx);
      gather3(ctx, comm, red, r3, any_failed, key != ~0ull);
      if (key != ~0ull) IE::check_linearization(ctx, s, it, g0);
      if (any_failed) throw ApiError(PODE_ERR_SINGULAR_FACTOR, "ieks_sharded: another shard failed", 0, 0.0, it);
    }
    const double innov = r3[0];
    cuda_check(cudaMemcpyAsync(red, &innov, sizeof(double), cudaMemcpyHostToDevice, st), "innov");
    SEd sagg = Engine<D>::template alloc<SOps<D>>(ctx, "fin_sagg", nc);
    lane::k_lane_fin_fold<D, d><<<lblocks, th, 0, st>>>(a, cst, soa, cf, cterm, sagg);
    note_launch(ctx, "fin_fold");
    {  // right carry of the full smoothing aggregates: (E = 0, g, L) at the halo node
      const SEd tot = Engine<D>::template reduce_total<SOps<D>>(ctx, sagg, nc, "sh_sred_");
      double* own = xs + size_t(R) * kSel;
      sel_move(ctx, tot, 0, sview(own), 0, true);
      gather(ctx, comm, own, kSel, xs);
      if (rank < R - 1) {
        double* acc = xs + size_t(R - 1) * kSel;
        for (int i = R - 2; i > rank; --i)
          Engine<D>::template combine_one<SOps<D>>(ctx, sview(xs + size_t(i) * kSel), sview(acc), sview(acc));
        double* tmp = xs + size_t(R + 1) * kSel;
        sel_move(ctx, sagg, nc - 1, sview(tmp), 0, true);
        Engine<D>::template combine_one<SOps<D>>(ctx, sview(tmp), sview(acc), sview(tmp));
        sel_move(ctx, sview(tmp), 0, sagg, nc - 1, true);
        d2d(ctx, cterm, sview(acc).l, D * D);
      }
    }
    Engine<D>::scan_smoothing(ctx, nc, sagg, sagg, true);
    const double count = double(Ng) * s.dim;
    lane::k_lane_fin_bwd<D, d><<<lblocks, th, 0, st>>>(a, cst, soa, cf, cterm, sagg, eta_a, term(eta_a), red, count,
                                                       lane::FinOut{means, cov, sol_m, sol_c});
    note_launch(ctx, "fin_bwd");
    IE::check_linearization(ctx, s, it, g0);  // syncs
    res.sigma_hat = std::sqrt(innov / count) * prior.sigma;
    return res;
  }

  // Lane finalize at the final linearisation point (the last iteration's
  // pass-B prefixes in `agg` are still valid for it): F1 filter + C_f(k) +
  // innovations, F2 chunk smoothing aggregates (E, g, L), a reverse ⊗_s scan
  // of the aggregates, F4 smoothed factors fused with the outputs.
  static void finalize(pode_context* ctx, const IeksSetup<D>& s, FastArgs a, const FastConst<D>& cst, const FEd& agg,
                       const lane::ElemSoA& soa, const double* eta_out, const double* eta_out_term,
                       const double* eta_lin, const double* eta_lin_term, double sigma, int it,
                       const lane::FinOut& out, IeksResult& res) {
    cudaStream_t st = ctx->stream;
    Workspace& ws = ctx->ws;
    const int64_t nc = a.nchunks;
    const size_t padded = size_t(nc) * a.L;
    double* cf = ws.arr<double>("fin_cf", padded * D * D + D * D);
    double* cterm = cf + padded * D * D;
    NvtxRange nv("finalize_covariances_outputs");
    const unsigned lblocks = Pass::blocks(nc);
    double* part = ws.arr<double>("fin_part", size_t(lblocks) * 3 + 3);
    double* red = part + size_t(lblocks) * 3;
    a.eta = eta_lin;
    a.eta_term = eta_lin_term;
    reset_error(ctx);
    Pass::fin_fwd(st, a, cst, agg, soa, cf, cterm, part);
    note_launch(ctx, "fin_fwd");
    k_finish3<<<1, kRedThreads, 0, st>>>(part, lblocks, red);
    note_launch(ctx, "finish3");
    IeksEngine<D>::check_linearization(ctx, s, it);  // syncs the stream
    SEd sagg = Engine<D>::template alloc<SOps<D>>(ctx, "fin_sagg", nc);
    Pass::fin_fold(st, a, cst, soa, cf, cterm, sagg);
    note_launch(ctx, "fin_fold");
    const ScanTally t = Engine<D>::scan_smoothing(ctx, nc, sagg, sagg, true);
    res.stats.combines = std::max(res.stats.combines, a.N + t.combines);
    const double count = double(a.N) * s.dim;
    Pass::fin_bwd(st, a, cst, soa, cf, cterm, sagg, eta_out, eta_out_term, red, count, out);
    note_launch(ctx, "fin_bwd");
    cuda_check(cudaMemcpyAsync(ctx->h_scalars, red, sizeof(double), cudaMemcpyDeviceToHost, st), "innov");
    IeksEngine<D>::check_linearization(ctx, s, it);  // syncs the stream
    res.sigma_hat = std::sqrt(ctx->h_scalars[0] / count) * sigma;
  }
};

}  // namespace pode
