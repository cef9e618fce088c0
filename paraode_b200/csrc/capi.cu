// The C ABI (include/paraode_b200.h): context management, host<->device
// staging, dispatch to the per-D engines and the mapping of device error
// words onto the reference's exception types.
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "dispatch.hpp"
#include "engine.cuh"
#include "host_model.hpp"
#include "field.cuh"
#include "ieks.cuh"
#include "nccl.hpp"

namespace pode {

#define PODE_DECL(n) const EngineOps* engine_ops_d##n();
PODE_DECL(1) PODE_DECL(2) PODE_DECL(3) PODE_DECL(4) PODE_DECL(5) PODE_DECL(6) PODE_DECL(7) PODE_DECL(8)
PODE_DECL(9) PODE_DECL(10) PODE_DECL(11) PODE_DECL(12) PODE_DECL(13) PODE_DECL(14) PODE_DECL(15) PODE_DECL(16)
#undef PODE_DECL

const EngineOps* engine_ops(int D) {
  switch (D) {
    case 1: return engine_ops_d1();
    case 2: return engine_ops_d2();
    case 3: return engine_ops_d3();
    case 4: return engine_ops_d4();
    case 5: return engine_ops_d5();
    case 6: return engine_ops_d6();
    case 7: return engine_ops_d7();
    case 8: return engine_ops_d8();
    case 9: return engine_ops_d9();
    case 10: return engine_ops_d10();
    case 11: return engine_ops_d11();
    case 12: return engine_ops_d12();
    case 13: return engine_ops_d13();
    case 14: return engine_ops_d14();
    case 15: return engine_ops_d15();
    case 16: return engine_ops_d16();
    default: return nullptr;
  }
}

void reset_error(pode_context* ctx) {
  cuda_check(cudaMemsetAsync(ctx->d_err, 0xff, sizeof(unsigned long long), ctx->stream), "reset error word");
}

unsigned long long fetch_error(pode_context* ctx) {
  cuda_check(cudaMemcpyAsync(ctx->h_err, ctx->d_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             ctx->stream),
             "fetch error word");
  cuda_check(cudaStreamSynchronize(ctx->stream), "stream sync");
  prof_mark(ctx);
  return *ctx->h_err;
}

namespace {

const EngineOps& ops_for(int D) {
  const EngineOps* ops = engine_ops(D);
  if (ops == nullptr)
    throw ApiError(PODE_ERR_UNSUPPORTED, "state dimension " + std::to_string(D) + " is outside the compiled range [" +
                                             std::to_string(kMinD) + ", " + std::to_string(kMaxD) + "]");
  return *ops;
}

void check_ctx(pode_context* ctx) {
  if (ctx == nullptr) throw ApiError(PODE_ERR_INVALID_INPUT, "NULL context");
  cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
}

// Raises the device error word (if set) as the matching ApiError.
void raise_device_error(pode_context* ctx, const char* stage, int scan_code = 0) {
  const unsigned long long key = fetch_error(ctx);
  if (key == ~0ull) return;
  const int code = int(key & 0xff);
  const int64_t idx = int64_t(key >> 8);
  if (scan_code) {
    ApiError e(PODE_ERR_SCAN,
               std::string("associative_scan: combine failed on elements [") + std::to_string(idx) + ", " +
                   std::to_string(idx) + "]: " + stage + ": triangular factor is singular",
               idx);
    throw e;
  }
  if (code == kErrLinearization)
    throw ApiError(PODE_ERR_LINEARIZATION, std::string(stage) + ": vector field evaluation is not finite", idx);
  if (code == kErrInvalid) throw ApiError(PODE_ERR_INVALID_INPUT, std::string(stage) + ": non-finite input", idx);
  throw ApiError(PODE_ERR_SINGULAR_FACTOR, std::string(stage) + ": triangular factor is singular", idx);
}

template <typename F>
int guarded(pode_status* st, F&& f) {
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->index = -1;
  }
  try {
    f();
    return PODE_OK;
  } catch (const ApiError& e) {
    if (st) {
      st->code = e.code;
      st->index = e.index;
      st->lo = st->hi = e.index;
      st->time = e.time;
      st->iteration = e.iteration;
      std::strncpy(st->msg, e.what(), sizeof(st->msg) - 1);
    }
    return e.code;
  } catch (const std::exception& e) {
    if (st) {
      st->code = PODE_ERR_CUDA;
      std::strncpy(st->msg, e.what(), sizeof(st->msg) - 1);
    }
    return PODE_ERR_CUDA;
  }
}

// Copies host arrays into a tagged workspace buffer (or passes device
// pointers through).
template <typename T>
T* stage_in(pode_context* ctx, const std::string& tag, const T* src, size_t count, bool device) {
  if (src == nullptr) return nullptr;
  if (device) return const_cast<T*>(src);
  T* d = ctx->ws.arr<T>(tag, count);
  cuda_check(cudaMemcpyAsync(d, src, sizeof(T) * count, cudaMemcpyHostToDevice, ctx->stream), tag.c_str());
  return d;
}

// Large device->host copies into caller (pageable) memory: DMA into a pinned
// two-slot staging ring while host threads copy the previous slot out (the
// caller's first-touch page faults are taken in parallel, not by the DMA
// engine's pageable path).
constexpr size_t kStageBytes = size_t(32) << 20;

// Classical RK4 on a uniform grid by one thread (the accuracy reference of
// the benchmark harness, problems.cpp:11-27; autonomous registered fields).
constexpr int kRk4MaxDim = 28;

template <int DMAX>
__global__ void k_rk4(DevProblem prob, double t_end, int64_t steps, const double* y0, double* table, int* bad) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int d = prob.dim;
  double y[DMAX], k1[DMAX], k2[DMAX], k3[DMAX], k4[DMAX], tmp[DMAX], jac[DMAX * DMAX];
  for (int i = 0; i < d; ++i) table[i] = y[i] = y0[i];
  const double h = t_end / double(steps);
  bool finite = true;
  for (int64_t n = 0; n < steps; ++n) {
    eval_field<DMAX>(prob, y, k1, jac);
    for (int i = 0; i < d; ++i) tmp[i] = y[i] + (0.5 * h) * k1[i];
    eval_field<DMAX>(prob, tmp, k2, jac);
    for (int i = 0; i < d; ++i) tmp[i] = y[i] + (0.5 * h) * k2[i];
    eval_field<DMAX>(prob, tmp, k3, jac);
    for (int i = 0; i < d; ++i) tmp[i] = y[i] + h * k3[i];
    eval_field<DMAX>(prob, tmp, k4, jac);
    for (int i = 0; i < d; ++i) {
      y[i] += (h / 6.0) * (((k1[i] + 2.0 * k2[i]) + 2.0 * k3[i]) + k4[i]);
      finite &= isfinite(y[i]);
      table[(n + 1) * d + i] = y[i];
    }
  }
  if (!finite) *bad = 1;
}

void copy_out_staged(pode_context* ctx, char* dst, const char* dev, size_t bytes) {
  cudaStream_t st = ctx->stream;
  for (int k = 0; k < 2; ++k) {
    if (ctx->h_stage[k] == nullptr) {
      cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_stage[k]), kStageBytes, cudaHostAllocDefault),
                 "staging");
      cuda_check(cudaEventCreateWithFlags(&ctx->stage_ev[k], cudaEventDisableTiming), "staging event");
    }
  }
  const size_t n = (bytes + kStageBytes - 1) / kStageBytes;
  auto issue = [&](size_t i) {
    const size_t off = i * kStageBytes, len = std::min(kStageBytes, bytes - off);
    cuda_check(cudaMemcpyAsync(ctx->h_stage[i & 1], dev + off, len, cudaMemcpyDeviceToHost, st), "copy out");
    cuda_check(cudaEventRecord(ctx->stage_ev[i & 1], st), "copy out event");
  };
  issue(0);
  if (n > 1) issue(1);
  const int threads = std::max(1, std::min(8, omp_get_max_threads()));
  for (size_t i = 0; i < n; ++i) {
    cuda_check(cudaEventSynchronize(ctx->stage_ev[i & 1]), "copy out wait");
    const size_t off = i * kStageBytes, len = std::min(kStageBytes, bytes - off);
    const char* src = ctx->h_stage[i & 1];
    const size_t per = (len + threads - 1) / threads;
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int t = 0; t < threads; ++t) {
      const size_t lo = size_t(t) * per;
      if (lo < len) std::memcpy(dst + off + lo, src + lo, std::min(per, len - lo));
    }
    if (i + 2 < n) issue(i + 2);
  }
}

template <typename T>
void stage_out(pode_context* ctx, T* dst, const T* dev, size_t count, bool device) {
  if (dst == nullptr || device) return;
  const size_t bytes = sizeof(T) * count;
  cudaPointerAttributes attr{};
  const bool pinned = cudaPointerGetAttributes(&attr, dst) == cudaSuccess && attr.type == cudaMemoryTypeHost;
  cudaGetLastError();  // clear a failed query on plain pageable memory
  if (!pinned && bytes >= (size_t(4) << 20)) {
    copy_out_staged(ctx, reinterpret_cast<char*>(dst), reinterpret_cast<const char*>(dev), bytes);
    return;
  }
  cuda_check(cudaMemcpyAsync(dst, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream), "copy out");
}

void check_dims(int D, int64_t count) {
  if (D < 1) throw ApiError(PODE_ERR_DIMENSION, "state dimension must be >= 1");
  if (count < 0) throw ApiError(PODE_ERR_DIMENSION, "negative count");
}

DevChain stage_chain(pode_context* ctx, const pode_chain* c) {
  if (c == nullptr) throw ApiError(PODE_ERR_INVALID_INPUT, "NULL chain");
  if (c->steps < 1) throw ApiError(PODE_ERR_DIMENSION, "smoother: need N >= 1 aligned transitions and observations");
  const int D = c->state_dim, M = c->obs_rows_max;
  if (D < 1 || M < 0 || M > D) throw ApiError(PODE_ERR_DIMENSION, "chain: need 0 <= obs_rows_max <= state_dim");
  const bool dev = c->location == PODE_DEVICE;
  const int64_t N = c->steps;
  const int Mm = std::max(M, 1);
  if (!dev) {
    for (int64_t n = 0; n < N; ++n)
      if (c->obs_rows[n] < 0 || c->obs_rows[n] > M)
        throw ApiError(PODE_ERR_DIMENSION, "smoother: observation dimensions disagree with the state", n);
  }
  DevChain ch;
  ch.D = D;
  ch.M = Mm;
  ch.N = N;
  ch.init_mean = stage_in(ctx, "ch_init_mean", c->init_mean, D, dev);
  ch.init_cov = stage_in(ctx, "ch_init_cov", c->init_cov_sqrt, size_t(D) * D, dev);
  ch.phi_shared = c->phi_shared;
  ch.q_shared = c->q_shared;
  ch.phi = stage_in(ctx, "ch_phi", c->phi, size_t(c->phi_shared ? 1 : N) * D * D, dev);
  ch.q = stage_in(ctx, "ch_q", c->q_sqrt, size_t(c->q_shared ? 1 : N) * D * D, dev);
  ch.obs_rows = stage_in(ctx, "ch_rows", c->obs_rows, size_t(N), dev);
  if (M == 0) {
    // no observation rows anywhere: give the kernels valid zero buffers
    double* z = ctx->ws.arr<double>("ch_zero", size_t(N) * (D + 2));
    cuda_check(cudaMemsetAsync(z, 0, sizeof(double) * size_t(N) * (D + 2), ctx->stream), "zero");
    ch.h = z;
    ch.off = z + size_t(N) * D;
    ch.r = z + size_t(N) * (D + 1);
  } else {
    ch.h = stage_in(ctx, "ch_h", c->h, size_t(N) * M * D, dev);
    ch.off = stage_in(ctx, "ch_off", c->offset, size_t(N) * M, dev);
    ch.r = stage_in(ctx, "ch_r", c->r_sqrt, size_t(N) * M * M, dev);
  }
  return ch;
}

FEd fe_view(const pode_filtering_elements& e) { return FEd{e.a, e.b, e.c_sqrt, e.eta, e.j_sqrt}; }
SEd se_view(const pode_smoothing_elements& e) { return SEd{e.e, e.g, e.l_sqrt}; }

FEd stage_fe(pode_context* ctx, const std::string& tag, const pode_filtering_elements& e, int64_t n, int D,
             bool dev, bool copy) {
  if (dev) return fe_view(e);
  const size_t mm = size_t(n) * D * D, vv = size_t(n) * D;
  double* base = ctx->ws.arr<double>(tag, 3 * mm + 2 * vv);
  FEd d{base, base + mm, base + mm + vv, base + 2 * mm + vv, base + 2 * mm + 2 * vv};
  if (copy) {
    cuda_check(cudaMemcpyAsync(d.a, e.a, sizeof(double) * mm, cudaMemcpyHostToDevice, ctx->stream), "a");
    cuda_check(cudaMemcpyAsync(d.b, e.b, sizeof(double) * vv, cudaMemcpyHostToDevice, ctx->stream), "b");
    cuda_check(cudaMemcpyAsync(d.c, e.c_sqrt, sizeof(double) * mm, cudaMemcpyHostToDevice, ctx->stream), "c");
    cuda_check(cudaMemcpyAsync(d.eta, e.eta, sizeof(double) * vv, cudaMemcpyHostToDevice, ctx->stream), "eta");
    cuda_check(cudaMemcpyAsync(d.j, e.j_sqrt, sizeof(double) * mm, cudaMemcpyHostToDevice, ctx->stream), "j");
  }
  return d;
}

void unstage_fe(pode_context* ctx, const pode_filtering_elements& e, const FEd& d, int64_t n, int D, bool dev) {
  if (dev) return;
  const size_t mm = size_t(n) * D * D, vv = size_t(n) * D;
  stage_out(ctx, e.a, d.a, mm, false);
  stage_out(ctx, e.b, d.b, vv, false);
  stage_out(ctx, e.c_sqrt, d.c, mm, false);
  stage_out(ctx, e.eta, d.eta, vv, false);
  stage_out(ctx, e.j_sqrt, d.j, mm, false);
}

SEd stage_se(pode_context* ctx, const std::string& tag, const pode_smoothing_elements& e, int64_t n, int D,
             bool dev, bool copy) {
  if (dev) return se_view(e);
  const size_t mm = size_t(n) * D * D, vv = size_t(n) * D;
  double* base = ctx->ws.arr<double>(tag, 2 * mm + vv);
  SEd d{base, base + mm, base + mm + vv};
  if (copy) {
    cuda_check(cudaMemcpyAsync(d.e, e.e, sizeof(double) * mm, cudaMemcpyHostToDevice, ctx->stream), "e");
    cuda_check(cudaMemcpyAsync(d.g, e.g, sizeof(double) * vv, cudaMemcpyHostToDevice, ctx->stream), "g");
    cuda_check(cudaMemcpyAsync(d.l, e.l_sqrt, sizeof(double) * mm, cudaMemcpyHostToDevice, ctx->stream), "l");
  }
  return d;
}

void unstage_se(pode_context* ctx, const pode_smoothing_elements& e, const SEd& d, int64_t n, int D, bool dev) {
  if (dev) return;
  const size_t mm = size_t(n) * D * D, vv = size_t(n) * D;
  stage_out(ctx, e.e, d.e, mm, false);
  stage_out(ctx, e.g, d.g, vv, false);
  stage_out(ctx, e.l_sqrt, d.l, mm, false);
}

void sync(pode_context* ctx) { cuda_check(cudaStreamSynchronize(ctx->stream), "stream sync"); }

}  // namespace
}  // namespace pode

using namespace pode;

extern "C" {

int pode_context_create(int32_t device, pode_context** out, pode_status* status) {
  return guarded(status, [&] {
    if (out == nullptr) throw ApiError(PODE_ERR_INVALID_INPUT, "NULL out");
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw ApiError(PODE_ERR_CUDA, "no CUDA device visible (paraode_b200 has no CPU fallback)");
    if (device < 0 || device >= count) throw ApiError(PODE_ERR_CUDA, "device index out of range");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop{};
    cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10)
      throw ApiError(PODE_ERR_CUDA, std::string("paraode_b200 is built for sm_100a (B200); found ") + prop.name);
    auto* ctx = new pode_context();
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    try {
      cuda_check(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
      cuda_check(cudaMalloc(&ctx->d_err, sizeof(unsigned long long)), "error word");
      cuda_check(cudaMallocHost(&ctx->h_err, sizeof(unsigned long long)), "pinned");
      cuda_check(cudaMallocHost(&ctx->h_scalars, sizeof(double) * 16), "pinned");
      reset_error(ctx);
      sync(ctx);
    } catch (...) {
      pode_context_destroy(ctx);
      throw;
    }
    *out = ctx;
  });
}

void pode_context_destroy(pode_context* ctx) {
  if (ctx == nullptr) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  nccl::destroy(ctx);
  for (auto& kv : ctx->graphs) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
  }
  ctx->graphs.clear();
  for (auto& kv : ctx->ws.bufs)
    if (kv.second.ptr) cudaFree(kv.second.ptr);
  ctx->ws.bufs.clear();
  for (int k = 0; k < 2; ++k) {
    if (ctx->h_stage[k]) cudaFreeHost(ctx->h_stage[k]);
    if (ctx->stage_ev[k]) cudaEventDestroy(ctx->stage_ev[k]);
  }
  if (ctx->d_err) cudaFree(ctx->d_err);
  if (ctx->h_err) cudaFreeHost(ctx->h_err);
  if (ctx->h_scalars) cudaFreeHost(ctx->h_scalars);
  for (cudaEvent_t e : ctx->prof_pool) cudaEventDestroy(e);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int32_t pode_max_state_dim(void) { return 112; }  // the large-state engine (big.cuh) above kMaxD

int pode_profile(pode_context* ctx, int32_t enable) {
  if (ctx == nullptr) return PODE_ERR_INVALID_INPUT;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->prof.clear();
  ctx->prof_used = 0;
  ctx->prof_on = enable != 0;
  if (ctx->prof_on) prof_mark(ctx);
  return PODE_OK;
}

int64_t pode_profile_read(pode_context* ctx, char* buf, int64_t size) {
  if (ctx == nullptr) return -1;
  cudaSetDevice(ctx->device);
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return -1;
  std::map<std::string, std::pair<int64_t, double>> agg;
  for (size_t i = 1; i < ctx->prof.size(); ++i) {
    if (ctx->prof[i].name == nullptr) continue;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->prof[i - 1].ev, ctx->prof[i].ev) != cudaSuccess) continue;
    auto& a = agg[ctx->prof[i].name];
    a.first += 1;
    a.second += ms;
  }
  std::string out;
  for (const auto& kv : agg) {
    char line[256];
    std::snprintf(line, sizeof(line), "%s %lld %.6f\n", kv.first.c_str(), static_cast<long long>(kv.second.first),
                  kv.second.second);
    out += line;
  }
  if (buf != nullptr && size > 0) {
    const size_t n = std::min<size_t>(out.size(), size_t(size - 1));
    std::memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return int64_t(out.size());
}

int64_t pode_kernel_launches(const pode_context* ctx) { return ctx ? ctx->launches : 0; }

void* pode_context_stream(pode_context* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int pode_nccl_unique_id(const char* nccl_path, uint8_t id[128], pode_status* status) {
  return guarded(status, [&] {
    if (id == nullptr) throw ApiError(PODE_ERR_INVALID_INPUT, "NULL id");
    nccl::UniqueId u;
    nccl::check(nccl::api(nccl_path).get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, sizeof(u.internal));
  });
}

int pode_context_nccl_init(pode_context* ctx, const char* nccl_path, const uint8_t id[128], int32_t rank,
                           int32_t ranks, pode_status* status) {
  return guarded(status, [&] {
    check_ctx(ctx);
    if (id == nullptr || ranks < 1 || rank < 0 || rank >= ranks)
      throw ApiError(PODE_ERR_INVALID_INPUT, "nccl_init: need an id and 0 <= rank < ranks");
    nccl::Api& a = nccl::api(nccl_path);
    nccl::destroy(ctx);
    nccl::UniqueId u;
    std::memcpy(u.internal, id, sizeof(u.internal));
    nccl::Comm comm = nullptr;
    nccl::check(a.comm_init_rank(&comm, ranks, u, rank), "ncclCommInitRank");
    ctx->nccl_comm = comm;
    ctx->nccl_rank = rank;
    ctx->nccl_ranks = ranks;
  });
}

int pode_context_set_option(pode_context* ctx, int32_t option, int64_t value) {
  if (ctx == nullptr) return PODE_ERR_INVALID_INPUT;
  switch (option) {
    case PODE_OPT_CHUNK_LEN:
      if (value < 0) return PODE_ERR_INVALID_INPUT;
      ctx->opt_chunk = value;
      return PODE_OK;
    case PODE_OPT_ENGINE:
      if (value < 0 || value > 2) return PODE_ERR_INVALID_INPUT;
      ctx->opt_engine = int(value);
      return PODE_OK;
    default:
      return PODE_ERR_INVALID_INPUT;
  }
}

int pode_combine_filtering(pode_context* ctx, int64_t count, int32_t D, pode_filtering_elements lhs,
                           pode_filtering_elements rhs, pode_filtering_elements out, int32_t location,
                           pode_status* status) {
  return guarded(status, [&] {
    check_ctx(ctx);
    check_dims(D, count);
    if (count == 0) return;
    const auto& ops = ops_for(D);
    const bool dev = location == PODE_DEVICE;
    const FEd l = stage_fe(ctx, "cf_l", lhs, count, D, dev, true);
    const FEd r = stage_fe(ctx, "cf_r", rhs, count, D, dev, true);
    const FEd o = stage_fe(ctx, "cf_o", out, count, D, dev, false);
    reset_error(ctx);
    ops.combine_filtering(ctx, count, l, r, o);
    unstage_fe(ctx, out, o, count, D, dev);
    raise_device_error(ctx, "combine_filtering: combination factor");
  });
}

int pode_combine_smoothing(pode_context* ctx, int64_t count, int32_t D, pode_smoothing_elements lhs,
                           pode_smoothing_elements rhs, pode_smoothing_elements out, int32_t location,
                           pode_status* status) {
  return guarded(status, [&] {
    check_ctx(ctx);
    check_dims(D, count);
    if (count == 0) return;
    const auto& ops = ops_for(D);
    const bool dev = location == PODE_DEVICE;
    const SEd l = stage_se(ctx, "cs_l", lhs, count, D, dev, true);
    const SEd r = stage_se(ctx, "cs_r", rhs, count, D, dev, true);
    const SEd o = stage_se(ctx, "cs_o", out, count, D, dev, false);
    reset_error(ctx);
    ops.combine_smoothing(ctx, count, l, r, o);
    unstage_se(ctx, out, o, count, D, dev);
    raise_device_error(ctx, "combine_smoothing");
  });
}

int pode_make_filtering_elements(pode_context* ctx, const pode_chain* chain, int32_t absorb_init,
                                 pode_filtering_elements out, pode_status* status) {
  return guarded(status, [&] {
    check_ctx(ctx);
    const DevChain ch = stage_chain(ctx, chain);
    const auto& ops = ops_for(ch.D);
    const bool dev = chain->location == PODE_DEVICE;
    const FEd o = stage_fe(ctx, "mf_o", out, ch.N, ch.D, dev, false);
    reset_error(ctx);
    ops.make_filtering(ctx, ch, absorb_init, o);
    unstage_fe(ctx, out, o, ch.N, ch.D, dev);
    raise_device_error(ctx, "make_filtering_element: innovation covariance");
  });
}

int pode_make_smoothing_elements(pode_context* ctx, const pode_chain* chain, const double* f_mean,
                                 const double* f_cov_sqrt, pode_smoothing_elements out, pode_status* status) {
  return guarded(status, [&] {
    check_ctx(ctx);
    const DevChain ch = stage_chain(ctx, chain);
    const auto& ops = ops_for(ch.D);
    const bool dev = chain->location == PODE_DEVICE;
    const int D = ch.D;
    const int64_t n1 = ch.N + 1;
    const double* fm = stage_in(ctx, "ms_fm", f_mean, size_t(n1) * D, dev);
    const double* fc = stage_in(ctx, "ms_fc", f_cov_sqrt, size_t(n1) * D * D, dev);
    const SEd o = stage_se(ctx, "ms_o", out, n1, D, dev, false);
    reset_error(ctx);
    ops.make_smoothing(ctx, ch, fm, fc, o);
    unstage_se(ctx, out, o, n1, D, dev);
    raise_device_error(ctx, "make_smoothing_element: predicted covariance");
  });
}

int pode_scan_filtering(pode_context* ctx, int64_t count, int32_t D, pode_filtering_elements in,
                        pode_filtering_elements out, int32_t reverse, int32_t location, pode_scan_stats* stats,
                        pode_status* status) {
  return guarded(status, [&] {
    check_ctx(ctx);
    check_dims(D, count);
    if (stats) *stats = {0, 0};
    if (count == 0) return;
    const auto& ops = ops_for(D);
    const bool dev = location == PODE_DEVICE;
    const FEd i = stage_fe(ctx, "sf_io", in, count, D, dev, true);
    const FEd o = dev ? fe_view(out) : i;
    reset_error(ctx);
    ScanTally t;
    ops.scan_filtering(ctx, count, i, o, reverse != 0, &t);
    unstage_fe(ctx, out, o, count, D, dev);
    raise_device_error(ctx, "combine_filtering: combination factor", 1);
    if (stats) *stats = {t.combines, t.depth};
  });
}

int pode_scan_smoothing(pode_context* ctx, int64_t count, int32_t D, pode_smoothing_elements in,
                        pode_smoothing_elements out, int32_t reverse, int32_t location, pode_scan_stats* stats,
                        pode_status* status) {
  return guarded(status, [&] {
    check_ctx(ctx);
    check_dims(D, count);
    if (stats) *stats = {0, 0};
    if (count == 0) return;
    const auto& ops = ops_for(D);
    const bool dev = location == PODE_DEVICE;
    const SEd i = stage_se(ctx, "ss_io", in, count, D, dev, true);
    const SEd o = dev ? se_view(out) : i;
    reset_error(ctx);
    ScanTally t;
    ops.scan_smoothing(ctx, count, i, o, reverse != 0, &t);
    unstage_se(ctx, out, o, count, D, dev);
    raise_device_error(ctx, "combine_smoothing", 1);
    if (stats) *stats = {t.combines, t.depth};
  });
}

int pode_rts(pode_context* ctx, const pode_chain* chain, pode_rts_out out, pode_scan_stats* stats,
             pode_status* status) {
  return guarded(status, [&] {
    check_ctx(ctx);
    const DevChain ch = stage_chain(ctx, chain);
    const auto& ops = ops_for(ch.D);
    const bool dev = chain->location == PODE_DEVICE;
    const int D = ch.D;
    const int64_t n1 = ch.N + 1;
    double* fm = dev && out.filtered_mean ? out.filtered_mean : ctx->ws.arr<double>("rts_fm", n1 * D);
    double* fc = dev && out.filtered_cov_sqrt ? out.filtered_cov_sqrt : ctx->ws.arr<double>("rts_fc", n1 * D * D);
    double* sm = dev && out.smoothed_mean ? out.smoothed_mean : ctx->ws.arr<double>("rts_sm", n1 * D);
    double* sc = dev && out.smoothed_cov_sqrt ? out.smoothed_cov_sqrt : ctx->ws.arr<double>("rts_sc", n1 * D * D);
    reset_error(ctx);
    ScanTally t;
    ops.rts(ctx, ch, fm, fc, sm, sc, &t);
    if (!dev) {
      stage_out(ctx, out.filtered_mean, fm, size_t(n1) * D, false);
      stage_out(ctx, out.filtered_cov_sqrt, fc, size_t(n1) * D * D, false);
      stage_out(ctx, out.smoothed_mean, sm, size_t(n1) * D, false);
      stage_out(ctx, out.smoothed_cov_sqrt, sc, size_t(n1) * D * D, false);
    }
    raise_device_error(ctx, "para_rts");
    if (stats) *stats = {t.combines, t.depth};
  });
}

// discretize's grid check (ieks.cpp:8-20).  A serial scan of a 2^20-node
// grid is ~1 ms of host time in front of every solve (the GPU idles behind
// it); large grids are split over up to 8 OpenMP threads.
static void check_grid_increasing(const double* grid, int64_t n_nodes) {
  int bad = 0;
  const int threads = n_nodes > (int64_t(1) << 16) ? std::max(1, std::min(8, omp_get_max_threads())) : 1;
#pragma omp parallel for num_threads(threads) schedule(static) reduction(| : bad)
  for (int64_t n = 0; n < n_nodes - 1; ++n) bad |= !(grid[n + 1] > grid[n]);
  if (bad) throw ApiError(PODE_ERR_INVALID_INPUT, "discretize: grid must be strictly increasing");
}

// pode_ieks and pode_eks: argument checks, output staging and the report.
static int solve_report(pode_context* ctx, const pode_problem* problem, const pode_prior* prior, const double* grid,
                        int64_t n_nodes, const pode_ieks_config* config, pode_ieks_report* report,
                        pode_status* status, bool eks) {
  return guarded(status, [&] {
    check_ctx(ctx);
    if (problem == nullptr || prior == nullptr || grid == nullptr || config == nullptr || report == nullptr)
      throw ApiError(PODE_ERR_INVALID_INPUT, eks ? "eks_solve: NULL argument" : "ieks: NULL argument");
    const host::Problem p = host::resolve_problem(*problem);
    if (p.dim != prior->dim)
      throw ApiError(PODE_ERR_DIMENSION, std::string(eks ? "eks_solve" : "ieks") + ": problem and prior dimensions disagree");
    if (config->max_iterations < 1) throw ApiError(PODE_ERR_INVALID_INPUT, "ieks: max_iterations must be at least 1");
    if (prior->nu < 1 || prior->dim < 1) throw ApiError(PODE_ERR_INVALID_INPUT, "IwpPrior: need nu >= 1 and dim >= 1");
    if (!(prior->sigma >= 0.0) || !std::isfinite(prior->sigma))
      throw ApiError(PODE_ERR_INVALID_INPUT, "IwpPrior: sigma must be finite and nonnegative");
    if (n_nodes < 2) throw ApiError(PODE_ERR_INVALID_INPUT, "discretize: grid needs at least two nodes");
    if (grid[0] != 0.0) throw ApiError(PODE_ERR_INVALID_INPUT, "discretize: grid must start at t = 0");
    check_grid_increasing(grid, n_nodes);
    const int D = prior->dim * (prior->nu + 1);
    const BigIeksFn big = (D > kMaxD && !eks) ? big_ieks(D, prior->dim) : nullptr;
    const EngineOps* ops = big ? nullptr : &ops_for(D);
    const bool dev = report->location == PODE_DEVICE;
    const int d = prior->dim;
    double* means = dev ? report->means : (report->means ? ctx->ws.arr<double>("out_means", n_nodes * D) : nullptr);
    double* cov = dev ? report->cov_sqrt : (report->cov_sqrt ? ctx->ws.arr<double>("out_cov", n_nodes * D * D) : nullptr);
    double* sm = dev ? report->solution_means
                     : (report->solution_means ? ctx->ws.arr<double>("out_sm", n_nodes * d) : nullptr);
    double* sc = dev ? report->solution_covs
                     : (report->solution_covs ? ctx->ws.arr<double>("out_sc", n_nodes * d * d) : nullptr);
    IeksResult r;
    if (big)
      big(ctx, p, *prior, grid, n_nodes, *config, means, cov, sm, sc, &r);
    else
      (eks ? ops->eks : ops->ieks)(ctx, p, *prior, grid, n_nodes, *config, means, cov, sm, sc, &r);
    if (!dev) {
      stage_out(ctx, report->means, means, size_t(n_nodes) * D, false);
      stage_out(ctx, report->cov_sqrt, cov, size_t(n_nodes) * D * D, false);
      stage_out(ctx, report->solution_means, sm, size_t(n_nodes) * d, false);
      stage_out(ctx, report->solution_covs, sc, size_t(n_nodes) * d * d, false);
    }
    raise_device_error(ctx, "ieks: calibration");
    report->iterations = r.iterations;
    report->converged = r.converged ? 1 : 0;
    report->sigma_hat = r.sigma_hat;
    report->scan_stats = {r.stats.combines, r.stats.depth};
    if (report->objective_trace)
      for (int k = 0; k < int(r.trace.size()) && k < report->trace_capacity; ++k)
        report->objective_trace[k] = r.trace[k];
  });
}

int pode_ieks(pode_context* ctx, const pode_problem* problem, const pode_prior* prior, const double* grid,
              int64_t n_nodes, const pode_ieks_config* config, pode_ieks_report* report, pode_status* status) {
  return solve_report(ctx, problem, prior, grid, n_nodes, config, report, status, false);
}

int pode_eks(pode_context* ctx, const pode_problem* problem, const pode_prior* prior, const double* grid,
             int64_t n_nodes, int32_t linearization, pode_ieks_report* report, pode_status* status) {
  const pode_ieks_config cfg{1, 0.0, 0.0, 0.0, linearization};
  return solve_report(ctx, problem, prior, grid, n_nodes, &cfg, report, status, true);
}

int pode_ieks_batch(pode_context* ctx, const pode_problem* problems, int32_t count, const pode_prior* prior,
                    const double* grid, int64_t n_nodes, const pode_ieks_config* config, pode_ieks_report* reports,
                    pode_status* status) {
  return guarded(status, [&] {
    check_ctx(ctx);
    if (problems == nullptr || prior == nullptr || grid == nullptr || config == nullptr || reports == nullptr)
      throw ApiError(PODE_ERR_INVALID_INPUT, "ieks_batch: NULL argument");
    if (count < 1) throw ApiError(PODE_ERR_INVALID_INPUT, "ieks_batch: need at least one problem");
    if (config->max_iterations < 1) throw ApiError(PODE_ERR_INVALID_INPUT, "ieks: max_iterations must be at least 1");
    if (prior->nu < 1 || prior->dim < 1) throw ApiError(PODE_ERR_INVALID_INPUT, "IwpPrior: need nu >= 1 and dim >= 1");
    if (!(prior->sigma >= 0.0) || !std::isfinite(prior->sigma))
      throw ApiError(PODE_ERR_INVALID_INPUT, "IwpPrior: sigma must be finite and nonnegative");
    if (n_nodes < 2) throw ApiError(PODE_ERR_INVALID_INPUT, "discretize: grid needs at least two nodes");
    if (grid[0] != 0.0) throw ApiError(PODE_ERR_INVALID_INPUT, "discretize: grid must start at t = 0");
    check_grid_increasing(grid, n_nodes);
    std::vector<host::Problem> ps;
    ps.reserve(size_t(count));
    for (int32_t i = 0; i < count; ++i) {
      ps.push_back(host::resolve_problem(problems[i]));
      if (ps.back().dim != prior->dim) throw ApiError(PODE_ERR_DIMENSION, "ieks: problem and prior dimensions disagree");
    }
    const int D = prior->dim * (prior->nu + 1);
    const int d = prior->dim;
    const EngineOps* ops = D <= kMaxD ? engine_ops(D) : nullptr;
    if (ops == nullptr || ops->ieks_batch == nullptr)
      throw ApiError(PODE_ERR_UNSUPPORTED, "ieks_batch: no batched engine for state dimension " + std::to_string(D));
    const size_t n1 = size_t(n_nodes), nb = size_t(count);
    bool want_cov = false, want_sm = false, want_sc = false;
    for (size_t i = 0; i < nb; ++i) {
      want_cov |= reports[i].cov_sqrt != nullptr;
      want_sm |= reports[i].solution_means != nullptr;
      want_sc |= reports[i].solution_covs != nullptr;
    }
    double* means = ctx->ws.arr<double>("bout_means", nb * n1 * D);
    double* cov = want_cov ? ctx->ws.arr<double>("bout_cov", nb * n1 * D * D) : nullptr;
    double* sm = want_sm ? ctx->ws.arr<double>("bout_sm", nb * n1 * d) : nullptr;
    double* sc = want_sc ? ctx->ws.arr<double>("bout_sc", nb * n1 * d * d) : nullptr;
    std::vector<IeksResult> rs;
    if (!ops->ieks_batch(ctx, ps, *prior, grid, n_nodes, *config, means, cov, sm, sc, &rs))
      throw ApiError(PODE_ERR_UNSUPPORTED, "ieks_batch: the batched engine needs d <= 3 and D <= 9");
    raise_device_error(ctx, "ieks_batch: calibration");
    for (size_t i = 0; i < nb; ++i) {
      pode_ieks_report& rep = reports[i];
      const bool dev = rep.location == PODE_DEVICE;
      auto copy = [&](double* dst, const double* src, size_t n) {
        if (dst == nullptr || src == nullptr) return;
        if (dev)
          cuda_check(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream),
                     "ieks_batch outputs");
        else
          stage_out(ctx, dst, src, n, false);
      };
      copy(rep.means, means + i * n1 * D, n1 * D);
      copy(rep.cov_sqrt, cov ? cov + i * n1 * D * D : nullptr, n1 * D * D);
      copy(rep.solution_means, sm ? sm + i * n1 * d : nullptr, n1 * d);
      copy(rep.solution_covs, sc ? sc + i * n1 * d * d : nullptr, n1 * d * d);
      const IeksResult& r = rs[i];
      rep.iterations = r.iterations;
      rep.converged = r.converged ? 1 : 0;
      rep.sigma_hat = r.sigma_hat;
      rep.scan_stats = {r.stats.combines, r.stats.depth};
      if (rep.objective_trace)
        for (int k = 0; k < int(r.trace.size()) && k < rep.trace_capacity; ++k) rep.objective_trace[k] = r.trace[k];
    }
    cuda_check(cudaStreamSynchronize(ctx->stream), "ieks_batch sync");
  });
}

int pode_rk4_table(pode_context* ctx, const pode_problem* problem, int64_t steps, double* table,
                   pode_status* status) {
  return guarded(status, [&] {
    check_ctx(ctx);
    if (problem == nullptr || table == nullptr) throw ApiError(PODE_ERR_INVALID_INPUT, "rk4_reference: NULL argument");
    if (steps < 1 || !(problem->t_end > 0.0))
      throw ApiError(PODE_ERR_INVALID_INPUT, "rk4_reference: need positive step and horizon");
    const host::Problem p = host::resolve_problem(*problem);
    if (p.dim > kRk4MaxDim) throw ApiError(PODE_ERR_UNSUPPORTED, "rk4_reference: dimension too large");
    DevProblem dp{};
    dp.kind = p.kind;
    dp.dim = p.dim;
    for (size_t k = 0; k < p.params.size() && k < size_t(kMaxParams); ++k) dp.params[k] = p.params[k];
    const size_t n = size_t(steps + 1) * p.dim;
    double* y0 = ctx->ws.arr<double>("rk4_y0", p.dim);
    double* dev = ctx->ws.arr<double>("rk4_table", n);
    int* bad = ctx->ws.arr<int>("rk4_bad", 1);
    cuda_check(cudaMemcpyAsync(y0, p.y0.data(), sizeof(double) * p.dim, cudaMemcpyHostToDevice, ctx->stream), "y0");
    cuda_check(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream), "rk4 flag");
    k_rk4<kRk4MaxDim><<<1, 32, 0, ctx->stream>>>(dp, p.t_end, steps, y0, dev, bad);
    note_launch(ctx, "rk4");
    int hbad = 0;
    cuda_check(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "rk4 flag");
    stage_out(ctx, table, dev, n, false);
    cuda_check(cudaStreamSynchronize(ctx->stream), "rk4 sync");
    if (hbad) throw ApiError(PODE_ERR_INVALID_INPUT, "rk4_reference: integration diverged");
  });
}

void pode_shard_range(int64_t n_nodes, int32_t rank, int32_t ranks, int64_t* first_node, int64_t* count) {
  const int64_t N = n_nodes - 1;
  const int64_t lo = shard_first_step(N, rank, ranks), hi = shard_first_step(N, rank + 1, ranks);
  if (first_node) *first_node = lo;
  if (count) *count = (hi - lo) + (rank == ranks - 1 ? 1 : 0);
}

int pode_ieks_sharded(pode_context* ctx, const pode_problem* problem, const pode_prior* prior, const double* grid,
                      int64_t n_nodes, const pode_ieks_config* config, const pode_shard_comm* comm,
                      pode_ieks_report* report, pode_status* status) {
  return guarded(status, [&] {
    check_ctx(ctx);
    if (problem == nullptr || prior == nullptr || grid == nullptr || config == nullptr || report == nullptr ||
        comm == nullptr || (comm->allgather == nullptr && ctx->nccl_comm == nullptr))
      throw ApiError(PODE_ERR_INVALID_INPUT, "ieks_sharded: NULL argument");
    if (ctx->nccl_comm && (ctx->nccl_rank != comm->rank || ctx->nccl_ranks != comm->ranks))
      throw ApiError(PODE_ERR_INVALID_INPUT, "ieks_sharded: rank / ranks disagree with the context's NCCL communicator");
    if (comm->ranks < 1 || comm->rank < 0 || comm->rank >= comm->ranks)
      throw ApiError(PODE_ERR_INVALID_INPUT, "ieks_sharded: rank outside [0, ranks)");
    const host::Problem p = host::resolve_problem(*problem);
    if (p.dim != prior->dim) throw ApiError(PODE_ERR_DIMENSION, "ieks: problem and prior dimensions disagree");
    if (config->max_iterations < 1) throw ApiError(PODE_ERR_INVALID_INPUT, "ieks: max_iterations must be at least 1");
    if (prior->nu < 1 || prior->dim < 1) throw ApiError(PODE_ERR_INVALID_INPUT, "IwpPrior: need nu >= 1 and dim >= 1");
    if (!(prior->sigma >= 0.0) || !std::isfinite(prior->sigma))
      throw ApiError(PODE_ERR_INVALID_INPUT, "IwpPrior: sigma must be finite and nonnegative");
    if (n_nodes - 1 < comm->ranks) throw ApiError(PODE_ERR_INVALID_INPUT, "ieks_sharded: fewer steps than shards");
    if (grid[0] != 0.0) throw ApiError(PODE_ERR_INVALID_INPUT, "discretize: grid must start at t = 0");
    check_grid_increasing(grid, n_nodes);
    const int D = prior->dim * (prior->nu + 1);
    const auto& ops = ops_for(D);
    if (ops.ieks_sharded == nullptr) throw ApiError(PODE_ERR_UNSUPPORTED, "ieks_sharded: state dimension not compiled");
    int64_t first = 0, nloc = 0;
    pode_shard_range(n_nodes, comm->rank, comm->ranks, &first, &nloc);
    const bool dev = report->location == PODE_DEVICE;
    const int d = prior->dim;
    // the last shard's engine writes node N too; others write nloc nodes
    double* means = dev ? report->means : (report->means ? ctx->ws.arr<double>("out_means", (nloc + 1) * D) : nullptr);
    double* cov =
        dev ? report->cov_sqrt : (report->cov_sqrt ? ctx->ws.arr<double>("out_cov", (nloc + 1) * D * D) : nullptr);
    double* sm = dev ? report->solution_means
                     : (report->solution_means ? ctx->ws.arr<double>("out_sm", (nloc + 1) * d) : nullptr);
    double* sc = dev ? report->solution_covs
                     : (report->solution_covs ? ctx->ws.arr<double>("out_sc", (nloc + 1) * d * d) : nullptr);
    IeksResult r;
    ops.ieks_sharded(ctx, p, *prior, grid, n_nodes, *config, *comm, means, cov, sm, sc, &r);
    if (!dev) {
      stage_out(ctx, report->means, means, size_t(nloc) * D, false);
      stage_out(ctx, report->cov_sqrt, cov, size_t(nloc) * D * D, false);
      stage_out(ctx, report->solution_means, sm, size_t(nloc) * d, false);
      stage_out(ctx, report->solution_covs, sc, size_t(nloc) * d * d, false);
    }
    raise_device_error(ctx, "ieks: calibration");
    report->iterations = r.iterations;
    report->converged = r.converged ? 1 : 0;
    report->sigma_hat = r.sigma_hat;
    report->scan_stats = {r.stats.combines, r.stats.depth};
    if (report->objective_trace)
      for (int k = 0; k < int(r.trace.size()) && k < report->trace_capacity; ++k)
        report->objective_trace[k] = r.trace[k];
  });
}

}  // extern "C"
