// Host-side context: one GPU, one stream, a grow-only device workspace and
// the device error word.  Shared by the C ABI (capi.cu) and the per-D
// engines (engine.cuh).
#pragma once

#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/paraode_b200.h"

namespace pode {

struct DevError;

// Error raised on the host side of the ABI; carries a pode_code.
struct ApiError : std::runtime_error {
  ApiError(int c, const std::string& m, int64_t idx = -1, double t = 0.0, int it = 0)
      : std::runtime_error(m), code(c), index(idx), time(t), iteration(it) {}
  int code;
  int64_t index;
  double time;
  int iteration;
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw ApiError(PODE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct Workspace {
  struct Buf {
    void* ptr = nullptr;
    size_t bytes = 0;
  };
  std::map<std::string, Buf> bufs;
  uint64_t generation = 0;  // bumped on every (re)allocation: cached graphs hold raw pointers
  void* get(const std::string& tag, size_t bytes) {
    Buf& b = bufs[tag];
    if (b.bytes < bytes) {
      ++generation;
      if (b.ptr) cudaFree(b.ptr);
      b.ptr = nullptr;
      b.bytes = 0;
      const size_t alloc = bytes < 256 ? 256 : bytes;
      cuda_check(cudaMalloc(&b.ptr, alloc), ("workspace alloc " + tag).c_str());
      b.bytes = alloc;
    }
    return b.ptr;
  }
  template <typename T>
  T* arr(const std::string& tag, size_t count) {
    return static_cast<T*>(get(tag, count * sizeof(T)));
  }
  ~Workspace() {
    for (auto& kv : bufs)
      if (kv.second.ptr) cudaFree(kv.second.ptr);
  }
};

}  // namespace pode

// Per-launch CUDA-event timing (pode_profile): an event is recorded on the
// context stream after every launch and at every host synchronisation point;
// a kernel's duration is the interval since the previous record.
struct ProfRec {
  const char* name;  // nullptr for a synchronisation marker
  cudaEvent_t ev;
};

struct pode_context {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  pode::Workspace ws;
  unsigned long long* d_err = nullptr;  // device error word (DevError)
  unsigned long long* h_err = nullptr;  // pinned mirror
  double* h_scalars = nullptr;          // pinned scalars (reductions)
  int64_t launches = 0;
  // pode_context_nccl_init: device-side shard exchange (nccl.hpp)
  void* nccl_comm = nullptr;
  int nccl_rank = 0, nccl_ranks = 0;
  // pode_context_set_option (0 = automatic / environment default)
  int64_t opt_chunk = 0;
  int opt_engine = 0;
  // Instantiated device-side IEKS loops (fast_driver.cuh), reused while the
  // captured kernel arguments (key) and the workspace generation match.
  struct GraphSlot {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::string key;
    int64_t per_iter = 0;
  };
  std::map<std::string, GraphSlot> graphs;
  // pinned staging ring for large device->host result copies (capi.cu)
  char* h_stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  bool prof_on = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> prof_pool;
  size_t prof_used = 0;
};

namespace pode {

inline cudaEvent_t prof_event(pode_context* ctx) {
  if (ctx->prof_used == ctx->prof_pool.size()) {
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "profile event");
    ctx->prof_pool.push_back(e);
  }
  return ctx->prof_pool[ctx->prof_used++];
}

inline void prof_record(pode_context* ctx, const char* name) {
  if (!ctx->prof_on) return;
  cudaEvent_t e = prof_event(ctx);
  cuda_check(cudaEventRecord(e, ctx->stream), "profile record");
  ctx->prof.push_back({name, e});
}

// NVTX range over one IEKS stage (visible in Nsight Systems / ncu's NVTX
// filters: --nvtx --nvtx-include "pass_C/"); header-only NVTX v3.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// PODE_TRACE_LAUNCHES=1 (debugging): synchronise after every launch and
// name it on stderr, so a fault or hang is attributed to its kernel.
inline bool trace_launches() {
  static const bool on = [] {
    const char* e = std::getenv("PODE_TRACE_LAUNCHES");
    return e != nullptr && *e != '\0' && *e != '0';
  }();
  return on;
}

inline void note_launch(pode_context* ctx, const char* what) {
  ctx->launches += 1;
  cuda_check(cudaGetLastError(), what);
  if (trace_launches()) {
    std::fprintf(stderr, "[pode] launch %lld %s ...", static_cast<long long>(ctx->launches), what);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(ctx->stream, &cs);
    if (cs == cudaStreamCaptureStatusNone) cuda_check(cudaStreamSynchronize(ctx->stream), what);
    std::fprintf(stderr, " done\n");
  }
  prof_record(ctx, what);
}

// After a host synchronisation: the next launch's interval starts here.
inline void prof_mark(pode_context* ctx) { prof_record(ctx, nullptr); }

// Resets the device error word (before a stage) / reads it back (after).
void reset_error(pode_context* ctx);
// Returns the packed key ((index << 8) | code), ~0ull when clean. Syncs.
unsigned long long fetch_error(pode_context* ctx);

}  // namespace pode
