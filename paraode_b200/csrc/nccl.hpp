// Run-time binding of NCCL (dlopen; no NCCL headers or link dependency):
// the device-side all-gather of the time-axis shards (fast_driver.cuh
// run_sharded).  Declarations follow NCCL's stable C ABI.
#pragma once

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "context.hpp"

namespace pode {
namespace nccl {

struct UniqueId {
  char internal[128];
};
using Comm = void*;
using Result = int;  // ncclResult_t: 0 = ncclSuccess
constexpr int kFloat64 = 8;  // ncclFloat64

struct Api {
  void* lib = nullptr;
  Result (*get_unique_id)(UniqueId*) = nullptr;
  Result (*comm_init_rank)(Comm*, int, UniqueId, int) = nullptr;
  Result (*all_gather)(const void*, void*, size_t, int, Comm, cudaStream_t) = nullptr;
  Result (*comm_destroy)(Comm) = nullptr;
  const char* (*error_string)(Result) = nullptr;
};

inline Api& api(const char* path) {
  static Api a;
  static std::mutex m;
  std::lock_guard<std::mutex> g(m);
  if (a.lib) return a;
  a.lib = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!a.lib) throw ApiError(PODE_ERR_UNSUPPORTED, std::string("NCCL not loadable: ") + dlerror());
  auto sym = [&](const char* name) {
    void* f = dlsym(a.lib, name);
    if (!f) throw ApiError(PODE_ERR_UNSUPPORTED, std::string("NCCL symbol missing: ") + name);
    return f;
  };
  a.get_unique_id = reinterpret_cast<Result (*)(UniqueId*)>(sym("ncclGetUniqueId"));
  a.comm_init_rank = reinterpret_cast<Result (*)(Comm*, int, UniqueId, int)>(sym("ncclCommInitRank"));
  a.all_gather = reinterpret_cast<Result (*)(const void*, void*, size_t, int, Comm, cudaStream_t)>(sym("ncclAllGather"));
  a.comm_destroy = reinterpret_cast<Result (*)(Comm)>(sym("ncclCommDestroy"));
  a.error_string = reinterpret_cast<const char* (*)(Result)>(sym("ncclGetErrorString"));
  return a;
}

inline void check(Result r, const char* what) {
  if (r != 0) {
    const Api& a = api(nullptr);
    throw ApiError(PODE_ERR_CUDA, std::string(what) + ": " + (a.error_string ? a.error_string(r) : "NCCL error"));
  }
}

// All-gather of `count` doubles per rank, device buffers, on the context stream.
inline void all_gather(pode_context* ctx, const double* send, int64_t count, double* recv) {
  check(api(nullptr).all_gather(send, recv, size_t(count), kFloat64, ctx->nccl_comm, ctx->stream), "ncclAllGather");
}

inline void destroy(pode_context* ctx) {
  if (ctx->nccl_comm) {
    api(nullptr).comm_destroy(ctx->nccl_comm);
    ctx->nccl_comm = nullptr;
  }
}

}  // namespace nccl
}  // namespace pode
