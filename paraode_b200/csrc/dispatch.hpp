// Runtime dispatch from the state dimension D to the compiled engine.
#pragma once

#include <vector>

#include "context.hpp"

namespace pode {

struct FEd;
struct SEd;
struct DevChain;
struct ScanTally;
struct IeksResult;
namespace host {
struct Problem;
}

struct EngineOps {
  int D;
  void (*combine_filtering)(pode_context*, int64_t, const FEd&, const FEd&, const FEd&);
  void (*combine_smoothing)(pode_context*, int64_t, const SEd&, const SEd&, const SEd&);
  void (*make_filtering)(pode_context*, const DevChain&, int, const FEd&);
  void (*make_smoothing)(pode_context*, const DevChain&, const double*, const double*, const SEd&);
  void (*scan_filtering)(pode_context*, int64_t, const FEd&, const FEd&, bool, ScanTally*);
  void (*scan_smoothing)(pode_context*, int64_t, const SEd&, const SEd&, bool, ScanTally*);
  void (*rts)(pode_context*, const DevChain&, double*, double*, double*, double*, ScanTally*);
  void (*ieks)(pode_context*, const host::Problem&, const pode_prior&, const double*, int64_t,
               const pode_ieks_config&, double*, double*, double*, double*, IeksResult*);
  // time-axis shard of the fused engine (nullptr where it is not compiled)
  void (*ieks_sharded)(pode_context*, const host::Problem&, const pode_prior&, const double*, int64_t,
                       const pode_ieks_config&, const pode_shard_comm&, double*, double*, double*, double*,
                       IeksResult*);
  // eks_solve (element engine; cfg.linearization only)
  void (*eks)(pode_context*, const host::Problem&, const pode_prior&, const double*, int64_t,
              const pode_ieks_config&, double*, double*, double*, double*, IeksResult*);
  // batched fused solve of many IVPs (batch_driver.cuh; lane engine only):
  // outputs stacked per IVP, false when no batched engine serves (D, d)
  bool (*ieks_batch)(pode_context*, const std::vector<host::Problem>&, const pode_prior&, const double*, int64_t,
                     const pode_ieks_config&, double*, double*, double*, double*, std::vector<IeksResult>*);
};

// Shard s of R owns steps [floor(N s / R), floor(N (s+1) / R)).
inline int64_t shard_first_step(int64_t N, int s, int R) { return (N * s) / R; }

constexpr int kMinD = 1;
constexpr int kMaxD = 16;

const EngineOps* engine_ops(int D);  // nullptr when D is not compiled

// The large-state fused IEKS engine (big.cuh; D > kMaxD): nullptr when
// (D, d) is not compiled.
using BigIeksFn = void (*)(pode_context*, const host::Problem&, const pode_prior&, const double*, int64_t,
                           const pode_ieks_config&, double*, double*, double*, double*, IeksResult*);
BigIeksFn big_ieks(int D, int d);

}  // namespace pode
