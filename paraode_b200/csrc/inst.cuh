// Instantiates the engine for one state dimension; included by inst_dN.cu
// with PODE_D defined, so the per-D kernels compile in parallel.
#include <cstdlib>
#include <string>

#include "dispatch.hpp"
#include "fast_driver.cuh"
#include "batch_driver.cuh"
#include "ieks.cuh"

#ifndef PODE_D
#error "define PODE_D"
#endif

namespace pode {

#define PODE_CAT2(a, b) a##b
#define PODE_CAT(a, b) PODE_CAT2(a, b)

namespace {
constexpr int kD = PODE_D;
using E = Engine<kD>;

void cf(pode_context* c, int64_t n, const FEd& l, const FEd& r, const FEd& o) { E::combine_filtering(c, n, l, r, o); }
void cs(pode_context* c, int64_t n, const SEd& l, const SEd& r, const SEd& o) { E::combine_smoothing(c, n, l, r, o); }
void mf(pode_context* c, const DevChain& ch, int a, const FEd& o) { E::make_filtering(c, ch, a, o); }
void ms(pode_context* c, const DevChain& ch, const double* fm, const double* fc, const SEd& o) {
  E::make_smoothing(c, ch, fm, fc, o);
}
void sf(pode_context* c, int64_t n, const FEd& i, const FEd& o, bool rev, ScanTally* t) {
  *t = E::scan_filtering(c, n, i, o, rev);
}
void ss(pode_context* c, int64_t n, const SEd& i, const SEd& o, bool rev, ScanTally* t) {
  *t = E::scan_smoothing(c, n, i, o, rev);
}
void rt(pode_context* c, const DevChain& ch, double* fm, double* fc, double* sm, double* sc, ScanTally* t) {
  *t = E::rts(c, ch, fm, fc, sm, sc);
}
template <int DD, int d>
// Lane-serial passes keep D x D matrices in registers: beyond D = 9 they
// spill heavily (and take tens of minutes to compile), so larger states use
// the group engine.
constexpr bool kFastOk = (d <= 3) && (DD % d == 0) && (DD / d >= 2) && (DD / d <= 5) && (DD <= 9);
// Above that, the fused iteration runs on groups of D lanes (grp_fused.cuh).
template <int DD, int d>
constexpr bool kGrpOk = (d <= 3) && (DD % d == 0) && (DD / d >= 2) && (DD / d <= 8) && (DD >= 10) && (DD <= 16);

template <int d>
bool run_fused(pode_context* c, const host::Problem& p, const pode_prior& pr, const double* g, int64_t n1,
               const pode_ieks_config& cfg, double* m, double* cv, double* sm, double* sc, IeksResult* out) {
  if constexpr (kFastOk<kD, d>) {
    *out = FastEngine<kD, d>::run(c, p, pr, g, n1, cfg, m, cv, sm, sc);
    return true;
  } else if constexpr (kGrpOk<kD, d>) {
    *out = FastEngine<kD, d, GroupPasses<kD, d>>::run(c, p, pr, g, n1, cfg, m, cv, sm, sc);
    return true;
  }
  return false;
}

// The fused engines (fast.cuh: lane passes D <= 9, group passes D = 10..16)
// serve ODE information operators with d <= 3;
// everything else (and PODE_IEKS_ENGINE=elements) runs the element/scan
// engine with the reference's per-iteration structure.
void ik(pode_context* c, const host::Problem& p, const pode_prior& pr, const double* g, int64_t n1,
        const pode_ieks_config& cfg, double* m, double* cv, double* sm, double* sc, IeksResult* out) {
  const char* env = std::getenv("PODE_IEKS_ENGINE");
  const bool elements = c->opt_engine == 2 || (c->opt_engine == 0 && env != nullptr && std::string(env) == "elements");
  if (!elements) {
    switch (pr.dim) {
      case 1:
        if (run_fused<1>(c, p, pr, g, n1, cfg, m, cv, sm, sc, out)) return;
        break;
      case 2:
        if (run_fused<2>(c, p, pr, g, n1, cfg, m, cv, sm, sc, out)) return;
        break;
      case 3:
        if (run_fused<3>(c, p, pr, g, n1, cfg, m, cv, sm, sc, out)) return;
        break;
      default:
        break;
    }
    if (c->opt_engine == 1)
      throw ApiError(PODE_ERR_UNSUPPORTED, "ieks: no fused engine serves state dimension " + std::to_string(kD) +
                                               " with d = " + std::to_string(pr.dim));
  }
  *out = IeksEngine<kD>::run(c, p, pr, g, n1, cfg, m, cv, sm, sc);
}
// Time-axis shard: the fused engine only.
void iks(pode_context* c, const host::Problem& p, const pode_prior& pr, const double* g, int64_t n1,
         const pode_ieks_config& cfg, const pode_shard_comm& comm, double* m, double* cv, double* sm, double* sc,
         IeksResult* out) {
  switch (pr.dim) {
    case 1:
      if constexpr (kFastOk<kD, 1>) {
        *out = FastEngine<kD, 1>::run_sharded(c, p, pr, g, n1, cfg, comm, m, cv, sm, sc);
        return;
      }
      break;
    case 2:
      if constexpr (kFastOk<kD, 2>) {
        *out = FastEngine<kD, 2>::run_sharded(c, p, pr, g, n1, cfg, comm, m, cv, sm, sc);
        return;
      }
      break;
    case 3:
      if constexpr (kFastOk<kD, 3>) {
        *out = FastEngine<kD, 3>::run_sharded(c, p, pr, g, n1, cfg, comm, m, cv, sm, sc);
        return;
      }
      break;
    default:
      break;
  }
  throw ApiError(PODE_ERR_UNSUPPORTED, "ieks_sharded: needs an ODE operator the fused engine serves (d <= 3, D <= 9)");
}
void ek(pode_context* c, const host::Problem& p, const pode_prior& pr, const double* g, int64_t n1,
        const pode_ieks_config& cfg, double* m, double* cv, double* sm, double* sc, IeksResult* out) {
  *out = IeksEngine<kD>::run_eks(c, p, pr, g, n1, cfg, m, cv, sm, sc);
}
// Batched fused solve: the lane engine's kBatch passes.
bool ikb(pode_context* c, const std::vector<host::Problem>& ps, const pode_prior& pr, const double* g, int64_t n1,
         const pode_ieks_config& cfg, double* m, double* cv, double* sm, double* sc, std::vector<IeksResult>* out) {
  switch (pr.dim) {
    case 1:
      if constexpr (kFastOk<kD, 1>) {
        *out = BatchEngine<kD, 1>::run(c, ps, pr, g, n1, cfg, m, cv, sm, sc);
        return true;
      }
      break;
    case 2:
      if constexpr (kFastOk<kD, 2>) {
        *out = BatchEngine<kD, 2>::run(c, ps, pr, g, n1, cfg, m, cv, sm, sc);
        return true;
      }
      break;
    case 3:
      if constexpr (kFastOk<kD, 3>) {
        *out = BatchEngine<kD, 3>::run(c, ps, pr, g, n1, cfg, m, cv, sm, sc);
        return true;
      }
      break;
    default:
      break;
  }
  return false;
}
const EngineOps kOps{kD, cf, cs, mf, ms, sf, ss, rt, ik, iks, ek, ikb};
}  // namespace

const EngineOps* PODE_CAT(engine_ops_d, PODE_D)() { return &kOps; }

}  // namespace pode
