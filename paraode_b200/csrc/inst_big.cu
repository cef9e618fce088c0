// Large-state fused IEKS engine instantiations (big.cuh): Pleiades-type
// problems, d = 28, IWP(1..3) (D = 56, 84, 112).
#include "big_driver.cuh"
#include "dispatch.hpp"

namespace pode {

namespace {
template <int D, int d>
void big_ik(pode_context* c, const host::Problem& p, const pode_prior& pr, const double* g, int64_t n1,
            const pode_ieks_config& cfg, double* m, double* cv, double* sm, double* sc, IeksResult* out) {
  *out = BigEngine<D, d>::run(c, p, pr, g, n1, cfg, m, cv, sm, sc);
}
}  // namespace

BigIeksFn big_ieks(int D, int d) {
  if (d == 28 && D == 56) return big_ik<56, 28>;
  if (d == 28 && D == 84) return big_ik<84, 28>;
  if (d == 28 && D == 112) return big_ik<112, 28>;
  return nullptr;
}

}  // namespace pode
