// Device vector-field registry.  The reference's InitialValueProblem holds
// host std::function callbacks (proj/include/paraode/statespace.hpp:24-31),
// which cannot run on the GPU; problems are therefore registered kinds with
// parameters, evaluated here per time step.  Field definitions follow
// proj/src/problems.cpp:81-107 (logistic, rigid body, Van der Pol) plus the
// FitzHugh-Nagumo, Pleiades and affine fields of SURVEY.md §8c, and the
// test kind PODE_POLE (y' = 1 / (t - a): the reference's non-finite-field
// case, test_statespace.cpp:123-139, with the pole on a grid node).
#pragma once

#include <cuda_runtime.h>

namespace pode {

constexpr int kMaxParams = 64;  // affine up to d = 7 (L d*d + c d)

struct DevProblem {
  int kind;
  int dim;
  double params[kMaxParams];
};

// f(y, t) and its Jacobian J(y) (row stride DMAX), for d = p.dim <= DMAX.
// Only PODE_POLE reads t.  Every index is static once DMAX is fixed (cases whose
// dimension exceeds DMAX are compiled out), so y/f/jac stay in registers.
template <int DMAX>
__device__ __forceinline__ void eval_field(const DevProblem& p, const double* y, double* f, double* jac,
                                           double t = 0.0) {
  const int d = p.dim;
  switch (p.kind) {
    case 1: {  // logistic (problems.cpp:83-88, 126-128)
      f[0] = y[0] * (1.0 - y[0]);
      jac[0] = 1.0 - 2.0 * y[0];
      break;
    }
    case 2: {  // rigid body (problems.cpp:90-97, 145-151)
      if constexpr (DMAX >= 3) {
        f[0] = -2.0 * (y[1] * y[2]);
        f[1] = 1.25 * (y[0] * y[2]);
        f[2] = -0.5 * (y[0] * y[1]);
        jac[0] = 0.0, jac[1] = -2.0 * y[2], jac[2] = -2.0 * y[1];
        jac[DMAX + 0] = 1.25 * y[2], jac[DMAX + 1] = 0.0, jac[DMAX + 2] = 1.25 * y[0];
        jac[2 * DMAX + 0] = -0.5 * y[1], jac[2 * DMAX + 1] = -0.5 * y[0], jac[2 * DMAX + 2] = 0.0;
      }
      break;
    }
    case 3: {  // Van der Pol (problems.cpp:99-105, 167-172)
      if constexpr (DMAX >= 2) {
        const double mu = p.params[0];
        f[0] = y[1];
        f[1] = mu * ((1.0 - y[0] * y[0]) * y[1] - y[0]);
        jac[0] = 0.0, jac[1] = 1.0;
        jac[DMAX + 0] = -2.0 * mu * y[0] * y[1] - mu, jac[DMAX + 1] = mu * (1.0 - y[0] * y[0]);
      }
      break;
    }
    case 4: {  // FitzHugh-Nagumo
      if constexpr (DMAX >= 2) {
        const double a = p.params[0], b = p.params[1], c = p.params[2];
        f[0] = c * ((y[0] - (y[0] * y[0] * y[0]) * (1.0 / 3.0)) + y[1]);
        f[1] = ((y[0] - a) + b * y[1]) * (-1.0 / c);
        jac[0] = c * (1.0 - y[0] * y[0]), jac[1] = c;
        jac[DMAX + 0] = -1.0 / c, jac[DMAX + 1] = -b / c;
      }
      break;
    }
    case 5: {  // Pleiades, 7 bodies, m_j = j + 1
      if constexpr (DMAX >= 28) {
        constexpr int B = 7;
        for (int i = 0; i < DMAX * DMAX; ++i) jac[i] = 0.0;
        for (int i = 0; i < B; ++i) {
          f[i] = y[2 * B + i];
          f[B + i] = y[3 * B + i];
          jac[i * DMAX + 2 * B + i] = 1.0;
          jac[(B + i) * DMAX + 3 * B + i] = 1.0;
        }
        for (int i = 0; i < B; ++i) {
          double ax = 0.0, ay = 0.0;
          for (int j = 0; j < B; ++j) {
            if (j == i) continue;
            const double dx = y[j] - y[i], dy = y[B + j] - y[B + i];
            const double r2 = dx * dx + dy * dy;
            const double r = sqrt(r2);
            const double r3 = r2 * r, r5 = r3 * r2;
            const double mj = static_cast<double>(j + 1);
            ax += (mj * dx) / r3;
            ay += (mj * dy) / r3;
            const double dxx = mj * (1.0 / r3 - 3.0 * dx * dx / r5);
            const double dxy = mj * (-3.0 * dx * dy / r5);
            const double dyy = mj * (1.0 / r3 - 3.0 * dy * dy / r5);
            jac[(2 * B + i) * DMAX + j] += dxx;
            jac[(2 * B + i) * DMAX + i] -= dxx;
            jac[(2 * B + i) * DMAX + B + j] += dxy;
            jac[(2 * B + i) * DMAX + B + i] -= dxy;
            jac[(3 * B + i) * DMAX + j] += dxy;
            jac[(3 * B + i) * DMAX + i] -= dxy;
            jac[(3 * B + i) * DMAX + B + j] += dyy;
            jac[(3 * B + i) * DMAX + B + i] -= dyy;
          }
          f[2 * B + i] = ax;
          f[3 * B + i] = ay;
        }
      }
      break;
    }
    case 7: {  // pole: y' = 1 / (t - a) (non-finite exactly at t = a)
      f[0] = 1.0 / (t - p.params[0]);
      jac[0] = 0.0;
      break;
    }
    default: {  // affine: y' = L y + c
#pragma unroll
      for (int i = 0; i < DMAX; ++i) {
        if (i >= d) break;
        double acc = p.params[d * d + i];
#pragma unroll
        for (int j = 0; j < DMAX; ++j) {
          if (j >= d) break;
          acc = acc + y[j] * p.params[i * d + j];
          jac[i * DMAX + j] = p.params[i * d + j];
        }
        f[i] = acc;
      }
      break;
    }
  }
}

}  // namespace pode
