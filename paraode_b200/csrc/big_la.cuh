// CTA-wide dense fp64 linear algebra for large state dimensions (D ~ 100,
// Pleiades D = 112): the operands of one IEKS time step are 12 K-entry
// matrices, so one CTA (kBT threads) owns one chunk and works on matrices
// that live in its global-memory workspace (L2-resident) and its shared
// memory.  Products run on the FP64 tensor pipe (DMMA, mma.sync m8n8k4
// .f64): at this size they are real dense contractions (SURVEY.md §8(d):
// AI ~ 200 flop/B).  Factorisations (Cholesky, LU) are column-serial with
// CTA-wide trailing updates.
//
// Every routine is called by all threads of the CTA and ends with a
// __syncthreads(); matrices are row-major with an explicit leading dimension.
#pragma once

#include <cuda_runtime.h>
#include <cfloat>
#include <cstdint>

namespace pode {
namespace big {

constexpr int kBT = 256;  // threads per CTA
constexpr int kBW = kBT / 32;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// C[M x N] = alpha op(A)[M x K] op(B)[K x N] + beta C (beta = 0: C is not
// read).  op(X) = X^T when TX.  Any M, N, K (edges predicated).  One warp per
// 8 x 16 output block (two 8 x 8 DMMA tiles sharing the A fragment).  C must
// not alias A or B.
template <bool TA, bool TB>
__device__ void gemm(int M, int N, int K, double alpha, const double* A, int lda, const double* B, int ldb,
                     double beta, double* C, int ldc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gr = lane >> 2, tg = lane & 3;
  const int mt = (M + 7) / 8, nt = (N + 15) / 16;
  for (int t = warp; t < mt * nt; t += kBW) {
    const int m0 = (t / nt) * 8, n0 = (t % nt) * 16;
    double c[4] = {0.0, 0.0, 0.0, 0.0};
    const int ar = m0 + gr;
    const int bc0 = n0 + gr, bc1 = n0 + 8 + gr;
    for (int k0 = 0; k0 < K; k0 += 4) {
      const int ak = k0 + tg;
      double a = 0.0, b0 = 0.0, b1 = 0.0;
      if (ar < M && ak < K) a = TA ? A[ak * lda + ar] : A[ar * lda + ak];
      if (ak < K) {
        if (bc0 < N) b0 = TB ? B[bc0 * ldb + ak] : B[ak * ldb + bc0];
        if (bc1 < N) b1 = TB ? B[bc1 * ldb + ak] : B[ak * ldb + bc1];
      }
      dmma(c[0], c[1], a, b0, c[0], c[1]);
      dmma(c[2], c[3], a, b1, c[2], c[3]);
    }
    const int r = m0 + gr;
    if (r < M) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int cc = n0 + 8 * h + 2 * tg + i;
          if (cc < N) {
            double* p = C + r * ldc + cc;
            *p = (beta == 0.0) ? alpha * c[2 * h + i] : fma(alpha, c[2 * h + i], beta * *p);
          }
        }
      }
    }
  }
  __syncthreads();
}

// y[M] = alpha op(A) x + beta y (one thread per output; x may live anywhere
// but must not alias y).
template <bool TA>
__device__ void gemv(int M, int K, double alpha, const double* A, int lda, const double* x, double beta, double* y) {
  for (int i = threadIdx.x; i < M; i += kBT) {
    double acc = 0.0;
    for (int k = 0; k < K; ++k) acc = fma(TA ? A[k * lda + i] : A[i * lda + k], x[k], acc);
    y[i] = (beta == 0.0) ? alpha * acc : fma(alpha, acc, beta * y[i]);
  }
  __syncthreads();
}

__device__ __forceinline__ void copy(int n, const double* src, double* dst) {
  for (int i = threadIdx.x; i < n; i += kBT) dst[i] = src[i];
  __syncthreads();
}

// (A + A^T) / 2 in place (n x n).
__device__ __forceinline__ void symmetrize(int n, double* A, int lda) {
  for (int idx = threadIdx.x; idx < n * n; idx += kBT) {
    const int i = idx / n, j = idx - (idx / n) * n;
    if (i < j) {
      const double v = 0.5 * (A[i * lda + j] + A[j * lda + i]);
      A[i * lda + j] = v;
      A[j * lda + i] = v;
    }
  }
  __syncthreads();
}

// CTA-wide max of one value per thread (red: kBW doubles of shared scratch).
__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double m = red[0];
#pragma unroll
  for (int w = 1; w < kBW; ++w) m = fmax(m, red[w]);
  __syncthreads();
  return m;
}
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double m = 0.0;
#pragma unroll
  for (int w = 0; w < kBW; ++w) m += red[w];
  __syncthreads();
  return m;
}

// In-place lower Cholesky factor of the SPD n x n matrix A (upper triangle
// zeroed).  Right-looking, one column per step.  Returns true (CTA-uniform)
// when a pivot is not positive or |L_jj| <= 1e-13 max_i |L_ii| — the
// reference's singular-factor test on the factor (linalg.cpp:54-62).
__device__ bool potrf(int n, double* A, int lda, double* red) {
  __shared__ double s_piv;
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  double dmax = 0.0;
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      const double dj = A[j * lda + j];
      const double l = dj > 0.0 ? sqrt(dj) : 0.0;
      if (!(dj > 0.0)) s_bad = 1;
      A[j * lda + j] = l;
      s_piv = l > 0.0 ? 1.0 / l : 0.0;
    }
    __syncthreads();
    const double inv = s_piv;
    for (int i = j + 1 + threadIdx.x; i < n; i += kBT) A[i * lda + j] *= inv;
    __syncthreads();
    // trailing update of the lower triangle
    const int m = n - j - 1;
    for (int idx = threadIdx.x; idx < m * m; idx += kBT) {
      const int i = j + 1 + idx / m, k = j + 1 + idx - (idx / m) * m;
      if (k <= i) A[i * lda + k] = fma(-A[i * lda + j], A[k * lda + j], A[i * lda + k]);
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < n * n; idx += kBT) {
    const int i = idx / n, k = idx - (idx / n) * n;
    if (k > i) A[i * lda + k] = 0.0;
    if (k == i) dmax = fmax(dmax, fabs(A[i * lda + k]));
  }
  __syncthreads();
  const double mx = block_max(dmax, red);
  double mine = 0.0;
  for (int i = threadIdx.x; i < n; i += kBT) mine = fmax(mine, fabs(A[i * lda + i]) <= 1e-13 * mx ? 1.0 : 0.0);
  const double sing = block_max(mine, red);
  return sing > 0.0 || s_bad != 0;
}

// X <- L^-1 in place for the lower-triangular n x n L (column j by thread
// j: forward substitution of L x = e_j; n <= kBT).  The strict upper part is
// zero on return.  Reads L from A and writes the inverse into W.
__device__ void trtri_lower(int n, const double* L, int ldl, double* W, int ldw) {
  for (int idx = threadIdx.x; idx < n * n; idx += kBT) W[(idx / n) * ldw + idx % n] = 0.0;
  __syncthreads();
  const int j = threadIdx.x;
  if (j < n) {
    W[j * ldw + j] = 1.0 / L[j * ldl + j];
    for (int i = j + 1; i < n; ++i) {
      double acc = 0.0;
      for (int k = j; k < i; ++k) acc = fma(L[i * ldl + k], W[k * ldw + j], acc);
      W[i * ldw + j] = -acc / L[i * ldl + i];
    }
  }
  __syncthreads();
}

// LU with partial pivoting of the n x n A, then X <- A^-1 X for the n x m
// right-hand sides (in place).  A is destroyed.
__device__ void lu_solve(int n, double* A, int lda, int m, double* X, int ldx, double* red) {
  __shared__ int s_p;
  __shared__ double s_inv;
  for (int j = 0; j < n; ++j) {
    // pivot: argmax |A[i][j]|, i >= j (warp 0)
    if (threadIdx.x < 32) {
      double best = -1.0;
      int bi = j;
      for (int i = j + threadIdx.x; i < n; i += 32) {
        const double v = fabs(A[i * lda + j]);
        if (v > best) {
          best = v;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
          best = ov;
          bi = oi;
        }
      }
      if (threadIdx.x == 0) s_p = bi;
    }
    __syncthreads();
    const int p = s_p;
    if (p != j) {
      for (int k = threadIdx.x; k < n; k += kBT) {
        const double t = A[j * lda + k];
        A[j * lda + k] = A[p * lda + k];
        A[p * lda + k] = t;
      }
      for (int k = threadIdx.x; k < m; k += kBT) {
        const double t = X[j * ldx + k];
        X[j * ldx + k] = X[p * ldx + k];
        X[p * ldx + k] = t;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_inv = 1.0 / A[j * lda + j];
    __syncthreads();
    const double inv = s_inv;
    for (int i = j + 1 + threadIdx.x; i < n; i += kBT) A[i * lda + j] *= inv;
    __syncthreads();
    const int rows = n - j - 1, cols = n - j - 1;
    for (int idx = threadIdx.x; idx < rows * (cols + m); idx += kBT) {
      const int i = j + 1 + idx / (cols + m), c = idx - (idx / (cols + m)) * (cols + m);
      const double l = A[i * lda + j];
      if (c < cols)
        A[i * lda + j + 1 + c] = fma(-l, A[j * lda + j + 1 + c], A[i * lda + j + 1 + c]);
      else
        X[i * ldx + (c - cols)] = fma(-l, X[j * ldx + (c - cols)], X[i * ldx + (c - cols)]);
    }
    __syncthreads();
  }
  // back substitution U x = y, column by column of X (thread per rhs column)
  for (int c = threadIdx.x; c < m; c += kBT) {
    for (int i = n - 1; i >= 0; --i) {
      double acc = X[i * ldx + c];
      for (int k = i + 1; k < n; ++k) acc = fma(-A[i * lda + k], X[k * ldx + c], acc);
      X[i * ldx + c] = acc / A[i * lda + i];
    }
  }
  __syncthreads();
  (void)red;
}

}  // namespace big
}  // namespace pode
