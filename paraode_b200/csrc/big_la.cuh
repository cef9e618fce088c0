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

// The kernels' dynamic shared memory: the staging area of every routine
// below (they do not nest).  Size: big_smem_bytes<D>() (big.cuh).
__device__ __forceinline__ double* dyn_smem() {
  extern __shared__ double big_dyn_smem[];
  return big_dyn_smem;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// C[M x N] = alpha op(A)[M x K] op(B)[K x N] + beta C (beta = 0: C is not
// read).  op(X) = X^T when TX.  M, K any; N <= 8 * kNT.  op(B) is staged in
// shared memory (dyn_smem: >= K (N + 1) doubles, odd row stride: conflict-free
// fragment reads); each warp owns 8-row blocks of C and sweeps all N/8
// column tiles with the A fragment in registers (one DMMA m8n8k4 per tile
// per k-step, the next A fragment loaded ahead).  C must not alias A or B.
constexpr int kNT = 16;  // N <= 128
template <bool TA, bool TB>
__device__ void gemm(int M, int N, int K, double alpha, const double* A, int lda, const double* B, int ldb,
                     double beta, double* C, int ldc) {
  double* sm = dyn_smem();
  const int ldb_s = N + 1;
  for (int idx = threadIdx.x; idx < K * N; idx += kBT) {
    int k, n;
    if (TB) {  // B stored N x K: read along k
      n = idx / K;
      k = idx - n * K;
    } else {
      k = idx / N;
      n = idx - k * N;
    }
    sm[k * ldb_s + n] = TB ? B[n * ldb + k] : B[k * ldb + n];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gr = lane >> 2, tg = lane & 3;
  const int nt = (N + 7) / 8;
  for (int m0 = warp * 8; m0 < M; m0 += kBW * 8) {
    double acc[kNT][2];
#pragma unroll
    for (int t = 0; t < kNT; ++t) acc[t][0] = acc[t][1] = 0.0;
    const int ar = m0 + gr;
    auto lda_at = [&](int k) -> double {
      return (ar < M && k < K) ? (TA ? A[k * lda + ar] : A[ar * lda + k]) : 0.0;
    };
    double a = lda_at(tg);
    for (int k0 = 0; k0 < K; k0 += 4) {
      const double an = lda_at(k0 + 4 + tg);  // next fragment in flight
      const int kb = k0 + tg;
      const bool kin = kb < K;
#pragma unroll
      for (int t = 0; t < kNT; ++t) {
        if (t < nt) {
          const int col = t * 8 + gr;
          const double b = (kin && col < N) ? sm[kb * ldb_s + col] : 0.0;
          dmma(acc[t][0], acc[t][1], a, b, acc[t][0], acc[t][1]);
        }
      }
      a = an;
    }
    const int r = m0 + gr;
    if (r < M) {
#pragma unroll
      for (int t = 0; t < kNT; ++t) {
        if (t < nt) {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int cc = t * 8 + 2 * tg + i;
            if (cc < N) {
              double* p = C + r * ldc + cc;
              *p = (beta == 0.0) ? alpha * acc[t][i] : fma(alpha, acc[t][i], beta * *p);
            }
          }
        }
      }
    }
  }
  __syncthreads();
}

// y[M] = alpha op(A) x + beta y; x must not alias y.  op(A) = A: one warp
// per row (coalesced row reads, shuffle reduction); A^T: one thread per
// output (coalesced column reads across the warp).
template <bool TA>
__device__ void gemv(int M, int K, double alpha, const double* A, int lda, const double* x, double beta, double* y) {
  if (TA) {
    for (int i = threadIdx.x; i < M; i += kBT) {
      double acc = 0.0;
      for (int k = 0; k < K; ++k) acc = fma(A[k * lda + i], x[k], acc);
      y[i] = (beta == 0.0) ? alpha * acc : fma(alpha, acc, beta * y[i]);
    }
  } else {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = warp; i < M; i += kBW) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // independent chains: loads in flight
      int k = lane;
      for (; k + 96 < K; k += 128) {
        a0 = fma(A[i * lda + k], x[k], a0);
        a1 = fma(A[i * lda + k + 32], x[k + 32], a1);
        a2 = fma(A[i * lda + k + 64], x[k + 64], a2);
        a3 = fma(A[i * lda + k + 96], x[k + 96], a3);
      }
      for (; k < K; k += 32) a0 = fma(A[i * lda + k], x[k], a0);
      double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) y[i] = (beta == 0.0) ? alpha * acc : fma(alpha, acc, beta * y[i]);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void copy(int n, const double* src, double* dst) {
  for (int i = threadIdx.x; i < n; i += kBT) dst[i] = src[i];
  __syncthreads();
}

// (A + A^T) / 2 in place (n x n).
__device__ __forceinline__ void symmetrize(int n, double* A, int lda) {
  for (int i = threadIdx.x >> 5; i < n; i += kBW)
    for (int j = i + 1 + (threadIdx.x & 31); j < n; j += 32) {
      const double v = 0.5 * (A[i * lda + j] + A[j * lda + i]);
      A[i * lda + j] = v;
      A[j * lda + i] = v;
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
// zeroed), factored in shared memory (dyn_smem: >= n (n + 1) doubles).
// Right-looking, one column per step.  Returns true (CTA-uniform) when a
// pivot is not positive or |L_jj| <= 1e-13 max_i |L_ii| — the reference's
// singular-factor test on the factor (linalg.cpp:54-62).
__device__ bool potrf(int n, double* A, int lda, double* red) {
  double* sm = dyn_smem();
  __shared__ double s_d[kBT];
  const int ls = n + 1;
  for (int idx = threadIdx.x; idx < n * n; idx += kBT) sm[(idx / n) * ls + idx % n] = A[(idx / n) * lda + idx % n];
  __syncthreads();
  // right-looking on unscaled columns: A(j+1) = A(j) - a_j a_j^T / d_j, one
  // barrier per column; L[i][j] = a_ij / sqrt(d_j) at the end
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  bool bad = false;
  for (int j = 0; j < n; ++j) {
    const double dj = sm[j * ls + j];
    bad |= !(dj > 0.0);
    const double inv = dj > 0.0 ? 1.0 / dj : 0.0;
    if (threadIdx.x == 0) s_d[j] = dj;
    for (int i = j + 1 + ty; i < n; i += 16) {
      const double lij = sm[i * ls + j] * inv;
      for (int k = j + 1 + tx; k <= i; k += 16) sm[i * ls + k] = fma(-lij, sm[k * ls + j], sm[i * ls + k]);
    }
    __syncthreads();
  }
  double dmax = 0.0;
  for (int idx = threadIdx.x; idx < n * n; idx += kBT) {
    const int i = idx / n, k = idx - (idx / n) * n;
    const double dk = s_d[k];
    const double v = (k > i || !(dk > 0.0)) ? 0.0 : sm[i * ls + k] / sqrt(dk);
    A[i * lda + k] = v;
    if (k == i) dmax = fmax(dmax, fabs(v));
  }
  __syncthreads();
  const double mx = block_max(dmax, red);
  double mine = bad ? 1.0 : 0.0;
  for (int i = threadIdx.x; i < n; i += kBT) mine = fmax(mine, fabs(A[i * lda + i]) <= 1e-13 * mx ? 1.0 : 0.0);
  return block_max(mine, red) > 0.0;
}

// W = L^-1 for the lower-triangular n x n L (W may alias L), inverted in
// place in shared memory (dyn_smem: >= n (n + 1) doubles) column by column from
// the right: W[i][j] = -W[j][j] sum_{k=j+1..i} W[i][k] L[k][j].
__device__ void trtri_lower(int n, const double* L, int ldl, double* W, int ldw) {
  double* sl = dyn_smem();
  const int ls = n + 1;
  double* sw = sl + n * ls;
  for (int idx = threadIdx.x; idx < n * n; idx += kBT) {
    const int i = idx / n, k = idx - (idx / n) * n;
    sl[i * ls + k] = (k > i) ? 0.0 : L[i * ldl + k];
    sw[i * ls + k] = 0.0;
  }
  __syncthreads();
  // W column j from the right: W[i][j] = -W[j][j] sum_{k=j+1..i} W[i][k] L[k][j]
  // (reads W columns > j, L column j: one barrier per column); rows split
  // over the threads, each row's dot split over 4 lanes
  const int q4 = threadIdx.x & 3, rgrp = threadIdx.x >> 2;
  for (int j = n - 1; j >= 0; --j) {
    const double inv = 1.0 / sl[j * ls + j];
    for (int base = j; base < n; base += kBT / 4) {  // warp-uniform trip count (shuffles below)
      const int i = base + rgrp;
      double acc = 0.0;
      if (i > j && i < n)
        for (int k = j + 1 + q4; k <= i; k += 4) acc = fma(sw[i * ls + k], sl[k * ls + j], acc);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (q4 == 0 && i < n) sw[i * ls + j] = (i == j) ? inv : -inv * acc;
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < n * n; idx += kBT) W[(idx / n) * ldw + idx % n] = sw[(idx / n) * ls + idx % n];
  __syncthreads();
}

// LU with partial pivoting of the n x n A, then X <- A^-1 X for the n x m
// right-hand sides (in place); A and X are staged in shared memory (dyn_smem:
// >= n (n + 1) + n (m + 1) doubles).  A is destroyed.
__device__ void lu_solve(int n, double* A, int lda, int m, double* X, int ldx) {
  double* sm = dyn_smem();
  __shared__ int s_p;
  __shared__ double s_inv;
  const int la = n + 1, lx = m + 1;
  double* sa = sm;
  double* sx = sm + n * la;
  for (int idx = threadIdx.x; idx < n * n; idx += kBT) sa[(idx / n) * la + idx % n] = A[(idx / n) * lda + idx % n];
  for (int idx = threadIdx.x; idx < n * m; idx += kBT) sx[(idx / m) * lx + idx % m] = X[(idx / m) * ldx + idx % m];
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x < 32) {  // pivot: argmax |A[i][j]|, i >= j
      double best = -1.0;
      int bi = j;
      for (int i = j + threadIdx.x; i < n; i += 32) {
        const double v = fabs(sa[i * la + j]);
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
      if (threadIdx.x == 0) {
        s_p = bi;
        s_inv = 1.0 / sa[bi * la + j];
      }
    }
    __syncthreads();
    const int p = s_p;
    if (p != j) {
      for (int k = threadIdx.x; k < n + m; k += kBT) {
        double* rj = k < n ? sa + j * la + k : sx + j * lx + (k - n);
        double* rp = k < n ? sa + p * la + k : sx + p * lx + (k - n);
        const double t = *rj;
        *rj = *rp;
        *rp = t;
      }
      __syncthreads();
    }
    const double inv = s_inv;
    const int ncol = n - j - 1;
    const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
    for (int i = j + 1 + ty; i < n; i += kBT / 16) {
      const double l = sa[i * la + j] * inv;
      for (int c = tx; c < ncol; c += 16) sa[i * la + j + 1 + c] = fma(-l, sa[j * la + j + 1 + c], sa[i * la + j + 1 + c]);
      for (int c = tx; c < m; c += 16) sx[i * lx + c] = fma(-l, sx[j * lx + c], sx[i * lx + c]);
    }
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < n; i += kBT) sa[i * la + j] *= inv;
    __syncthreads();
  }
  // back substitution U x = y, one thread per right-hand side column
  for (int c = threadIdx.x; c < m; c += kBT) {
    for (int i = n - 1; i >= 0; --i) {
      double acc = sx[i * lx + c];
      for (int k = i + 1; k < n; ++k) acc = fma(-sa[i * la + k], sx[k * lx + c], acc);
      sx[i * lx + c] = acc / sa[i * la + i];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n * m; idx += kBT) X[(idx / m) * ldx + idx % m] = sx[(idx / m) * lx + idx % m];
  __syncthreads();
}

}  // namespace big
}  // namespace pode
