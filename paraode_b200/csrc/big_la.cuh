// CTA-wide dense fp64 linear algebra for large state dimensions (D ~ 100,
// Pleiades D = 112): the operands of one IEKS time step are 12 K-entry
// matrices, so one CTA (kBT threads) owns one chunk and works on matrices
// that live in its global-memory workspace (L2-resident) and its shared
// memory.  Products run on the FP64 tensor pipe (DMMA, mma.sync m8n8k4
// .f64): at this size they are real dense contractions (SURVEY.md §8(d):
// AI ~ 200 flop/B).  Cholesky and the triangular solves are blocked (8-wide
// panels, DMMA trailing updates) on matrices resident in shared memory at a
// bank-conflict-free stride (smem_ld); global operands arrive by cp.async.
// The chain kernels' LU (partial pivoting) is column-serial.
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
  extern __shared__ __align__(16) double big_dyn_smem[];
  return big_dyn_smem;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// Asynchronous global -> shared copies (cp.async, 16 bytes each): all of a
// matrix in flight at once, no registers, then one wait + barrier.
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// dst (rows x cols, stride ldd) <- src (stride lds).  Global -> shared with
// even strides and 16-byte aligned bases: cp.async; otherwise 8 loads in
// flight per thread (generic pointers: without batching every load waits
// on the previous store).
__device__ __forceinline__ void stage(int rows, int cols, const double* src, int lds, double* dst, int ldd) {
  const bool async = __isGlobal(src) && __isShared(dst) && !(cols & 1) && !(lds & 1) && !(ldd & 1) &&
                     !(reinterpret_cast<uintptr_t>(src) & 15) && !(reinterpret_cast<uintptr_t>(dst) & 15);
  if (async) {
    const int h = cols >> 1;
    for (int idx = threadIdx.x; idx < rows * h; idx += kBT) {
      const int r = idx / h, q = idx - r * h;
      cp_async16(dst + r * ldd + 2 * q, src + r * lds + 2 * q);
    }
    cp_async_wait_all();
    __syncthreads();
    return;
  }
  const int n = rows * cols;
  for (int base = threadIdx.x; base < n; base += 8 * kBT) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * kBT;
      v[u] = idx < n ? src[(idx / cols) * lds + idx % cols] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * kBT;
      if (idx < n) dst[(idx / cols) * ldd + idx % cols] = v[u];
    }
  }
  __syncthreads();
}

// Z = alpha X + beta Y + gamma I (n x n, stride n; Z may alias X or Y),
// 8 elements in flight per thread.
__device__ __forceinline__ void axpby_eye(int n, double alpha, const double* X, double beta, const double* Y,
                                          double gamma, double* Z) {
  const int nn = n * n;
  for (int base = threadIdx.x; base < nn; base += 8 * kBT) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * kBT;
      v[u] = 0.0;
      if (idx < nn) {
        v[u] = alpha * X[idx];
        if (Y) v[u] = fma(beta, Y[idx], v[u]);
        if (idx / n == idx % n) v[u] += gamma;
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * kBT;
      if (idx < nn) Z[idx] = v[u];
    }
  }
  __syncthreads();
}

// C[M x N] = alpha op(A)[M x K] op(B)[K x N] + beta C (beta = 0: C is not
// read).  op(X) = X^T when TX.  M, K any; N <= 8 * kNT.  op(B) is staged in
// shared memory (dyn_smem: >= K (N + 1) doubles, odd row stride: conflict-free
// fragment reads); each warp owns 8-row blocks of C and sweeps all N/8
// column tiles with its A panel in registers (one DMMA m8n8k4 per tile
// per k-step; the panel's fragments all loaded up front).  C must not alias A or B.
constexpr int kNT = 16;  // N <= 128

// Row stride of a shared-memory matrix with n columns: >= n and = 4 mod 16
// doubles, so the 8 x 4 DMMA fragment reads (8 rows x 4 columns, or 4 rows x
// 8 columns) of a half-warp hit 16 distinct 8-byte bank pairs.
__host__ __device__ constexpr int smem_ld(int n) { return ((n + 11) / 16) * 16 + 4; }

// The DMMA core with op(B) already in shared memory (Bs, K x N, stride ldbs).
template <bool TA>
__device__ void gemm_core(int M, int N, int K, double alpha, const double* A, int lda, const double* sm, int ldb_s,
                          double beta, double* C, int ldc);

template <bool TA, bool TB>
__device__ void gemm(int M, int N, int K, double alpha, const double* A, int lda, const double* B, int ldb,
                     double beta, double* C, int ldc) {
  double* sm = dyn_smem();
  const int ldb_s = smem_ld(N);
  if (!TB) {
    stage(K, N, B, ldb, sm, ldb_s);
  } else {  // B stored N x K: read along k, 8 loads in flight
    for (int base = threadIdx.x; base < K * N; base += 8 * kBT) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = base + u * kBT;
        v[u] = idx < K * N ? B[(idx / K) * ldb + idx % K] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = base + u * kBT;
        if (idx < K * N) sm[(idx % K) * ldb_s + idx / K] = v[u];
      }
    }
    __syncthreads();
  }
  gemm_core<TA>(M, N, K, alpha, A, lda, sm, ldb_s, beta, C, ldc);
}

template <bool TA>
__device__ void gemm_core(int M, int N, int K, double alpha, const double* A, int lda, const double* sm, int ldb_s,
                          double beta, double* C, int ldc) {
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
    // the warp's whole 8 x 112 A panel in registers first (28 fragments in
    // flight), then 28 k-steps of nt independent DMMA chains
    for (int kb0 = 0; kb0 < K; kb0 += 112) {
      double af[28];
#pragma unroll
      for (int q = 0; q < 28; ++q) af[q] = lda_at(kb0 + q * 4 + tg);
#pragma unroll
      for (int q = 0; q < 28; ++q) {
        const int kb = kb0 + q * 4 + tg;
        if (kb0 + q * 4 < K) {
          const bool kin = kb < K;
#pragma unroll
          for (int t = 0; t < kNT; ++t) {
            if (t < nt) {
              const int col = t * 8 + gr;
              const double b = (kin && col < N) ? sm[kb * ldb_s + col] : 0.0;
              dmma(acc[t][0], acc[t][1], af[q], b, acc[t][0], acc[t][1]);
            }
          }
        }
      }
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
    constexpr int R = 4, C = 4;  // rows per warp pass, 32-column chunks per load batch (K <= 128 in one batch)
    for (int i0 = warp * R; i0 < M; i0 += kBW * R) {
      double acc[R];
#pragma unroll
      for (int u = 0; u < R; ++u) acc[u] = 0.0;
      for (int kb = 0; kb < K; kb += 32 * C) {
        double v[R][C];
#pragma unroll
        for (int u = 0; u < R; ++u)
#pragma unroll
          for (int q = 0; q < C; ++q) {
            const int k = kb + q * 32 + lane, i = i0 + u;
            v[u][q] = (i < M && k < K) ? A[i * lda + k] * x[k] : 0.0;
          }
#pragma unroll
        for (int u = 0; u < R; ++u)
#pragma unroll
          for (int q = 0; q < C; ++q) acc[u] += v[u][q];
      }
#pragma unroll
      for (int u = 0; u < R; ++u) {
        double t = acc[u];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        const int i = i0 + u;
        if (lane == 0 && i < M) y[i] = (beta == 0.0) ? alpha * t : fma(alpha, t, beta * y[i]);
      }
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

// LU with partial pivoting of the n x n A, then X <- A^-1 X for the n x m
// right-hand sides (in place).  [A | X] is staged in shared memory as one
// augmented n x (n + m) matrix (dyn_smem: n smem_ld(n + m) doubles), so the
// eliminations carry the right-hand sides along.  Blocked: 8-column panels
// (per column: pivot found by every warp, one row swap, one rank-1 update
// of the panel: 2 barriers), the panel's rows of U by an 8-row unit-lower
// solve, the trailing update (right-hand sides included) a DMMA rank-8
// product; then a blocked back substitution on DMMA.  A is not modified.
__device__ void lu_solve(int n, const double* A, int lda, int m, double* X, int ldx) {
  __shared__ double s_rd[128];
  double* g = dyn_smem();
  const int nm = n + m, lg = smem_ld(nm);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gr = lane >> 2, tg = lane & 3;
  stage(n, n, A, lda, g, lg);
  stage(n, m, X, ldx, g + n, lg);
  for (int j0 = 0; j0 < n; j0 += 8) {
    const int w = min(8, n - j0);
    for (int c = 0; c < w; ++c) {
      const int j = j0 + c;
      double best = -1.0;
      int bi = j;
      for (int i = j + lane; i < n; i += 32) {
        const double v = fabs(g[i * lg + j]);
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
      if (bi != j) {
        for (int t = threadIdx.x; t < nm; t += kBT) {
          const double x = g[j * lg + t];
          g[j * lg + t] = g[bi * lg + t];
          g[bi * lg + t] = x;
        }
      }
      __syncthreads();
      const double inv = 1.0 / g[j * lg + j];
      for (int i = j + 1 + threadIdx.x; i < n; i += kBT) {
        const double l = g[i * lg + j] * inv;
        g[i * lg + j] = l;
        for (int k = j + 1; k < j0 + w; ++k) g[i * lg + k] = fma(-l, g[j * lg + k], g[i * lg + k]);
      }
      __syncthreads();
    }
    const int t0 = j0 + w;
    if (t0 < nm) {
      // U12 = L11^-1 A12 on the panel rows, one column per thread
      for (int t = t0 + threadIdx.x; t < nm; t += kBT) {
        double u[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          if (r < w) {
            double acc = g[(j0 + r) * lg + t];
#pragma unroll
            for (int r2 = 0; r2 < r; ++r2) acc = fma(-g[(j0 + r) * lg + j0 + r2], u[r2], acc);
            u[r] = acc;
            g[(j0 + r) * lg + t] = acc;
          }
        }
      }
      __syncthreads();
      // A22 -= L21 U12 (rows >= t0, columns >= t0 incl. right-hand sides)
      if (t0 < n) {
        const int rt = (n - t0 + 7) / 8, ct = (nm - t0 + 7) / 8;
        for (int q = warp; q < rt * ct; q += kBW) {
          const int ti = q / ct, tj = q - ti * ct;
          const int rr = t0 + ti * 8 + gr, cc = t0 + tj * 8 + 2 * tg, bc = t0 + tj * 8 + gr;
          double c0 = (rr < n && cc < nm) ? g[rr * lg + cc] : 0.0;
          double c1 = (rr < n && cc + 1 < nm) ? g[rr * lg + cc + 1] : 0.0;
#pragma unroll
          for (int kk = 0; kk < 8; kk += 4) {
            if (kk < w) {
              const int k = j0 + kk + tg;
              const double a = (rr < n && kk + tg < w) ? -g[rr * lg + k] : 0.0;
              const double b = (bc < nm && kk + tg < w) ? g[k * lg + bc] : 0.0;
              dmma(c0, c1, a, b, c0, c1);
            }
          }
          if (rr < n && cc < nm) g[rr * lg + cc] = c0;
          if (rr < n && cc + 1 < nm) g[rr * lg + cc + 1] = c1;
        }
        __syncthreads();
      }
    }
  }
  // back substitution U Xs = Y (Y = columns n.. of g), row blocks bottom-up
  for (int j = threadIdx.x; j < n; j += kBT) s_rd[j] = 1.0 / g[j * lg + j];
  __syncthreads();
  double* y = g + n;
  const int nblk = (n + 7) / 8;
  for (int bb = nblk - 1; bb >= 0; --bb) {
    const int ib = bb * 8, w = min(8, n - ib), k0s = ib + w;
    if (k0s < n) {  // Y[ib:ib+w, :] -= U[ib:ib+w, k0s:n] X[k0s:n, :]
      for (int ct = warp; ct * 8 < m; ct += kBW) {
        const int r = ib + gr, cc = ct * 8 + 2 * tg, bc = ct * 8 + gr;
        const bool rin = gr < w;
        double c0 = (rin && cc < m) ? y[r * lg + cc] : 0.0;
        double c1 = (rin && cc + 1 < m) ? y[r * lg + cc + 1] : 0.0;
        double e0 = 0.0, e1 = 0.0;
        for (int k0 = k0s; k0 < n; k0 += 8) {
          const int k = k0 + tg, k2 = k0 + 4 + tg;
          const double a = (rin && k < n) ? -g[r * lg + k] : 0.0;
          const double b = (k < n && bc < m) ? y[k * lg + bc] : 0.0;
          const double a2 = (rin && k2 < n) ? -g[r * lg + k2] : 0.0;
          const double b2 = (k2 < n && bc < m) ? y[k2 * lg + bc] : 0.0;
          dmma(c0, c1, a, b, c0, c1);
          dmma(e0, e1, a2, b2, e0, e1);
        }
        if (rin && cc < m) y[r * lg + cc] = c0 + e0;
        if (rin && cc + 1 < m) y[r * lg + cc + 1] = c1 + e1;
      }
      __syncthreads();
    }
    for (int t = threadIdx.x; t < m; t += kBT) {
      double x[8];
#pragma unroll
      for (int r = 7; r >= 0; --r) {
        if (r < w) {
          double acc = y[(ib + r) * lg + t];
#pragma unroll
          for (int r2 = 7; r2 > r; --r2)
            if (r2 < w) acc = fma(-g[(ib + r) * lg + ib + r2], x[r2], acc);
          x[r] = acc * s_rd[ib + r];
          y[(ib + r) * lg + t] = x[r];
        }
      }
    }
    __syncthreads();
  }
  stage(n, m, y, lg, X, ldx);
}

// ------------------------------------------------ blocked, smem-resident ---
// A column-serial factorisation pays one CTA barrier and one pass of
// shared-memory latency per column.  The blocked forms below work on
// matrices already staged in shared memory (stride ls), 8 columns per panel:
// the panel is factored column by column on its 8 columns only, the trailing
// update is a DMMA rank-8 product.

// In-place lower Cholesky of the n x n SPD matrix in shared memory (upper
// part undefined on return).  Panel columns are kept unscaled while the
// panel factors (A <- A - a_j a_j^T / d_j), then scaled by 1/sqrt(d_j).
// Returns true (CTA-uniform) on a non-positive pivot or |L_jj| <= 1e-13 max.
__device__ bool potrf_smem(int n, double* sa, int ls, double* red) {
  __shared__ double s_piv[128];     // pivots d_j
  __shared__ double s_col[2][8];    // column j of the diagonal block (double-buffered)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gr = lane >> 2, tg = lane & 3;
  bool bad = false;
  for (int jb = 0; jb < n; jb += 8) {
    const int w = min(8, n - jb);
    // panel: thread t owns row jb + t (columns jb..jb+w-1 in registers)
    const int t = threadIdx.x, i = jb + t;
    const bool own = i < n;
    double r[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) r[c] = (own && c < w) ? sa[i * ls + jb + c] : 0.0;
    if (t < w) s_col[0][t] = r[0];
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c < w) {
        const double* col = s_col[c & 1];
        const double dj = col[c];  // a_jj (updated), j = jb + c
        const double inv = dj > 0.0 ? 1.0 / dj : 0.0;
        bad |= !(dj > 0.0);
        if (t == 0) s_piv[jb + c] = dj;
        // a_ik -= a_ij a_kj / d_j for the panel columns k > j (rows i > j)
        const double lij = r[c] * inv;
#pragma unroll
        for (int c2 = c + 1; c2 < 8; ++c2)
          if (c2 < w && t > c) r[c2] = fma(-lij, col[c2], r[c2]);
        if (c + 1 < w && t < w) s_col[(c + 1) & 1][t] = r[c + 1];
        __syncthreads();
      }
    }
    // scale: L_ij = a_ij / sqrt(d_j) on and below the diagonal
    if (own) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < w && c <= t) {
          const double dj = s_piv[jb + c];
          sa[i * ls + jb + c] = dj > 0.0 ? r[c] * rsqrt(dj) : 0.0;
        }
    }
    __syncthreads();
    // trailing update A22 -= L21 L21^T (lower tiles), rank w, on DMMA
    const int r0b = jb + w, M = n - r0b;
    if (M > 0) {
      const int tiles = (M + 7) / 8;
      int ti = 0, base = 0;  // tile (ti, tj), tj <= ti, flat index q = base + tj
      for (int q = warp; q < tiles * (tiles + 1) / 2; q += kBW) {
        while (q >= base + ti + 1) base += ++ti;
        const int tj = q - base;
        const int rr = r0b + ti * 8 + gr, cc = r0b + tj * 8 + 2 * tg;
        double c0 = (rr < n && cc < n) ? sa[rr * ls + cc] : 0.0;
        double c1 = (rr < n && cc + 1 < n) ? sa[rr * ls + cc + 1] : 0.0;
        const int rb = r0b + tj * 8 + gr;  // B column (L21 row) for this lane
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4) {
          if (kk < w) {
            const int k = jb + kk + tg;
            const double a = (rr < n && kk + tg < w) ? -sa[rr * ls + k] : 0.0;
            const double b = (rb < n && kk + tg < w) ? sa[rb * ls + k] : 0.0;
            dmma(c0, c1, a, b, c0, c1);
          }
        }
        if (rr < n && cc < n) sa[rr * ls + cc] = c0;
        if (rr < n && cc + 1 < n) sa[rr * ls + cc + 1] = c1;
      }
      __syncthreads();
    }
  }
  double dmax = 0.0;
  for (int i = threadIdx.x; i < n; i += kBT) dmax = fmax(dmax, fabs(sa[i * ls + i]));
  const double mx = block_max(dmax, red);
  double mine = bad ? 1.0 : 0.0;
  for (int i = threadIdx.x; i < n; i += kBT) mine = fmax(mine, fabs(sa[i * ls + i]) <= 1e-13 * mx ? 1.0 : 0.0);
  return block_max(mine, red) > 0.0;
}

// X L^T = Y in place (Y: m x n in shared memory, stride ly; L: n x n lower in
// shared memory, stride ll): column blocks of 8 left to right, the update
// by the solved blocks on DMMA, the 8-wide diagonal solve one row per thread.
__device__ void trsm_right_lower_t(int m, int n, const double* sl, int ll, double* sy, int ly) {
  __shared__ double s_rd[128];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gr = lane >> 2, tg = lane & 3;
  for (int j = threadIdx.x; j < n; j += kBT) s_rd[j] = 1.0 / sl[j * ll + j];
  __syncthreads();
  for (int jb = 0; jb < n; jb += 8) {
    const int w = min(8, n - jb);
    if (jb > 0) {  // Y[:, jb:jb+w] -= X[:, 0:jb] L[jb:jb+w, 0:jb]^T
      for (int rt = warp; rt * 8 < m; rt += kBW) {
        const int r = rt * 8 + gr, cc = jb + 2 * tg;
        double c0 = (r < m && 2 * tg < w) ? sy[r * ly + cc] : 0.0;
        double c1 = (r < m && 2 * tg + 1 < w) ? sy[r * ly + cc + 1] : 0.0;
        const int lrow = jb + gr;  // B[k][col] = L[jb + col][k]
        double e0 = 0.0, e1 = 0.0;  // second accumulation chain (jb is a multiple of 8)
        for (int k0 = 0; k0 < jb; k0 += 8) {
          const double a = r < m ? -sy[r * ly + k0 + tg] : 0.0;
          const double b = gr < w ? sl[lrow * ll + k0 + tg] : 0.0;
          const double a2 = r < m ? -sy[r * ly + k0 + 4 + tg] : 0.0;
          const double b2 = gr < w ? sl[lrow * ll + k0 + 4 + tg] : 0.0;
          dmma(c0, c1, a, b, c0, c1);
          dmma(e0, e1, a2, b2, e0, e1);
        }
        c0 += e0;
        c1 += e1;
        if (r < m && 2 * tg < w) sy[r * ly + cc] = c0;
        if (r < m && 2 * tg + 1 < w) sy[r * ly + cc + 1] = c1;
      }
      __syncthreads();
    }
    for (int r = threadIdx.x; r < m; r += kBT) {  // x L_bb^T = y on the block
      double x[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < w) {
          double acc = sy[r * ly + jb + c];
#pragma unroll
          for (int c2 = 0; c2 < c; ++c2) acc = fma(-x[c2], sl[(jb + c) * ll + jb + c2], acc);
          x[c] = acc * s_rd[jb + c];
          sy[r * ly + jb + c] = x[c];
        }
      }
    }
    __syncthreads();
  }
}

// X L = Z in place (Z: m x n in shared memory; L lower): column blocks right
// to left, the update by the solved blocks on DMMA.
__device__ void trsm_right_lower_n(int m, int n, const double* sl, int ll, double* sy, int ly) {
  __shared__ double s_rd[128];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gr = lane >> 2, tg = lane & 3;
  for (int j = threadIdx.x; j < n; j += kBT) s_rd[j] = 1.0 / sl[j * ll + j];
  __syncthreads();
  const int nblk = (n + 7) / 8;
  for (int bb = nblk - 1; bb >= 0; --bb) {
    const int jb = bb * 8, w = min(8, n - jb), kstart = jb + w;
    if (kstart < n) {  // Z[:, jb:jb+w] -= X[:, kstart:n] L[kstart:n, jb:jb+w]
      for (int rt = warp; rt * 8 < m; rt += kBW) {
        const int r = rt * 8 + gr, cc = jb + 2 * tg;
        double c0 = (r < m && 2 * tg < w) ? sy[r * ly + cc] : 0.0;
        double c1 = (r < m && 2 * tg + 1 < w) ? sy[r * ly + cc + 1] : 0.0;
        double e0 = 0.0, e1 = 0.0;  // second accumulation chain
        for (int k0 = kstart; k0 < n; k0 += 8) {
          const int k = k0 + tg, k2 = k0 + 4 + tg;
          const double a = (r < m && k < n) ? -sy[r * ly + k] : 0.0;
          const double b = (k < n && gr < w) ? sl[k * ll + jb + gr] : 0.0;  // B[k][col] = L[k][jb + col]
          const double a2 = (r < m && k2 < n) ? -sy[r * ly + k2] : 0.0;
          const double b2 = (k2 < n && gr < w) ? sl[k2 * ll + jb + gr] : 0.0;
          dmma(c0, c1, a, b, c0, c1);
          dmma(e0, e1, a2, b2, e0, e1);
        }
        c0 += e0;
        c1 += e1;
        if (r < m && 2 * tg < w) sy[r * ly + cc] = c0;
        if (r < m && 2 * tg + 1 < w) sy[r * ly + cc + 1] = c1;
      }
      __syncthreads();
    }
    for (int r = threadIdx.x; r < m; r += kBT) {  // x L_bb = z on the block
      double x[8];
#pragma unroll
      for (int c = 7; c >= 0; --c) {
        if (c < w) {
          double acc = sy[r * ly + jb + c];
#pragma unroll
          for (int c2 = 7; c2 > c; --c2)
            if (c2 < w) acc = fma(-x[c2], sl[(jb + c2) * ll + jb + c], acc);
          x[c] = acc * s_rd[jb + c];
          sy[r * ly + jb + c] = x[c];
        }
      }
    }
    __syncthreads();
  }
}

// L X = B in place (B: n x m in shared memory, stride lx; L: n x n lower,
// stride ll): row blocks of 8 top to bottom, the update by the solved rows on
// DMMA (warps over 8-column tiles), the 8-row forward substitution one
// column per thread.
__device__ void trsm_left_lower(int n, int m, const double* sl, int ll, double* sx, int lx) {
  __shared__ double s_rd[128];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gr = lane >> 2, tg = lane & 3;
  for (int j = threadIdx.x; j < n; j += kBT) s_rd[j] = 1.0 / sl[j * ll + j];
  __syncthreads();
  for (int ib = 0; ib < n; ib += 8) {
    const int w = min(8, n - ib);
    if (ib > 0) {  // X[ib:ib+w, :] -= L[ib:ib+w, 0:ib] X[0:ib, :]
      for (int ct = warp; ct * 8 < m; ct += kBW) {
        const int r = ib + gr, cc = ct * 8 + 2 * tg;
        const bool rin = gr < w;
        double c0 = (rin && cc < m) ? sx[r * lx + cc] : 0.0;
        double c1 = (rin && cc + 1 < m) ? sx[r * lx + cc + 1] : 0.0;
        const int bc = ct * 8 + gr;  // B[k][col] = X[k][ct 8 + col]
        for (int k0 = 0; k0 < ib; k0 += 4) {
          const double a = rin ? -sl[r * ll + k0 + tg] : 0.0;
          const double b = bc < m ? sx[(k0 + tg) * lx + bc] : 0.0;
          dmma(c0, c1, a, b, c0, c1);
        }
        if (rin && cc < m) sx[r * lx + cc] = c0;
        if (rin && cc + 1 < m) sx[r * lx + cc + 1] = c1;
      }
      __syncthreads();
    }
    for (int j = threadIdx.x; j < m; j += kBT) {
      double x[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < w) {
          double acc = sx[(ib + c) * lx + j];
#pragma unroll
          for (int c2 = 0; c2 < c; ++c2) acc = fma(-sl[(ib + c) * ll + ib + c2], x[c2], acc);
          x[c] = acc * s_rd[ib + c];
          sx[(ib + c) * lx + j] = x[c];
        }
      }
    }
    __syncthreads();
  }
}
}  // namespace big
}  // namespace pode
