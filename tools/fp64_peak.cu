// Measures the FP64 FMA (DFMA) and FP64 tensor (DMMA m8n8k4) throughput of
// this B200, the denominators of the FP64 roofline (MEASURED_PEAKS.json has
// only HBM and bf16).  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double s) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], s, 1e-7);
  }
  double t = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) t += acc[c];
  if (t == 12345.678) out[0] = t;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c0[2] = {0, 0}, c1[2] = {0, 0}, c2[2] = {0, 0}, c3[2] = {0, 0};
  for (int i = 0; i < iters; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0[0]), "+d"(c0[1]) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c1[0]), "+d"(c1[1]) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c2[0]), "+d"(c2[1]) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c3[0]), "+d"(c3[1]) : "d"(a), "d"(b));
  }
  double t = c0[0] + c0[1] + c1[0] + c1[1] + c2[0] + c2[1] + c3[0] + c3[1];
  if (t == 12345.678) out[0] = t;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 1 << 16;
  double best_dfma = 0, best_dmma = 0;
  for (int blocks_per_sm : {2, 4, 8}) {
    const int blocks = sms * blocks_per_sm, threads = 256;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.999999);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double tf = 2.0 * 8 * double(iters) * blocks * threads / (ms * 1e-3) / 1e12;
      if (tf > best_dfma) best_dfma = tf;
    }
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      dmma_kernel<<<blocks, threads>>>(out, iters / 4);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      // one m8n8k4 per warp = 2*8*8*4 flop
      const double tf = 4.0 * 2 * 8 * 8 * 4 * double(iters / 4) * blocks * (threads / 32) /
                        (ms * 1e-3) / 1e12;
      if (tf > best_dmma) best_dmma = tf;
    }
  }
  CK(cudaGetLastError());
  printf("{\"sms\": %d, \"fp64_fma_tflops\": %.3f, \"fp64_dmma_tflops\": %.3f}\n", sms, best_dfma,
         best_dmma);
  return 0;
}
