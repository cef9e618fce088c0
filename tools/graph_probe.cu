#include <cuda_runtime.h>
#include <cstdio>
__global__ void k_cond(cudaGraphConditionalHandle h, int* cnt) {
  int c = ++(*cnt);
  cudaGraphSetConditional(h, c < 5 ? 1u : 0u);
}
extern "C" int run() {
  cudaStream_t s; cudaStreamCreate(&s);
  int* d; cudaMalloc(&d, 4); cudaMemset(d, 0, 4);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
  cudaGraphNode_t n; cudaGraphAddNode(&n, g, nullptr, 0, &p);
  cudaGraph_t body = p.conditional.phGraph_out[0];
  cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  k_cond<<<1,1,0,s>>>(h, d);
  cudaStreamEndCapture(s, &body);
  cudaGraphExec_t e; cudaError_t r = cudaGraphInstantiate(&e, g, 0);
  if (r) { printf("inst %s\n", cudaGetErrorString(r)); return 1; }
  cudaGraphLaunch(e, s); cudaStreamSynchronize(s);
  int hv; cudaMemcpy(&hv, d, 4, cudaMemcpyDeviceToHost);
  printf("count %d err %s\n", hv, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
int main() { return run(); }
