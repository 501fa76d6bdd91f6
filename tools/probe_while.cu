#include <cuda_runtime.h>
#include <cstdio>
__global__ void ctl(cudaGraphConditionalHandle h, int* ctr, int n) {
  int c = ++(*ctr);
  cudaGraphSetConditional(h, c < n ? 1u : 0u);
}
__global__ void body(float* x) { x[threadIdx.x] += 1.f; }
int main() {
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
  cudaGraphNode_t n; cudaGraphAddNode(&n, g, nullptr, 0, &p);
  cudaGraph_t b = p.conditional.phGraph_out[0];
  cudaStream_t s; cudaStreamCreate(&s);
  float* x; int* ctr; cudaMalloc(&x, 128); cudaMalloc(&ctr, 4); cudaMemset(ctr, 0, 4); cudaMemset(x,0,128);
  cudaStreamBeginCaptureToGraph(s, b, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  body<<<1, 32, 0, s>>>(x);
  ctl<<<1, 1, 0, s>>>(h, ctr, 10);
  cudaGraph_t out; cudaError_t e = cudaStreamEndCapture(s, &out);
  printf("capture %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0); printf("inst %s\n", cudaGetErrorString(e));
  cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  float hx; cudaMemcpy(&hx, x, 4, cudaMemcpyDeviceToHost); printf("x = %f (expect 10)\n", hx);
}
