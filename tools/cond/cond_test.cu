// Feasibility probe: CUDA graph with a conditional WHILE node driven from a kernel.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void body(int* counter, cudaGraphConditionalHandle h) {
  int v = atomicAdd(counter, 1) + 1;
  cudaGraphSetConditional(h, v < 10 ? 1 : 0);
}
int main() {
  int* d; cudaMalloc(&d, sizeof(int)); cudaMemset(d, 0, sizeof(int));
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  if (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) { printf("handle fail\n"); return 1; }
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  cudaError_t e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
  if (e != cudaSuccess) { printf("addnode %s\n", cudaGetErrorString(e)); return 1; }
  cudaGraph_t bodyg = p.conditional.phGraph_out[0];
  cudaStream_t s; cudaStreamCreate(&s);
  e = cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) { printf("capture %s\n", cudaGetErrorString(e)); return 1; }
  body<<<1, 1, 0, s>>>(d, h);
  cudaGraph_t tmp; e = cudaStreamEndCapture(s, &tmp);
  if (e != cudaSuccess) { printf("endcapture %s\n", cudaGetErrorString(e)); return 1; }
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0);
  if (e != cudaSuccess) { printf("inst %s\n", cudaGetErrorString(e)); return 1; }
  for (int r = 0; r < 3; ++r) {
    cudaMemset(d, 0, sizeof(int));
    cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
    int hcount = 0; cudaMemcpy(&hcount, d, sizeof(int), cudaMemcpyDeviceToHost);
    printf("run %d: body executed %d times (expect 10) %s\n", r, hcount, cudaGetErrorString(cudaGetLastError()));
  }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, s); for (int r = 0; r < 100; ++r) cudaGraphLaunch(ex, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); printf("per graph (10 iterations): %.2f us\n", ms * 10);
  return 0;
}
