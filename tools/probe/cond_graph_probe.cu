#include <cuda_runtime.h>
#include <cstdio>
__global__ void body_k(int* ctr) { atomicAdd(ctr, 1); }
__global__ void cond_k(cudaGraphConditionalHandle h, int* ctr, int n) {
  cudaGraphSetConditional(h, *ctr < n ? 1 : 0);
}
int main() {
  int* ctr; cudaMalloc(&ctr, 4); cudaMemset(ctr, 0, 4);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  cudaError_t e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
  printf("add %s\n", cudaGetErrorString(e));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  printf("cap %s\n", cudaGetErrorString(e));
  body_k<<<1,1,0,s>>>(ctr);
  cond_k<<<1,1,0,s>>>(h, ctr, 7);
  e = cudaStreamEndCapture(s, &body);
  printf("end %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0);
  printf("inst %s\n", cudaGetErrorString(e));
  e = cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  int v; cudaMemcpy(&v, ctr, 4, cudaMemcpyDeviceToHost);
  printf("launch %s ctr=%d\n", cudaGetErrorString(e), v);
}
