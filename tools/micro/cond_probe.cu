#include <cuda_runtime.h>
#include <cstdio>
__global__ void setc(cudaGraphConditionalHandle h, const int* flag) { cudaGraphSetConditional(h, *flag ? 1u : 0u); }
__global__ void body(int* x) { atomicAdd(x, 1); }
int main() {
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h; cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault);
  int* d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  cudaGraphNode_t n1; cudaKernelNodeParams kp = {}; void* args[2] = {&h, &d}; kp.func = (void*)setc; kp.gridDim = 1; kp.blockDim = 1; kp.kernelParams = args;
  cudaGraphAddKernelNode(&n1, g, nullptr, 0, &kp);
  cudaGraphNodeParams cp = {}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeIf; cp.conditional.size = 1;
  cudaGraphNode_t n2; cudaError_t e = cudaGraphAddNode(&n2, g, &n1, 1, &cp);
  printf("add cond: %s\n", cudaGetErrorString(e));
  cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
  cudaStream_t s; cudaStreamCreate(&s);
  e = cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  printf("capture: %s\n", cudaGetErrorString(e));
  body<<<1,1,0,s>>>(d + 1);
  cudaGraph_t out; e = cudaStreamEndCapture(s, &out); printf("end: %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0); printf("inst: %s\n", cudaGetErrorString(e));
  int one = 1; cudaMemcpy(d, &one, 4, cudaMemcpyHostToDevice);
  cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  int h2[2]; cudaMemcpy(h2, d, 8, cudaMemcpyDeviceToHost); printf("body ran %d times (flag 1)\n", h2[1]);
  int zero = 0; cudaMemcpy(d, &zero, 4, cudaMemcpyHostToDevice);
  cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  cudaMemcpy(h2, d, 8, cudaMemcpyDeviceToHost); printf("body ran %d times total (flag 0 added none)\n", h2[1]);
}
