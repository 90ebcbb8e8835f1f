// Dependent-kernel gap inside a CUDA graph, with and without programmatic
// dependent launch (PDL).  N kernels in one stream, each reading what the
// previous one wrote (one CTA per SM, a few us of work or none).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step_kernel(float* buf, int n, int iters, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    float v = buf[i];
    for (int k = 0; k < iters; ++k) v = v * 0.999f + 0.001f;
    buf[i] = v;
  }
}

static float run(int chain, int iters, int pdl, int blocks) {
  float* buf;
  cudaMalloc(&buf, 148 * 256 * 16 * sizeof(float));
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaGraph_t g;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int c = 0; c < chain; ++c) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, step_kernel, buf, blocks * 256, iters, pdl);
  }
  cudaStreamEndCapture(st, &g);
  cudaGraphExec_t ex;
  cudaGraphInstantiate(&ex, g, 0);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ex, st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (int r = 0; r < 10; ++r) cudaGraphLaunch(ex, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(buf);
  return ms * 1000.f / (10 * chain);
}

int main() {
  for (int blocks : {148, 148 * 4})
    for (int iters : {0, 200, 2000})
      printf("blocks %4d iters %5d: plain %.2f us/kernel  pdl %.2f us/kernel\n", blocks, iters,
             run(200, iters, 0, blocks), run(200, iters, 1, blocks));
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
