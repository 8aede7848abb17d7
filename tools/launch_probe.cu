// Probe: per-step cost of back-to-back 148-CTA kernels captured in a CUDA graph (the
// bench's step structure), with and without programmatic dependent launch (PDL), for an
// empty kernel and for one that touches HBM once per CTA (a dependent load chain).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/launch_probe.cu -o tools/launch_probe
#include <cuda_runtime.h>

#include <cstdio>

__global__ void work(const float* __restrict__ x, float* __restrict__ y, int iters, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  float a = 0.f;
  const float* p = x + blockIdx.x * 2048 + threadIdx.x;
  for (int i = 0; i < iters; ++i) a += __ldcg(p + (i & 7) * 256);
  if (iters) y[blockIdx.x * blockDim.x + threadIdx.x] = a;
}

int main() {
  float *x, *y;
  cudaMalloc(&x, 148 * 2048 * 4 * 2);
  cudaMalloc(&y, 148 * 1024 * 4);
  cudaMemset(x, 0, 148 * 2048 * 4 * 2);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int steps = 200;
  for (int iters : {0, 8}) {
    for (int threads : {128, 512}) {
      for (int pdl : {0, 1}) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int k = 0; k < steps; ++k) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(148);
          cfg.blockDim = dim3(threads);
          cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = pdl ? 1 : 0;
          cudaLaunchKernelEx(&cfg, work, (const float*)x, y, iters, pdl);
        }
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
        cudaEventRecord(a, s);
        for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("iters %d threads %d pdl %d: %.3f us per step (%s)\n", iters, threads, pdl, 1000.f * ms / (5 * steps),
               cudaGetErrorString(cudaGetLastError()));
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
      }
    }
  }
  return 0;
}
