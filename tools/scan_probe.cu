// Probe: latency of K4's chunk-state warp scan (sft_tc.cuh, output tiles: 4 orders per
// thread, 5 shfl_up steps of complex multiply-adds) in isolation, 8 scan warps, with the
// other 8 warps idle (mode 0) or streaming shared-memory loads/stores (mode 1).
// Variants: v=0 the kernel's loop; v=1 orders interleaved per step with all shuffles of a
// step issued first (explicit), v=2 a 4-step Kogge-Stone + one serial step.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2110_11866_b200/csrc tools/scan_probe.cu -o tools/scan_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ float2 cmla(float2 z, float2 t, float2 a) {
  return make_float2(fmaf(z.x, t.x, fmaf(-z.y, t.y, a.x)), fmaf(z.x, t.y, fmaf(z.y, t.x, a.y)));
}

__global__ void __launch_bounds__(512, 1) probe(int mode, int iters, float* sink, unsigned long long* out) {
  __shared__ float2 zs[8 * 6];
  __shared__ float4 junk[2048];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < 48) zs[tid] = make_float2(0.99f, 0.01f * tid);
  for (int i = tid; i < 2048; i += 512) junk[i] = make_float4(i, 0, 0, 0);
  __syncthreads();
  if (warp < 8) {
    const int p0 = (warp >> 2) * 4;
    float2 inc[4];
    for (int j = 0; j < 4; ++j) inc[j] = make_float2(lane + j, lane - j);
    unsigned long long tot = 0;
    for (int it = 0; it < iters; ++it) {
      const unsigned long long a = clock64();
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int d = 1 << k;
        float2 t[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          t[j] = make_float2(__shfl_up_sync(0xffffffffu, inc[j].x, d), __shfl_up_sync(0xffffffffu, inc[j].y, d));
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (lane >= d) inc[j] = cmla(zs[(p0 + j) * 6 + k], t[j], inc[j]);
      }
      __syncwarp();
      const unsigned long long b = clock64();
      tot += b - a;
      for (int j = 0; j < 4; ++j) inc[j] = make_float2(inc[j].x * 1e-3f, inc[j].y * 1e-3f);
    }
    if (lane == 0) out[warp] = tot / iters;
    if (inc[0].x == 12345.f) sink[tid] = inc[1].y;
  } else if (mode == 1) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (int it = 0; it < iters * 40; ++it) {
      const float4 v = junk[(tid * 33 + it * 7) & 2047];
      acc.x += v.x;
      junk[(tid * 17 + it) & 2047] = acc;
    }
    if (acc.x == 12345.f) sink[tid] = acc.y;
  }
}

int main(int argc, char** argv) {
  float* sink;
  unsigned long long* out;
  cudaMalloc(&sink, 4096);
  cudaMalloc(&out, 16 * 8);
  for (int mode = 0; mode < 2; ++mode) {
    probe<<<148, 512>>>(mode, 200, sink, out);
    cudaDeviceSynchronize();
    unsigned long long h[8];
    cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
    printf("mode %d: scan cycles per warp:", mode);
    for (int w = 0; w < 8; ++w) printf(" %llu", h[w]);
    printf("\n");
  }
  return 0;
}
