// Microbenchmark: FP32 FMA issue/throughput on sm_100a for the instruction forms K1
// uses (register FFMA, constant-bank FFMA, packed FFMA2). Prints FMAs/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>

struct C8 { float v[64]; };

template <int MODE>
__global__ void probe(float* out, int iters, const __grid_constant__ C8 c) {
  float a[8], b[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 0.001f + i; b[i] = 1.0001f + i * 1e-4f; }
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (MODE == 0) a[i] = fmaf(a[i], b[i], b[(i + 1) & 7]);          // 3 registers
        if (MODE == 1) a[i] = fmaf(a[i], c.v[(r * 8 + i) & 63], b[i]);     // constant bank operand
      }
      if (MODE == 2) {
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          unsigned long long x, y, z, rr;
          x = *reinterpret_cast<unsigned long long*>(&a[i]);
          y = *reinterpret_cast<unsigned long long*>(&b[i]);
          z = *reinterpret_cast<unsigned long long*>(&b[(i + 2) & 7]);
          asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rr) : "l"(x), "l"(y), "l"(z));
          *reinterpret_cast<unsigned long long*>(&a[i]) = rr;
        }
      }
    }
  }
  unsigned long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 1 << 26);
  C8 c; for (int i = 0; i < 64; ++i) c.v[i] = 1.0f + i * 1e-5f;
  const int iters = 2000;
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps : {4, 8, 16, 32}) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      auto launch = [&] {
        if (mode == 0) probe<0><<<sms, warps * 32>>>(out, iters, c);
        if (mode == 1) probe<1><<<sms, warps * 32>>>(out, iters, c);
        if (mode == 2) probe<2><<<sms, warps * 32>>>(out, iters, c);
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      float cyc; cudaMemcpy(&cyc, out, 4, cudaMemcpyDeviceToHost);
      double fmas = (double)sms * warps * 32 * iters * 16 * 8;
      double per_sm_clk = fmas / sms / cyc;
      printf("mode %d (%s) warps/SM %2d: %.1f FMA/clk/SM  (%.2f TFMA/s)\n", mode,
             mode == 0 ? "FFMA reg" : mode == 1 ? "FFMA const" : "FFMA2", warps, per_sm_clk, fmas / ms / 1e9);
    }
  }
  return 0;
}
