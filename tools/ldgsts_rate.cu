// Probe: cp.async (LDGSTS) issue cost on one SM: W warps each issue 64 coalesced 4-byte
// (or 16 x 16-byte) copies of L2-resident data, then wait; cycles per warp-iteration.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

template <int BYTES>
__global__ void k(const float* src, long long* out, int iters) {
  extern __shared__ float sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t s0 = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + warp * 16384;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float* p = src + ((it * 8 + warp) % 64) * 4096;
    if (BYTES == 4) {
#pragma unroll
      for (int r = 0; r < 64; ++r)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s0 + (r * 32 + lane) * 4 % 16384), "l"(p + r * 32 + lane) : "memory");
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s0 + (r * 32 + lane) * 16 % 16384), "l"(p + (r * 32 + lane) * 4) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * 32 + warp] = (t1 - t0) / iters;
}

int main() {
  float* src;
  long long* out;
  cudaMalloc(&src, 64 * 4096 * 4 * 4);
  cudaMemset(src, 0, 64 * 4096 * 4 * 4);
  cudaMalloc(&out, 148 * 32 * 8);
  for (int bytes : {4, 16})
    for (int w : {1, 2, 4, 8}) {
      if (bytes == 4) {
        cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
        k<4><<<148, 32 * w, 8 * 16384>>>(src, out, 200);
      } else {
        cudaFuncSetAttribute(k<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
        k<16><<<148, 32 * w, 8 * 16384>>>(src, out, 200);
      }
      long long h[32];
      cudaMemcpy(h, out, 32 * 8, cudaMemcpyDeviceToHost);
      printf("%2d-byte cp.async, %d warps/SM (all 148 SMs): %lld cycles per 8 KB-per-warp iteration (warp 0) -> %.1f B/clk/SM (%s)\n",
             bytes, w, h[0], 8192.0 * w / h[0], cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
