// Probe: does a thread blocked in TMA box issue (UTMALDG) or in tcgen05.mma issue slow
// down the shuffles of other warps on the same SM sub-partition? Warp 0 lane 0 streams
// TMA box loads (129 x 32 fp32, SW128) through a 3-slot ring; warps 4 (same
// sub-partition as warp 0) and 5 (another one) time a dependent 512-step SHFL chain.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2110_11866_b200/csrc tools/mio_probe.cu -lcuda -o tools/mio_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "umma.cuh"

__global__ void __launch_bounds__(256, 1) probe(const __grid_constant__ CUtensorMap in_map, int tma, int q, int pol_mode,
                                                 unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = raw + ((1024u - (umma::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[3];
  __shared__ int stop;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int k = 0; k < 3; ++k) umma::mbar_init(&full[k], 1);
    umma::mbar_fence_init();
    stop = 0;
  }
  __syncthreads();
  unsigned long long pol = 0;
  if (pol_mode == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  if (pol_mode == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (warp == 0) {
    if (lane == 0 && tma) {
      uint32_t ph = 0;
      long long g = 0, issued = 0;
      unsigned long long t_issue = 0;
      for (; g < 400 && !stop; ++g) {
        const int slot = static_cast<int>(g % 3);
        if (g >= 3) {
          umma::mbar_wait(&full[slot], (ph >> slot) & 1u);
          ph ^= 1u << slot;
        }
        const long long al = (blockIdx.x * 97 + g * 128) % 3000 * 32;
        const unsigned long long a = clock64();
        umma::mbar_arrive_tx(&full[slot], 16512u);
        umma::tma_load_3d(umma::smem_u32(sm + slot * 17408), &in_map, &full[slot], q, static_cast<int>(al >> 5),
                          static_cast<int>(blockIdx.x), pol);
        t_issue += clock64() - a;
        ++issued;
      }
      if (blockIdx.x == 0) out[2] = t_issue / (issued ? issued : 1);
    }
  } else if (warp == 4 || warp == 5) {
    // wait a little so the TMA stream is running
    const unsigned long long t0 = clock64();
    while (clock64() - t0 < 20000) {
    }
    float v = static_cast<float>(lane);
    const unsigned long long a = clock64();
#pragma unroll 1
    for (int i = 0; i < 512; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1 + (i & 15)) + 1.0f;
    const unsigned long long b = clock64();
    if (lane == 0 && blockIdx.x == 0) out[warp - 4] = (b - a) / 512 + (v == -1.f ? 1 : 0);
    if (warp == 5 && lane == 0) stop = 1;
  }
}

int main(int argc, char** argv) {
  const long long n = 102400;
  float* x;
  cudaMalloc(&x, 148 * n * 4);
  cudaMemset(x, 0, 148 * n * 4);
  unsigned long long* out;
  cudaMalloc(&out, 24);
  CUtensorMap in_map;
  const cuuint64_t dims[3] = {64, 3199, 148};
  const cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(n * 4)};
  const cuuint32_t box[3] = {32, 129, 1}, es[3] = {1, 1, 1};
  if (cuTensorMapEncodeTiled(&in_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
    return 1;
  const int smem = 3 * 17408 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int q = argc > 1 ? atoi(argv[1]) : 0, pm = argc > 2 ? atoi(argv[2]) : 0;
  for (int tma = 1; tma < 2; ++tma) {
    cudaMemset(out, 0, 24);
    probe<<<148, 256, smem>>>(in_map, tma, q, pm, out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[3];
    cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
    printf("q=%d pol=%d tma=%d (%s): shfl step same-SMSP %llu cycles, other-SMSP %llu cycles, TMA issue %llu cycles\n", q, pm, tma,
           cudaGetErrorString(e), h[0], h[1], h[2]);
  }
  return 0;
}
