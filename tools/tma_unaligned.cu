// Probe: does a TMA tile box start at an arbitrary (not 16-byte aligned) element coordinate?
// View [row][64 floats], rows 128 B apart (overlapping), box 32 x 64 rows, SWIZZLE_128B.
// nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2110_11866_b200/csrc tools/tma_unaligned.cu -o /tmp/tu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "umma.cuh"
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap map, int c0, int r0, float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    umma::mbar_init(&bar, 1);
    umma::mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    umma::mbar_arrive_tx(&bar, 64 * 128);
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(umma::smem_u32(sm)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(r0), "r"(0),
                 "r"(umma::smem_u32(&bar)) : "memory");
  }
  umma::mbar_wait(&bar, 0);
  for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {
    const int row = e / 32, i = e % 32, q = i / 4;
    out[e] = *reinterpret_cast<const float*>(sm + row * 128 + ((q ^ (row & 7)) << 4) + (i % 4) * 4);
  }
}
int main() {
  const int n = 8192;
  std::vector<float> h(n);
  for (int i = 0; i < n; ++i) h[i] = static_cast<float>(i);
  float *x, *o;
  cudaMalloc(&x, n * 4);
  cudaMalloc(&o, 64 * 32 * 4);
  cudaMemcpy(x, h.data(), n * 4, cudaMemcpyHostToDevice);
  void* p;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncFn enc = reinterpret_cast<EncFn>(p);
  CUtensorMap map;
  const cuuint64_t dims[3] = {64, static_cast<cuuint64_t>((n - 64) / 32 + 1), 1}, strides[2] = {128, n * 4ull};
  const cuuint32_t box[3] = {32, 64, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", static_cast<int>(r));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 128 + 1024);
  int bad_total = 0;
  for (int c0 = 0; c0 < 32; ++c0) {
    k<<<1, 128, 64 * 128 + 1024>>>(map, c0, 3, o);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> g(64 * 32);
    cudaMemcpy(g.data(), o, g.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int row = 0; row < 64; ++row)
      for (int i = 0; i < 32; ++i)
        if (g[row * 32 + i] != static_cast<float>(32 * (3 + row) + c0 + i)) ++bad;
    printf("c0=%2d err=%s bad=%d first=%g\n", c0, cudaGetErrorString(e), bad, g[0]);
    bad_total += bad;
    if (e != cudaSuccess) return 1;
  }
  printf("TOTAL_BAD %d\n", bad_total);
}
