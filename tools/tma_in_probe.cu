// Probe: a tiled TMA tensor map over a signal viewed as OVERLAPPING rows (dim0 extent 68
// floats, dim1 stride 128 B) loading [32 rows][36 floats] boxes at unaligned element
// coordinates (c0 = 0..31), SWIZZLE_NONE: checks the driver accepts the overlapping view
// and that the box lands as padded 36-float rows with row r = x[32 (r0 + r) + c0 + k].
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2110_11866_b200/csrc tools/tma_in_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "umma.cuh"

__global__ void probe(const __grid_constant__ CUtensorMap map, const float* x, long long ld, int* bad, int nrows,
                      int cstep, int hint) {
  __shared__ __align__(128) float stg[32 * 36];
  __shared__ uint64_t bar;
  const int tid = threadIdx.x;
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::mbar_fence_init();
  }
  __syncthreads();
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  int phase = 0, nb = 0;
  for (int sig = 0; sig < 2; ++sig)
    for (int c0 = 0; c0 < 32; c0 += cstep)
      for (int r0 = 0; r0 + 32 <= nrows; r0 += 777) {
        if (tid == 0) {
          umma::mbar_arrive_tx(&bar, 32 * 36 * 4);
          if (hint)
            umma::tma_load_3d(umma::smem_u32(stg), &map, &bar, c0, r0, sig, pol);
          else
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(umma::smem_u32(stg)),
                "l"(reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(r0), "r"(sig), "r"(umma::smem_u32(&bar))
                : "memory");
        }
        umma::mbar_wait(&bar, phase);
        phase ^= 1;
        for (int e = tid; e < 32 * 36; e += blockDim.x) {
          const int r = e / 36, k = e % 36;
          const float want = x[sig * ld + 32LL * (r0 + r) + c0 + k];
          if (stg[e] != want) ++nb;
        }
        __syncthreads();
      }
  atomicAdd(bad, nb);
}

int main(int argc, char** argv) {
  const int cstep = argc > 1 ? atoi(argv[1]) : 1, hint = argc > 2 ? atoi(argv[2]) : 1, inner = argc > 3 ? atoi(argv[3]) : 36;
  const long long n = 102400, ld = 102400;
  std::vector<float> h(2 * ld);
  for (long long i = 0; i < 2 * ld; ++i) h[i] = static_cast<float>(i);
  float* x;
  int* bad;
  cudaMalloc(&x, h.size() * 4);
  cudaMalloc(&bad, 4);
  cudaMemset(bad, 0, 4);
  cudaMemcpy(x, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap map;
  const int nrows = static_cast<int>(n / 32) - 2;
  const cuuint64_t dims[3] = {68, static_cast<cuuint64_t>(nrows), 2};
  const cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(ld * 4)};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(inner), 32, 1}, es[3] = {1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode overlapping view: %d\n", static_cast<int>(r));
  if (r != CUDA_SUCCESS) return 1;
  probe<<<1, 128>>>(map, x, ld, bad, nrows, cstep, hint);
  cudaError_t e = cudaDeviceSynchronize();
  int hb = -1;
  cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  printf("kernel: %s, mismatches: %d\n", cudaGetErrorString(e), hb);
  return hb == 0 ? 0 : 2;
}
