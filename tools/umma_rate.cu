// Probe: tcgen05.mma kind::tf32 throughput on one SM, A from TMEM (ts) or shared memory
// (ss), B from shared memory, as in K4's chains: cycles per MMA for several N.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2110_11866_b200/csrc tools/umma_rate.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "umma.cuh"

template <int N, bool TS>
__global__ void rate(long long* out, int reps) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i & 255);
  if (warp == 0) umma::tmem_alloc(&tbase, 512);
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::mbar_fence_init();
  }
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    const uint64_t db = umma::desc_sw128(umma::smem_u32(sm));
    const uint32_t id = umma::idesc_tf32(128, N);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int k = 0; k < 24; ++k) {
        if (TS)
          umma::mma_tf32_ts<16384>(tmem + 256, tmem + 8 * (k & 15), db, id, k > 0);
        else
          umma::mma_tf32_off<0, 16384>(tmem + 256, db, id, k > 0);
      }
    }
    umma::commit_elect(&bar);
    umma::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (tid == 0) out[0] = t1 - t0;
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free(tmem, 512);
}

template <int N, bool TS>
void run() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int reps : {1, 64}) {
    rate<N, TS><<<1, 128, 70000>>>(d, reps);
    long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("N=%3d %s reps=%2d: %lld cycles, %.1f cycles/MMA (%s)\n", N, TS ? "A=TMEM" : "A=SMEM", reps, c,
           double(c) / (24.0 * reps), cudaGetErrorString(cudaGetLastError()));
  }
  cudaFree(d);
}

int main() {
  run<16, true>();
  run<64, true>();
  run<80, true>();
  run<128, true>();
  run<256, true>();
  run<64, false>();
  run<80, false>();
  return 0;
}
