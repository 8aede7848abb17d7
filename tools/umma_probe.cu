// Probe: tcgen05.mma kind::tf32 with SW128 K-major operands written by threads,
// D[128 x N] = A[128 x 32] . B[N x 32]^T accumulated over four K=8 steps, read back
// with tcgen05.ld 32x32b. Checks the descriptor encodings of csrc/umma.cuh, the
// operand rounding (truncation vs nearest) and the 3xTF32 split accuracy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2110_11866_b200/csrc tools/umma_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "umma.cuh"

template <int N, bool SPLIT>
__global__ void probe(const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = sm;                 // 128 x 32 (hi)
  unsigned char* sAl = sm + 16384;        // 128 x 32 (lo)
  unsigned char* sB = sm + 32768;         // N x 32 (hi)
  unsigned char* sBl = sm + 32768 + 8192; // N x 32 (lo)
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * 32; e += 128) {
    const int r = e / 32, k = e % 32;
    float h, l;
    umma::split_tf32(A[e], h, l);
    *reinterpret_cast<float*>(sA + umma::sw128_off(r, k)) = SPLIT ? h : A[e];
    *reinterpret_cast<float*>(sAl + umma::sw128_off(r, k)) = l;
  }
  for (int e = tid; e < N * 32; e += 128) {
    const int r = e / 32, k = e % 32;
    float h, l;
    umma::split_tf32(B[e], h, l);
    *reinterpret_cast<float*>(sB + umma::sw128_off(r, k)) = SPLIT ? h : B[e];
    *reinterpret_cast<float*>(sBl + umma::sw128_off(r, k)) = l;
  }
  if (warp == 0) umma::tmem_alloc(&tbase, 64 < N ? 128 : 64);
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::mbar_fence_init();
  }
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    constexpr uint32_t id = umma::idesc_tf32(128, N);
    const uint32_t a0 = umma::smem_u32(sA), al0 = umma::smem_u32(sAl), b0 = umma::smem_u32(sB),
                   bl0 = umma::smem_u32(sBl);
    int n = 0;
    for (int k = 0; k < 4; ++k) {
      umma::mma_tf32(tmem, umma::desc_sw128(a0 + 32 * k), umma::desc_sw128(b0 + 32 * k), id, n++ > 0);
      if (SPLIT) {
        umma::mma_tf32(tmem, umma::desc_sw128(al0 + 32 * k), umma::desc_sw128(b0 + 32 * k), id, true);
        umma::mma_tf32(tmem, umma::desc_sw128(a0 + 32 * k), umma::desc_sw128(bl0 + 32 * k), id, true);
      }
    }
    umma::commit(&bar);
  }
  umma::mbar_wait(&bar, 0);
  umma::fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    umma::tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
    umma::tmem_wait_ld();
    for (int j = 0; j < 16; ++j) D[(warp * 32 + (tid & 31)) * N + c + j] = __uint_as_float(r[j]);
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free(tmem, 64 < N ? 128 : 64);
}

static float trunc_tf32(float x) {
  unsigned u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}
static float rn_tf32(float x) {
  unsigned u;
  memcpy(&u, &x, 4);
  const unsigned lsb = (u >> 13) & 1u;
  u = (u + 0xFFFu + lsb) & 0xFFFFE000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

template <int N, bool SPLIT>
static int run() {
  std::vector<float> A(128 * 32), B(N * 32), D(128 * N, -999.f);
  srand(7);
  for (auto& v : A) v = (rand() / float(RAND_MAX)) * 2.f - 1.f;
  for (auto& v : B) v = (rand() / float(RAND_MAX)) * 2.f - 1.f;
  A[0] = 1.0f + 3.0f * ldexpf(1.f, -13);  // trunc -> 1, nearest -> 1 + 2^-11
  for (int k = 1; k < 32; ++k) A[k] = 0.f;
  B[0] = 1.0f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 32768 + 16384 + 1024;
  cudaFuncSetAttribute(probe<N, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N, SPLIT><<<1, 128, smem>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("N=%d split=%d: CUDA error %s\n", N, SPLIT, cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double et = 0, er = 0, ex = 0, mx = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < N; ++j) {
      double st = 0, sr = 0, sx = 0;
      for (int k = 0; k < 32; ++k) {
        st += double(trunc_tf32(A[i * 32 + k])) * trunc_tf32(B[j * 32 + k]);
        sr += double(rn_tf32(A[i * 32 + k])) * rn_tf32(B[j * 32 + k]);
        sx += double(A[i * 32 + k]) * B[j * 32 + k];
      }
      const double d = D[i * N + j];
      et = fmax(et, fabs(d - st));
      er = fmax(er, fabs(d - sr));
      ex = fmax(ex, fabs(d - sx));
      mx = fmax(mx, fabs(sx));
    }
  printf("N=%d split=%d: D[0][0]=%.9g  max|D-trunc|=%.3e max|D-rn|=%.3e max|D-exact|=%.3e (max|D| %.3f)\n", N, SPLIT,
         D[0], et, er, ex, mx);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return 0;
}

int main() {
  int bad = 0;
  bad += run<16, false>();
  bad += run<64, false>();
  bad += run<32, false>();
  bad += run<64, true>();
  bad += run<16, true>();
  return bad;
}
