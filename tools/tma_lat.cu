// Probe: K4's memory pattern without its compute. 148 persistent CTAs walk (signal, tile)
// items like sft_tc_kernel (31 tiles per signal of 102400 samples): per tile one thread
// TMA-loads the lead and trail boxes (129 x 32 fp32, SW128, overlapping-row view) into a
// ring of S slots and a second thread TMA-stores 32 KB of output (two 128 x 32 boxes).
// A spin of D cycles per tile stands in for the compute. Reports the kernel time, the
// HBM rate and the mean / max issue-to-landed latency of the loads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2110_11866_b200/csrc tools/tma_lat.cu -lcuda -o tools/tma_lat
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "umma.cuh"

constexpr int kSlotBytes = 2 * 17408;

__global__ void __launch_bounds__(576, 1)
    walk(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map, int nsig, int S,
         int D, int stores, int trail, int PF, const float* x, const CUtensorMap* gmaps, int M, unsigned long long* lat) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = raw + ((1024u - (umma::smem_u32(raw) & 1023u)) & 1023u);
  unsigned char* ring = sm;
  unsigned char* ostg = sm + S * kSlotBytes;
  __shared__ uint64_t full[8];
  __shared__ unsigned long long t_iss[8];
  const int tid = threadIdx.x;
  const CUtensorMap* imap = &in_map;
  const CUtensorMap* omap = &out_map;
  if (M == 1 && (tid == 0 || tid == 32)) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(imap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(omap)) : "memory");
  }
  if (tid == 0) {
    for (int k = 0; k < 8; ++k) umma::mbar_init(&full[k], 1);
    umma::mbar_fence_init();
  }
  __syncthreads();
  unsigned long long keep, first;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(first));
  const int tiles = 31, warm = 6;
  unsigned long long sum = 0, mx = 0, cnt = 0;
  if (tid == 0) {
    // loader: tile g of the CTA's walk = (signal blockIdx.x + 148 (g / tiles), tile g % tiles)
    const long long total = static_cast<long long>((nsig - blockIdx.x + gridDim.x - 1) / gridDim.x) * tiles;
    unsigned long long cb = 0;
    auto issue = [&](long long g) {
      if (g >= total) return;
      const int gi = static_cast<int>(g), sig = blockIdx.x + gridDim.x * (gi / tiles), t = gi % tiles;
      const int slot = static_cast<int>(static_cast<unsigned>(g) % static_cast<unsigned>(S));
      const long long al = 24576 - 8 + static_cast<long long>(t - warm) * 4096;  // lead start (aligned)
      const long long at = al - 49152;
      const bool tl = al >= 0 && (al >> 5) + 129 <= 3199, tt = trail && t >= warm && at >= 0;
      t_iss[slot] = clock64();
      const unsigned long long b0 = clock64();
      umma::mbar_arrive_tx(&full[slot], (tl ? 16512u : 0u) + (tt ? 16512u : 0u));
      const unsigned long long b1 = clock64();
      cb += b1 - b0;
      unsigned char* sl = ring + slot * kSlotBytes;
      if (tl) umma::tma_load_3d(umma::smem_u32(sl), imap, &full[slot], static_cast<int>(al & 31), static_cast<int>(al >> 5), sig, keep);
      if (tt) umma::tma_load_3d(umma::smem_u32(sl + 17408), imap, &full[slot], static_cast<int>(at & 31), static_cast<int>(at >> 5), sig, first);
    };
    auto prefetch = [&](long long g) {
      if (PF == 0 || g >= total) return;
      const int gi = static_cast<int>(g), sig = blockIdx.x + gridDim.x * (gi / tiles), t = gi % tiles;
      const long long al = 24576 - 8 + static_cast<long long>(t - warm) * 4096;
      if (al < 0 || al + 4096 > 102400) return;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x + sig * 102400LL + al), "r"(16384u) : "memory");
    };
    for (int k = 0; k < S - 1; ++k) issue(k);
    for (int k = S - 1; k < S - 1 + PF; ++k) prefetch(k);
    uint32_t ph = 0;
    unsigned long long ci = 0, cw = 0;
    for (long long g = 0; g < total; ++g) {
      const unsigned long long a0 = clock64();
      issue(g + S - 1);
      prefetch(g + S - 1 + PF);
      const int slot = static_cast<int>(static_cast<unsigned>(g) % static_cast<unsigned>(S));
      const unsigned long long a1 = clock64();
      umma::mbar_wait(&full[slot], (ph >> slot) & 1u);
      const unsigned long long a2 = clock64();
      ci += a1 - a0;
      cw += a2 - a1;
      ph ^= 1u << slot;
      const unsigned long long l = clock64() - t_iss[slot];
      sum += l;
      mx = l > mx ? l : mx;
      ++cnt;
      const unsigned long long t0 = clock64();
      while (clock64() - t0 < static_cast<unsigned long long>(D)) {
      }
    }
    t_iss[7] = 1;
    atomicAdd(&lat[3], ci);
    atomicAdd(&lat[5], cb);
    atomicAdd(&lat[4], cw);
    atomicAdd(&lat[0], sum);
    atomicAdd(&lat[1], cnt);
    atomicMax(&lat[2], mx);
  } else if (tid >= 64 && M >= 10) {
    // shared-memory load pressure (M - 10 warps' worth of LDS.128 streaming), no stores
    if ((tid >> 5) - 2 < M - 10) {
      const float4* src = reinterpret_cast<const float4*>(ring);
      float4 acc = make_float4(0, 0, 0, 0);
      volatile int* stop = reinterpret_cast<volatile int*>(&t_iss[7]);
      for (int it = 0; it < 2000000 && *stop == 0; ++it) {
        const float4 v = src[(tid * 8 + it * 32) & 2047];
        acc.x += v.x;
        acc.y += v.y;
      }
      if (acc.x == 1.2345f) lat[6] = 1;
    }
  } else if (tid == 32 && stores) {
    // storer: output tiles of the same walk, 2 x (128 rows x 128 B) per tile
    const long long total = static_cast<long long>((nsig - blockIdx.x + gridDim.x - 1) / gridDim.x) * tiles;
    for (long long g = 0; g < total; ++g) {
      const int gi = static_cast<int>(g), sig = blockIdx.x + gridDim.x * (gi / tiles), t = gi % tiles;
      if (t < warm) continue;
      const unsigned long long s0 = clock64();
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      const int row0 = (t - warm) * 128;
      for (int h = 0; h < 2; ++h)
        asm volatile(
            "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                reinterpret_cast<uint64_t>(omap)),
            "r"(0), "r"(h), "r"(row0), "r"(sig), "r"(umma::smem_u32(ostg + h * 16384))
            : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      atomicAdd(&lat[5], clock64() - s0);
      const unsigned long long t0 = clock64();
      while (clock64() - t0 < static_cast<unsigned long long>(D)) {
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main(int argc, char** argv) {
  const int S = argc > 1 ? atoi(argv[1]) : 3, D = argc > 2 ? atoi(argv[2]) : 0, stores = argc > 3 ? atoi(argv[3]) : 1,
            trail = argc > 4 ? atoi(argv[4]) : 1, PF = argc > 5 ? atoi(argv[5]) : 0, M = argc > 6 ? atoi(argv[6]) : 0;
  const int nsig = 4096;
  const long long n = 102400;
  float *x, *out;
  cudaMalloc(&x, nsig * n * 4);
  cudaMalloc(&out, nsig * n * 8);
  cudaMemset(x, 0, nsig * n * 4);
  unsigned long long* lat;
  cudaMalloc(&lat, 64);
  CUtensorMap in_map, out_map;
  {
    const cuuint64_t dims[3] = {64, 3199, static_cast<cuuint64_t>(nsig)};
    const cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(n * 4)};
    const cuuint32_t box[3] = {32, 129, 1}, es[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&in_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) return printf("in map %d\n", r), 1;
  }
  {
    const cuuint64_t dims[4] = {32, 2, static_cast<cuuint64_t>(n / 32), static_cast<cuuint64_t>(nsig)};
    const cuuint64_t strides[3] = {128, 256, static_cast<cuuint64_t>(n * 8)};
    const cuuint32_t box[4] = {32, 1, 128, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&out_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, out, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) return printf("out map %d\n", r), 1;
  }
  CUtensorMap* gmaps;
  cudaMalloc(&gmaps, 2 * sizeof(CUtensorMap));
  cudaMemcpy(gmaps, &in_map, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  cudaMemcpy(gmaps + 1, &out_map, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  const int smem = S * kSlotBytes + 32768 + 1024;
  cudaFuncSetAttribute(walk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) {
    cudaMemset(lat, 0, 64);
    cudaEventRecord(e0);
    walk<<<148, M >= 10 ? 576 : 64, smem>>>(in_map, out_map, nsig, S, D, stores, trail, PF, x, gmaps, M, lat);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    if (e) return printf("err %s\n", cudaGetErrorString(e)), 1;
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[6];
    cudaMemcpy(h, lat, 48, cudaMemcpyDeviceToHost);
    const double bytes = nsig * n * 4.0 * (stores ? 3.0 : 1.0);
    if (it == 2)
      printf("M=%d S=%d D=%d stores=%d trail=%d PF=%d: %.3f ms, %.0f GB/s (algorithmic), load latency mean %.0f max %llu cycles; per tile: issue %.0f wait %.0f arrive %.0f\n", M, S,
             D, stores, trail, PF, ms, bytes / ms / 1e6, static_cast<double>(h[0]) / h[1], h[2],
             static_cast<double>(h[3]) / h[1], static_cast<double>(h[4]) / h[1], static_cast<double>(h[5]) / h[1]);
  }
  return 0;
}
