// C ABI for the GPU sliding sums (K5 flat, K6 blocked8) plus the reference's plan /
// cost-model arithmetic (proj/include/sft/sliding_sum.hpp:23-64, proj/src/sliding_sum.cpp:7-40).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "../../include/sftgpu.h"
#include "device_util.cuh"
#include "sliding_sum.cuh"

extern "C" const char* sftgpu_last_error(void);
void sftgpu_set_error(const std::string& m);  // sftgpu_api.cu

namespace {

struct SsPlan {
  long long n = 0, L = 0, padded = 0;
  int rounds = 0, stages = 0;
};

int stages_for(long long L) {
  int st = 0;
  for (long long rest = L; rest > 0; rest /= 8) ++st;
  return st;
}

bool make_plan(long long n, long long L, SsPlan* p) {
  if (n < 1) {
    sftgpu_set_error("SlidingSumPlan: N must be >= 1");
    return false;
  }
  if (L < 1 || L > n) {
    sftgpu_set_error("SlidingSumPlan: need 1 <= L <= N");
    return false;
  }
  p->n = n;
  p->L = L;
  p->rounds = 1;
  while ((1LL << p->rounds) <= L) ++p->rounds;
  p->stages = stages_for(L);
  long long floor8 = 1;
  for (int t = 0; t < p->stages; ++t) floor8 *= 8;
  p->padded = 1;
  while (p->padded < n || p->padded < floor8) p->padded *= 8;
  return true;
}

void cost(const SsPlan& p, int blocked, long long* steps, long long* adds) {
  long long a = 0;
  if (!blocked) {
    *steps = p.rounds;
    for (int r = 0; r < p.rounds; ++r) a += p.n * (1 + static_cast<int>((p.L >> r) & 1));
  } else {
    *steps = 3LL * p.stages;
    long long rows = p.padded, cols = 1, rest = p.L;
    while (rest > 0) {
      const long long blocks = ((rows + 63) / 64) * cols;
      for (int r = 0; r < 3; ++r) a += static_cast<long long>(16 - (1 << r)) * 8 * blocks * (1 + ((rest >> r) & 1));
      rows /= 8;
      cols *= 8;
      rest /= 8;
    }
  }
  *adds = a;
}

template <typename T>
int run(int blocked, const void* f, const SsPlan& p, void* out, cudaStream_t st) {
  const size_t cap = static_cast<size_t>(blocked ? p.padded : p.n);
  T *g1 = nullptr, *h1 = nullptr, *g2 = nullptr, *h2 = nullptr;
  auto fail = [&](cudaError_t e) {
    cudaFree(g1);
    cudaFree(h1);
    cudaFree(g2);
    cudaFree(h2);
    sftgpu_set_error(std::string("sliding sum: ") + cudaGetErrorString(e));
    return SFTGPU_ECUDA;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&g1, cap * sizeof(T))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&h1, cap * sizeof(T))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&g2, cap * sizeof(T))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&h2, cap * sizeof(T))) != cudaSuccess) return fail(e);
  cudaMemsetAsync(g1, 0, cap * sizeof(T), st);
  cudaMemsetAsync(h1, 0, cap * sizeof(T), st);
  cudaMemcpyAsync(g1, f, static_cast<size_t>(p.n) * sizeof(T), cudaMemcpyDeviceToDevice, st);
  const int threads = 256;
  const long long count = p.n - p.L + 1;
  if (!blocked) {
    const long long blocks = std::min<long long>((p.n + threads - 1) / threads, sftk::sm_count() * 32LL);
    for (int r = 0; r < p.rounds; ++r) {
      sftk::sliding_flat_round<T><<<blocks, threads, 0, st>>>(g1, h1, g2, h2, p.n, 1LL << r,
                                                              static_cast<int>((p.L >> r) & 1));
      std::swap(g1, g2);
      std::swap(h1, h2);
    }
    cudaMemcpyAsync(out, h1, static_cast<size_t>(count) * sizeof(T), cudaMemcpyDeviceToDevice, st);
  } else {
    long long rows = p.padded, cols = 1, rest = p.L;
    int stage = 0;
    while (rest > 0) {
      const long long nb = ((rows + 63) / 64) * cols;
      sftk::sliding_blocked8_stage<T><<<nb, 128, 0, st>>>(g1, h1, g2, h2, rows, cols, rest);
      std::swap(g1, g2);
      std::swap(h1, h2);
      rows /= 8;
      cols *= 8;
      rest /= 8;
      ++stage;
    }
    const long long blocks = std::min<long long>((count + threads - 1) / threads, sftk::sm_count() * 32LL);
    sftk::sliding_blocked8_gather<T><<<blocks, threads, 0, st>>>(h1, static_cast<T*>(out), count, stage, cols);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return fail(e);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail(e);
  cudaFree(g1);
  cudaFree(h1);
  cudaFree(g2);
  cudaFree(h2);
  return SFTGPU_OK;
}

}  // namespace

extern "C" int sftgpu_sliding_sum_plan(int64_t n, int64_t L, int blocked, int64_t* info) {
  SsPlan p;
  if (!make_plan(n, L, &p)) return SFTGPU_EINVAL;
  long long steps = 0, adds = 0;
  cost(p, blocked, &steps, &adds);
  if (info) {
    info[0] = p.rounds;
    info[1] = p.padded;
    info[2] = p.stages;
    info[3] = steps;
    info[4] = adds;
  }
  return SFTGPU_OK;
}

extern "C" int sftgpu_sliding_sum(int dtype, int blocked, const void* f, int64_t n, int64_t L, void* out,
                                  void* stream) {
  SsPlan p;
  if (!make_plan(n, L, &p)) return SFTGPU_EINVAL;
  if (!f || !out) {
    sftgpu_set_error("sliding sum: null buffer");
    return SFTGPU_EINVAL;
  }
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    sftgpu_set_error("no CUDA device available (libsftgpu has no CPU fallback)");
    return SFTGPU_ECUDA;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (dtype) {
    case SFTGPU_SS_I64: return run<long long>(blocked, f, p, out, st);
    case SFTGPU_SS_F64: return run<double>(blocked, f, p, out, st);
    case SFTGPU_SS_C128: return run<double2>(blocked, f, p, out, st);
    default: sftgpu_set_error("sliding sum: unknown dtype"); return SFTGPU_EINVAL;
  }
}
