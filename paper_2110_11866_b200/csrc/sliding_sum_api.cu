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

// sft_via_sliding_sum (proj/src/engine.cpp:183-219, 323-337): the reference's sliding-sum
// route for one SftConfig, on the GPU: phased sequence, K5 flat window sums (paper
// Algorithm 1, complex128), rescale and phase removal. Host fp64 in / out, synchronous.
// The GPU route accumulates in fp64 for both precisions (the reference sums complex<float>
// for Single; the parity bar is the fp64 result).
extern "C" int sftgpu_sft_via_sliding_sum(const sftgpu_config* cfg, const double* x_host, int64_t n, int boundary,
                                          double* c_host, double* s_host) {
  if (!cfg || !x_host || !c_host || !s_host) {
    sftgpu_set_error("sft_via_sliding_sum: null argument");
    return SFTGPU_EINVAL;
  }
  if (n < 1) {
    sftgpu_set_error("Signal: need at least one sample");
    return SFTGPU_EINVAL;
  }
  if (cfg->half_width < 1) {
    sftgpu_set_error("SftConfig: K must be >= 1");
    return SFTGPU_EINVAL;
  }
  if (cfg->integer_order && !(cfg->beta > 0.0)) {
    sftgpu_set_error("SftConfig: beta must be > 0");
    return SFTGPU_EINVAL;
  }
  if (cfg->alpha < 0.0) {
    sftgpu_set_error("SftConfig: alpha must be >= 0");
    return SFTGPU_EINVAL;
  }
  if (cfg->integer_order && cfg->p < 0) {
    sftgpu_set_error("OrderSpec: p must be >= 0");
    return SFTGPU_EINVAL;
  }
  if (boundary != SFTGPU_BOUNDARY_ZERO && boundary != SFTGPU_BOUNDARY_CLAMP) {
    sftgpu_set_error("unknown boundary policy");
    return SFTGPU_EINVAL;
  }
  const long long K = cfg->half_width, lo = 0, hi = n - 1, count = n, len = count + 2 * K;
  const double omega = cfg->integer_order ? cfg->beta * cfg->p : cfg->omega;
  const double center = 0.5 * static_cast<double>(lo + hi);
  if (cfg->alpha * (0.5 * static_cast<double>(count) + K) > 600.0) {
    sftgpu_set_error("sft_via_sliding_sum: alpha * N / 2 too large for the attenuated phased sequence");
    return SFTGPU_EINVAL;
  }
  int devs = 0;
  if (cudaGetDeviceCount(&devs) != cudaSuccess || devs == 0) {
    sftgpu_set_error("no CUDA device available (libsftgpu has no CPU fallback)");
    return SFTGPU_ECUDA;
  }
  SsPlan p;
  if (!make_plan(len, 2 * K + 1, &p)) return SFTGPU_EINVAL;
  double* dx = nullptr;
  double2 *f = nullptr, *sums = nullptr;
  double *dc = nullptr, *ds = nullptr;
  auto cleanup = [&]() {
    cudaFree(dx);
    cudaFree(f);
    cudaFree(sums);
    cudaFree(dc);
    cudaFree(ds);
  };
  auto cuda_fail = [&](cudaError_t e) {
    cleanup();
    sftgpu_set_error(std::string("sft_via_sliding_sum: ") + cudaGetErrorString(e));
    return SFTGPU_ECUDA;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&dx, n * sizeof(double))) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaMalloc(&f, len * sizeof(double2))) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaMalloc(&sums, count * sizeof(double2))) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaMalloc(&dc, count * sizeof(double))) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaMalloc(&ds, count * sizeof(double))) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaMemcpy(dx, x_host, n * sizeof(double), cudaMemcpyHostToDevice)) != cudaSuccess) return cuda_fail(e);
  const int sms = sftk::sm_count();
  sftk::phased_sequence_kernel<<<4 * sms, 256>>>(dx, n, boundary, lo, static_cast<int>(K), omega, cfg->alpha, center,
                                                 len, f);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e);
  const int rc = run<double2>(0, f, p, sums, nullptr);
  if (rc != SFTGPU_OK) {
    cleanup();
    return rc;
  }
  sftk::sliding_route_output_kernel<<<4 * sms, 256>>>(sums, lo, count, omega, cfg->alpha, center, dc, ds);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaMemcpy(c_host, dc, count * sizeof(double), cudaMemcpyDeviceToHost)) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaMemcpy(s_host, ds, count * sizeof(double), cudaMemcpyDeviceToHost)) != cudaSuccess) return cuda_fail(e);
  cleanup();
  return SFTGPU_OK;
}

// Host-memory variant of sftgpu_sliding_sum (device buffers managed here; synchronous).
extern "C" int sftgpu_sliding_sum_host(int dtype, int blocked, const void* f_host, int64_t n, int64_t L,
                                       void* out_host) {
  SsPlan p;
  if (!make_plan(n, L, &p)) return SFTGPU_EINVAL;
  if (!f_host || !out_host) {
    sftgpu_set_error("sliding sum: null buffer");
    return SFTGPU_EINVAL;
  }
  const size_t es = dtype == SFTGPU_SS_C128 ? 16 : 8;
  if (dtype != SFTGPU_SS_I64 && dtype != SFTGPU_SS_F64 && dtype != SFTGPU_SS_C128) {
    sftgpu_set_error("sliding sum: unknown dtype");
    return SFTGPU_EINVAL;
  }
  int devs = 0;
  if (cudaGetDeviceCount(&devs) != cudaSuccess || devs == 0) {
    sftgpu_set_error("no CUDA device available (libsftgpu has no CPU fallback)");
    return SFTGPU_ECUDA;
  }
  void *df = nullptr, *dout = nullptr;
  const size_t count = static_cast<size_t>(n - L + 1);
  cudaError_t e = cudaMalloc(&df, static_cast<size_t>(n) * es);
  if (e == cudaSuccess) e = cudaMalloc(&dout, count * es);
  if (e == cudaSuccess) e = cudaMemcpy(df, f_host, static_cast<size_t>(n) * es, cudaMemcpyHostToDevice);
  int rc = SFTGPU_OK;
  if (e == cudaSuccess) {
    rc = sftgpu_sliding_sum(dtype, blocked, df, n, L, dout, nullptr);
    if (rc == SFTGPU_OK) e = cudaMemcpy(out_host, dout, count * es, cudaMemcpyDeviceToHost);
  }
  cudaFree(df);
  cudaFree(dout);
  if (e != cudaSuccess) {
    sftgpu_set_error(std::string("sliding sum: ") + cudaGetErrorString(e));
    return SFTGPU_ECUDA;
  }
  return rc;
}
