// K2 — device test-signal generator (proj/src/signal.cpp:9-51).
// K3 — direct truncated convolution (proj/src/kernels.cpp:35-51), the reference's
//      "conventional" GCT3/MCT3 path and the exactness check at large sigma.
#pragma once

#include <cuda_runtime.h>

namespace sftk {

// splitmix64 stream: element i of a signal with seed s is draw i+1 of the stream,
// so every element is generated independently (bit-identical to the serial loop).
__device__ __forceinline__ double splitmix_uniform(unsigned long long seed, long long i) {
  unsigned long long z = seed + 0x9e3779b97f4a7c15ULL * static_cast<unsigned long long>(i + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  z ^= z >> 31;
  return 2.0 * (static_cast<double>(z >> 11) * 0x1.0p-53) - 1.0;
}

template <typename T>
__global__ void generate_signal_kernel(int kind, long long n, unsigned long long seed, long long batch,
                                       T* __restrict__ out) {
  const long long total = n * batch;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = idx / n, i = idx - b * n;
    double v;
    switch (kind) {
      case 0: v = (i == n / 2) ? 1.0 : 0.0; break;
      case 1: v = 1.0; break;
      case 2: {
        const double inv = 1.0 / (static_cast<double>(n) * static_cast<double>(n));
        v = sin(2.0 * 3.14159265358979323846 * 8.0 * static_cast<double>(i * i) * inv);
        break;
      }
      default: v = splitmix_uniform(seed + static_cast<unsigned long long>(b), i); break;
    }
    out[idx] = static_cast<T>(v);
  }
}

// out[n] = sum_j taps[j] * x[n - (tap_lo + j)], fp64 accumulate. One output per
// thread; taps and the matching signal window are staged through shared memory.
template <typename T, int BO, int BT>
__global__ void __launch_bounds__(BO) truncated_conv_kernel(const T* __restrict__ x, long long n, int bnd,
                                                            const double2* __restrict__ taps,
                                                            long long ntaps, long long tap_lo,
                                                            double2* __restrict__ out) {
  __shared__ double2 s_t[BT];
  __shared__ double s_x[BO + BT];
  const long long n0 = static_cast<long long>(blockIdx.x) * BO;
  const long long my = n0 + threadIdx.x;
  double ar = 0.0, ai = 0.0;
  for (long long j0 = 0; j0 < ntaps; j0 += BT) {
    // x index for (out m, tap j) = m - tap_lo - j; window over m in [n0, n0+BO), j in [j0, j0+BT)
    const long long xbase = n0 - tap_lo - (j0 + BT - 1);
    for (int k = threadIdx.x; k < BT; k += BO) s_t[k] = (j0 + k < ntaps) ? taps[j0 + k] : make_double2(0.0, 0.0);
    for (int k = threadIdx.x; k < BO + BT; k += BO) {
      const long long j = xbase + k;
      double v;
      if (j >= 0 && j < n)
        v = static_cast<double>(x[j]);
      else
        v = bnd == 0 ? 0.0 : static_cast<double>(x[j < 0 ? 0 : n - 1]);
      s_x[k] = v;
    }
    __syncthreads();
    // element for tap j0+k: x[my - tap_lo - j0 - k] = s_x[threadIdx.x + BT - 1 - k]
    const int lim = static_cast<int>(ntaps - j0 < BT ? ntaps - j0 : BT);
    for (int k = 0; k < lim; ++k) {
      const double xv = s_x[threadIdx.x + BT - 1 - k];
      ar = fma(s_t[k].x, xv, ar);
      ai = fma(s_t[k].y, xv, ai);
    }
    __syncthreads();
  }
  if (my < n) out[my] = make_double2(ar, ai);
}

}  // namespace sftk
