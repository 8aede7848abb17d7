// K5 / K6 — the paper's data-parallel sliding sum h[n] = sum_{k<L} f[n+k] on the GPU
// (§IV, Algorithms 1-3). The reference only simulates these on CPU threads
// (proj/include/sft/sliding_sum.hpp:89-234); here they run as real kernels with the
// exact same addition trees, so results are bit-identical to the reference's for
// integers and doubles.
//   K5 flat doubling (Alg. 1): R = ceil(log2(L+1)) bulk rounds over double buffers,
//      g'[i] = g[i] + g[i+2^r], h'[i] = bit(L,r) ? g[i] + h[i+2^r] : h[i] (0 past the end).
//   K6 blocked8 (Alg. 2-3): (16,8) shared-memory tiles, three doubling rounds per base-8
//      digit of L, transposed write-back so stride-8 neighbours become adjacent, final
//      un-permute through the blocked layout.
#pragma once

#include <cuda_runtime.h>

namespace sftk {

template <typename T>
struct SsOps {
  static __device__ __forceinline__ T zero() { return T(0); }
  static __device__ __forceinline__ T add(T a, T b) { return a + b; }
};
template <>
struct SsOps<double2> {
  static __device__ __forceinline__ double2 zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
};

// One bulk round of Algorithm 1 (proj/include/sft/sliding_sum.hpp:99-119).
template <typename T>
__global__ void sliding_flat_round(const T* __restrict__ g, const T* __restrict__ h, T* __restrict__ g2,
                                   T* __restrict__ h2, long long n, long long shift, int fold) {
  using O = SsOps<T>;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const T gi = g[i];
    const T gs = i + shift < n ? g[i + shift] : O::zero();
    g2[i] = O::add(gi, gs);
    if (fold) {
      const T hs = i + shift < n ? h[i + shift] : O::zero();
      h2[i] = O::add(gi, hs);
    } else {
      h2[i] = h[i];
    }
  }
}

// One driver stage of Algorithms 2-3 (proj/include/sft/sliding_sum.hpp:160-210): block
// (16 x 8 threads) bx, col covers rows x_T + 8 y_T + 64 bx of column col.
template <typename T>
__global__ void __launch_bounds__(128) sliding_blocked8_stage(const T* __restrict__ g1, const T* __restrict__ h1,
                                                              T* __restrict__ g2, T* __restrict__ h2, long long rows,
                                                              long long cols, long long rest) {
  using O = SsOps<T>;
  __shared__ T S[16][8], Tt[16][8];
  const int xt = threadIdx.x & 15, yt = threadIdx.x >> 4;
  const long long id = blockIdx.x;
  const long long bx = id / cols, col = id - bx * cols;
  const long long row = xt + 8LL * yt + 64LL * bx;
  const bool in = row < rows;
  S[xt][yt] = in ? g1[row * cols + col] : O::zero();
  Tt[xt][yt] = in ? h1[row * cols + col] : O::zero();
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int fold = static_cast<int>((static_cast<unsigned long long>(rest) >> r) & 1ull);
    const int reach = 1 << r;
    T sn, tn;
    if (xt < 16 - reach) {
      tn = fold ? O::add(S[xt][yt], Tt[xt + reach][yt]) : Tt[xt][yt];
      sn = O::add(S[xt][yt], S[xt + reach][yt]);
    } else {
      tn = Tt[xt][yt];
      sn = S[xt][yt];
    }
    __syncthreads();
    S[xt][yt] = sn;
    Tt[xt][yt] = tn;
    __syncthreads();
  }
  // transposed write-back: g2[y_T + 8 x_B][x_T + 8 y_B] for the low half of the rows
  if (xt < 8) {
    const long long out_rows = rows / 8;
    const long long orow = yt + 8LL * bx;
    if (orow < out_rows) {
      const long long ocol = xt + 8LL * col;
      g2[orow * (cols * 8) + ocol] = S[xt][yt];
      h2[orow * (cols * 8) + ocol] = Tt[xt][yt];
    }
  }
}

// Final un-permute (proj/include/sft/sliding_sum.hpp:127-139, :226-233).
template <typename T>
__global__ void sliding_blocked8_gather(const T* __restrict__ h, T* __restrict__ out, long long count, int stages,
                                       long long cols) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long div = 1;
    for (int t = 0; t < stages; ++t) div *= 8;
    long long rem = i % div, c = 0;
    for (int t = 0; t < stages; ++t) {
      c = c * 8 + rem % 8;
      rem /= 8;
    }
    out[i] = h[(i / div) * cols + c];
  }
}

// Sliding-sum route of the components (proj/src/engine.cpp:183-219): the attenuated,
// phased sequence f[i] = x_ext[j] e^{alpha (j - center)} e^{i omega j}, j = lo - K + i,
// rebased at the window center so that e^{+-alpha ...} stays in range; then the window
// sums of K5; then each output is rescaled and its phase removed.
__device__ __forceinline__ double ext_sample(const double* x, long long n, int boundary, long long j) {
  if (j >= 0 && j < n) return x[j];
  if (boundary == 0) return 0.0;
  return j < 0 ? x[0] : x[n - 1];
}
__global__ void phased_sequence_kernel(const double* __restrict__ x, long long n, int boundary, long long lo,
                                       int K, double omega, double alpha, double center, long long len,
                                       double2* __restrict__ f) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long j = lo - K + i;
    const double w = alpha == 0.0 ? 1.0 : exp(alpha * (static_cast<double>(j) - center));
    const double xj = ext_sample(x, n, boundary, j) * w;
    double sn, cs;
    sincos(omega * static_cast<double>(j), &sn, &cs);
    f[i] = make_double2(xj * cs, xj * sn);
  }
}
__global__ void sliding_route_output_kernel(const double2* __restrict__ sums, long long lo, long long count,
                                            double omega, double alpha, double center, double* __restrict__ c,
                                            double* __restrict__ s) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < count;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long nn = lo + k;
    const double2 w = sums[k];
    const double scale = alpha == 0.0 ? 1.0 : exp(-alpha * (static_cast<double>(nn) - center));
    double sn, cs;
    sincos(omega * static_cast<double>(nn), &sn, &cs);
    // remove_phase (engine.cpp:129-134), stored as c = Re, s = -Im (ComponentSink)
    const double re = w.x * cs + w.y * sn, im = w.y * cs - w.x * sn;
    c[k] = scale * re;
    s[k] = -scale * im;
  }
}

}  // namespace sftk
