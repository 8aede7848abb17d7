// K7: the reference's recursive strategies replayed on the GPU with its own rounding
// (proj/src/engine.cpp:53-120, recursive_components).
//
// Recursive1 (v = z v1 + x) and Recursive2 (the real second-order form) are sequential
// recurrences: a parallel scan computes the same values with different rounding (that is
// what K1 does for every strategy, and it is the more accurate of the two). A
// caller who needs the reference's numbers bit for bit gets them here:
//   pass 1 (one thread per order): the recurrence from zero state at warm = lo - 3K - 1 to
//     hi + K, every step in the reference's operation order with round-to-nearest
//     intrinsics (no FMA contraction; the reference is compiled for x86-64 without FMA), the
//     filter states v[m] stored to HBM;
//   pass 2 (one thread per output and order): the truncation window (2K or 2K+1 form), the
//     unwind factor z^{-K} and the sink (c = Re, s = -Im), also in the reference's order.
// The constants (z, 2 e^{-a} cos w, e^{-2a}, z^{2K}, z^{2K+1}, z^{-K}) are computed on the
// host with the same libm calls and casts as the reference. Scalar is float for Single and
// double for Double, as in the reference's dispatch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/sftgpu.h"

void sftgpu_set_error(const std::string& m);  // sftgpu_api.cu

namespace {

template <typename S>
struct RcParams {
  S zr, zi;          // z = e^{-alpha} (cos w, -sin w)
  S two_cos, dsq;    // 2 e^{-alpha} cos w, e^{-2 alpha}
  S zcr, zci;        // conj(z)
  S z2kr, z2ki;      // z^{2K}
  S z2k1r, z2k1i;    // z^{2K+1}
  S unr, uni;        // z^{-K}
  int strategy;      // SFTGPU_RECURSIVE1 / SFTGPU_RECURSIVE2
  int window_2k1;
  long long K, warm, len;  // chain positions warm .. warm + len - 1
  S* v;              // [len] complex states (interleaved)
  double* peak;      // max |v| over the chain (the reference's max_state, engine.cpp:101)
  double* c;         // [count]
  double* s;
};

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// extended_sample (proj/include/sft/signal.hpp:35-45)
__device__ __forceinline__ double ext(const double* x, long long n, int boundary, long long m) {
  if (m >= 0 && m < n) return x[m];
  if (boundary == SFTGPU_BOUNDARY_ZERO) return 0.0;
  return m < 0 ? x[0] : x[n - 1];
}

// pass 1: one thread per order (proj/src/engine.cpp:88-105); the strategy is a template
// parameter so the serial loop carries no branch
template <typename S, int ST>
__global__ void recursive_chain_kernel(const RcParams<S>* ps, int n_orders, const double* x, long long n,
                                       int boundary) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n_orders) return;
  const RcParams<S> P = ps[o];
  S v1r = 0, v1i = 0, v2r = 0, v2i = 0, px = 0;
  double pk = 0.0;
  auto step = [&](S xm, S& outr, S& outi, double& m2) {
    S vr, vi;
    if constexpr (ST == SFTGPU_RECURSIVE1) {
      // (zr v1r - zi v1i) + x,  zr v1i + zi v1r
      vr = add_rn(sub_rn(mul_rn(P.zr, v1r), mul_rn(P.zi, v1i)), xm);
      vi = add_rn(mul_rn(P.zr, v1i), mul_rn(P.zi, v1r));
    } else {
      // ((2c v1r - d v2r) + x) - zcr px,  (2c v1i - d v2i) - zci px
      vr = sub_rn(add_rn(sub_rn(mul_rn(P.two_cos, v1r), mul_rn(P.dsq, v2r)), xm), mul_rn(P.zcr, px));
      vi = sub_rn(sub_rn(mul_rn(P.two_cos, v1i), mul_rn(P.dsq, v2i)), mul_rn(P.zci, px));
    }
    v2r = v1r;
    v2i = v1i;
    v1r = vr;
    v1i = vi;
    px = xm;
    outr = vr;
    outi = vi;
    // |v|^2 in fp64, off the chain (reduced per batch; the root is taken once at the end)
    m2 = fma(static_cast<double>(vr), static_cast<double>(vr), static_cast<double>(vi) * vi);
  };
  // samples are loaded two batches ahead of the dependent chain (software pipeline), so
  // their latency hides behind 2 kU serial steps; full batches have no
  // bounds checks (the arrays stay in registers), the tail runs step by step
  constexpr int kU = 16;
  const long long full = P.len / kU * kU;
  S nx[kU], nx2[kU];  // batches b + 1 and b + 2 in flight
#pragma unroll
  for (int u = 0; u < kU; ++u) nx[u] = static_cast<S>(ext(x, n, boundary, P.warm + u));
#pragma unroll
  for (int u = 0; u < kU; ++u) nx2[u] = static_cast<S>(ext(x, n, boundary, P.warm + kU + u));
  long long b = 0;
  for (; b < full; b += kU) {
    S xs[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      xs[u] = nx[u];
      nx[u] = nx2[u];
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) nx2[u] = static_cast<S>(ext(x, n, boundary, P.warm + b + 2 * kU + u));
    S vs[2 * kU];
    double m2[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) step(xs[u], vs[2 * u], vs[2 * u + 1], m2[u]);
#pragma unroll
    for (int w = kU / 2; w >= 1; w >>= 1)
#pragma unroll
      for (int u = 0; u < w; ++u) m2[u] = fmax(m2[u], m2[u + w]);
    pk = fmax(pk, m2[0]);
    // the batch's states leave in 16-byte stores (the plan's state buffer is 256-B aligned
    // and kU * 2 * sizeof(S) is a multiple of 16)
    uint4* dst = reinterpret_cast<uint4*>(P.v + 2 * b);
#pragma unroll
    for (int i = 0; i < static_cast<int>(2 * kU * sizeof(S) / 16); ++i)
      dst[i] = *reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(vs) + 16 * i);
  }
  for (; b < P.len; ++b) {
    double m2;
    step(static_cast<S>(ext(x, n, boundary, P.warm + b)), P.v[2 * b], P.v[2 * b + 1], m2);
    pk = fmax(pk, m2);
  }
  *P.peak = sqrt(pk);
}

// pass 2: outputs n in [lo, hi] (proj/src/engine.cpp:107-117, sink :33-45)
template <typename S>
__global__ void recursive_window_kernel(const RcParams<S>* ps, int n_orders, const double* x, long long n,
                                        int boundary, long long lo, long long count) {
  const int o = blockIdx.y;
  if (o >= n_orders) return;
  const RcParams<S> P = ps[o];
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long nn = lo + i, m = nn + P.K, q = m - P.warm;
    const S vr = P.v[2 * q], vi = P.v[2 * q + 1];
    S wr, wi;
    if (P.window_2k1) {
      // v - z^{2K+1} v[m-2K-1]   (m - 2K - 1 >= warm always: the ring never reads zero)
      const long long r = q - 2 * P.K - 1;
      const S rr = P.v[2 * r], ri = P.v[2 * r + 1];
      const S tr = sub_rn(mul_rn(P.z2k1r, rr), mul_rn(P.z2k1i, ri));
      const S ti = add_rn(mul_rn(P.z2k1r, ri), mul_rn(P.z2k1i, rr));
      wr = sub_rn(vr, tr);
      wi = sub_rn(vi, ti);
    } else {
      // (v - z^{2K} v[m-2K]) + z^{2K} x[n-K]
      const long long r = q - 2 * P.K;
      const S rr = P.v[2 * r], ri = P.v[2 * r + 1];
      const S tr = sub_rn(mul_rn(P.z2kr, rr), mul_rn(P.z2ki, ri));
      const S ti = add_rn(mul_rn(P.z2kr, ri), mul_rn(P.z2ki, rr));
      const S xs = static_cast<S>(ext(x, n, boundary, nn - P.K));
      wr = add_rn(sub_rn(vr, tr), mul_rn(P.z2kr, xs));
      wi = add_rn(sub_rn(vi, ti), mul_rn(P.z2ki, xs));
    }
    // unwind * window
    const S outr = sub_rn(mul_rn(P.unr, wr), mul_rn(P.uni, wi));
    const S outi = add_rn(mul_rn(P.unr, wi), mul_rn(P.uni, wr));
    P.c[o * count + i] = static_cast<double>(outr);
    P.s[o * count + i] = -static_cast<double>(outi);
  }
}

// host constants exactly as recursive_components builds them (engine.cpp:58-79)
template <typename S>
RcParams<S> host_params(const sftgpu_config& c) {
  RcParams<S> P{};
  const int k = c.half_width;
  const double omega = c.integer_order ? c.beta * static_cast<double>(c.p) : c.omega;
  const double decay = std::exp(-c.alpha);
  P.zr = static_cast<S>(decay * std::cos(omega));
  P.zi = static_cast<S>(-decay * std::sin(omega));
  P.two_cos = static_cast<S>(2.0 * decay * std::cos(omega));
  P.dsq = static_cast<S>(decay * decay);
  P.zcr = P.zr;
  P.zci = -P.zi;
  auto zp = [&](double count, S* re, S* im) {
    const double mod = std::exp(-c.alpha * count);
    *re = static_cast<S>(mod * std::cos(omega * count));
    *im = static_cast<S>(-mod * std::sin(omega * count));
  };
  zp(2.0 * k, &P.z2kr, &P.z2ki);
  zp(2.0 * k + 1.0, &P.z2k1r, &P.z2k1i);
  const double mod = std::exp(c.alpha * k);
  P.unr = static_cast<S>(mod * std::cos(omega * k));
  P.uni = static_cast<S>(mod * std::sin(omega * k));
  P.strategy = c.strategy;
  P.window_2k1 = c.window_2k1 ? 1 : 0;
  P.K = k;
  return P;
}

struct DevBufs {
  std::vector<void*> ptrs;
  ~DevBufs() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <typename T>
  cudaError_t alloc(T** p, size_t bytes) {
    void* q = nullptr;
    const cudaError_t e = cudaMalloc(&q, bytes);
    if (e == cudaSuccess) ptrs.push_back(q);
    *p = static_cast<T*>(q);
    return e;
  }
};

template <typename S>
cudaError_t run(const sftgpu_config* cfgs, const std::vector<int>& idx, const double* dx, long long n, int boundary,
                long long lo, long long hi, double* dc, double* ds, double* dpeak, DevBufs& bufs) {
  if (idx.empty()) return cudaSuccess;
  const long long count = hi - lo + 1;
  std::vector<RcParams<S>> ps;
  std::vector<int> order(idx);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return cfgs[a].strategy == SFTGPU_RECURSIVE1 && cfgs[b].strategy != SFTGPU_RECURSIVE1; });
  for (int i : order) {
    RcParams<S> P = host_params<S>(cfgs[i]);
    P.warm = lo - P.K - (2 * P.K + 1);
    P.len = hi + P.K - P.warm + 1;
    cudaError_t e = bufs.alloc(&P.v, static_cast<size_t>(P.len) * 2 * sizeof(S));
    if (e != cudaSuccess) return e;
    P.c = dc + static_cast<long long>(i) * count;
    P.s = ds + static_cast<long long>(i) * count;
    P.peak = dpeak + i;
    ps.push_back(P);
  }
  // pass 2 writes c/s of order o at o * count: give each its own base (o = 0 per entry)
  RcParams<S>* dps = nullptr;
  cudaError_t e = bufs.alloc(&dps, ps.size() * sizeof(RcParams<S>));
  if (e != cudaSuccess) return e;
  if ((e = cudaMemcpy(dps, ps.data(), ps.size() * sizeof(RcParams<S>), cudaMemcpyHostToDevice)) != cudaSuccess)
    return e;
  const int no = static_cast<int>(ps.size());
  // one thread per order (ps is sorted by strategy): one launch per strategy
  const int n1 = static_cast<int>(std::count_if(ps.begin(), ps.end(),
                                                [](const RcParams<S>& q) { return q.strategy == SFTGPU_RECURSIVE1; }));
  if (n1 > 0) recursive_chain_kernel<S, SFTGPU_RECURSIVE1><<<(n1 + 31) / 32, 32>>>(dps, n1, dx, n, boundary);
  if (no > n1)
    recursive_chain_kernel<S, SFTGPU_RECURSIVE2><<<(no - n1 + 31) / 32, 32>>>(dps + n1, no - n1, dx, n, boundary);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  for (int j = 0; j < no; ++j) {
    const long long blocks = std::min<long long>((count + 255) / 256, 4096);
    recursive_window_kernel<S><<<dim3(static_cast<unsigned>(blocks), 1), 256>>>(dps + j, 1, dx, n, boundary, lo, count);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

extern "C" int sftgpu_components_replay(const sftgpu_config* cfgs, int n_orders, const double* x_host, int64_t n,
                                        int boundary, int64_t lo, int64_t hi, double* c_host, double* s_host,
                                        double* max_state) {
  auto bad = [](const char* m) {
    sftgpu_set_error(m);
    return SFTGPU_EINVAL;
  };
  if (!cfgs || n_orders < 1 || !x_host || !c_host || !s_host) return bad("components_replay: null argument");
  if (n < 1) return bad("Signal: need at least one sample");
  if (boundary != SFTGPU_BOUNDARY_ZERO && boundary != SFTGPU_BOUNDARY_CLAMP) return bad("unknown boundary policy");
  for (int i = 0; i < n_orders; ++i) {
    const sftgpu_config& c = cfgs[i];
    // SftConfig::validate (proj/include/sft/engine.hpp:51-59)
    if (c.half_width < 1) return bad("SftConfig: K must be >= 1");
    if (c.integer_order && !(c.beta > 0.0)) return bad("SftConfig: beta must be > 0");
    if (c.alpha < 0.0) return bad("SftConfig: alpha must be >= 0");
    if (c.integer_order && c.p < 0) return bad("OrderSpec: p must be >= 0");
    if (!c.integer_order && c.strategy != SFTGPU_KERNEL_INTEGRAL)
      return bad("SftConfig: real-frequency components require the kernel-integral strategy");
    if (c.strategy != SFTGPU_RECURSIVE1 && c.strategy != SFTGPU_RECURSIVE2)
      return bad("components_replay: replays the recursive strategies (the kernel-integral strategy runs on K1)");
  }
  if (lo > hi) return bad("components_over: empty range");
  int devs = 0;
  if (cudaGetDeviceCount(&devs) != cudaSuccess || devs == 0) {
    sftgpu_set_error("no CUDA device available (libsftgpu has no CPU fallback)");
    return SFTGPU_ECUDA;
  }
  const long long count = hi - lo + 1;
  std::vector<int> f32, f64;
  for (int i = 0; i < n_orders; ++i) (cfgs[i].precision == SFTGPU_SINGLE ? f32 : f64).push_back(i);
  DevBufs bufs;
  double *dx = nullptr, *dc = nullptr, *ds = nullptr, *dpeak = nullptr;
  const size_t out_bytes = static_cast<size_t>(n_orders) * count * sizeof(double);
  cudaError_t e = bufs.alloc(&dx, n * sizeof(double));
  if (e == cudaSuccess) e = bufs.alloc(&dc, out_bytes);
  if (e == cudaSuccess) e = bufs.alloc(&ds, out_bytes);
  if (e == cudaSuccess) e = bufs.alloc(&dpeak, static_cast<size_t>(n_orders) * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(dx, x_host, n * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = run<float>(cfgs, f32, dx, n, boundary, lo, hi, dc, ds, dpeak, bufs);
  if (e == cudaSuccess) e = run<double>(cfgs, f64, dx, n, boundary, lo, hi, dc, ds, dpeak, bufs);
  if (e == cudaSuccess) e = cudaMemcpy(c_host, dc, out_bytes, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(s_host, ds, out_bytes, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && max_state)
    e = cudaMemcpy(max_state, dpeak, static_cast<size_t>(n_orders) * sizeof(double), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    sftgpu_set_error(std::string("components_replay: ") + cudaGetErrorString(e));
    return SFTGPU_ECUDA;
  }
  return SFTGPU_OK;
}
