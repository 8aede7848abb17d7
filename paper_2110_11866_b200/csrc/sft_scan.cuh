// K1 — fused SFT/ASFT window scan + coefficient combine, single pass, sm_100a.
//
// Replaces, for every order at once, the reference's per-order component loops
// (proj/src/engine.cpp:53-219: recursive_components / kernel_integral_components /
// sliding_sum_components) followed by the separate combine passes of
// proj/src/transforms.cpp:279-428 (gauss_smooth / morlet_direct_transform /
// morlet_multiply_transform). One kernel reads the signal, writes only the final
// output, and never materialises the per-order component arrays.
//
// Math. Per order p with z = e^{-alpha - i omega}:
//   y[n]  = sum_{k=-K..K} x[n-k] z^k            (c = Re y, s = -Im y, engine.hpp:62-68)
//   V[n]  = sum_{j=n-K+1..n+K} x[j] z^{n+K-j}    (2K window, bounded state)
//   V[n]  = z V[n-1] + x[n+K] - z^{2K} x[n-K]   (first-order linear recurrence)
//   y[n]  = z^{-K} V[n] + z^{K} x[n-K]
// The combine sum_p wc_p c_p + ws_p s_p is folded into 4 real weights per order
// on (Re V, Im V) plus one complex weight D on x[n-K] shared by all orders.
// The recurrence is evaluated as a parallel scan: per-thread Horner over L
// positions, warp shuffle scan, inter-warp scan, and a decoupled look-back over
// tiles (aggregates/inclusive prefixes in fp64) for the carry between CTAs.
// The signal is consumed from a virtual zero state 2K positions before the first
// output ("warm tiles"), which makes the state at the first output exact.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace sftk {

constexpr int kMaxOrd = 12;
constexpr int kTabStride = 64;  // table entries per order (see TableLayout)
constexpr int kTileTab = 33;    // z^{T l}, l = 0..32

enum Mode { kModeReal = 0, kModeComplex = 1, kModeComps = 2 };

template <typename T>
struct Vec2;
template <>
struct Vec2<float> {
  using t = float2;
};
template <>
struct Vec2<double> {
  using t = double2;
};

// Hot per-order constants (kernel parameter space -> constant bank operands).
// Transform modes: k1..k4 map (Re V, Im V) to (Re out, Im out).
// Components mode: k1 = Re a, k2 = Im a, k3 = Re b, k4 = Im b with a = z^{-K}, b = z^{K}.
template <typename T>
struct OrdConst {
  T zr, zi;  // z
  T cr, ci;  // z^{2K} (trailing-sample injection)
  T k1, k2, k3, k4;
};

// Table layout per order (T2 entries, stride kTabStride):
//   [ 0, 32)  z^{L*lane}
//   [32, 37)  z^{L*2^k}      warp-scan multipliers
//   [40, 56)  z^{32L*w}      per-warp carry rotation, w < NW
//   [56, 60)  z^{32L*2^k}    inter-warp scan multipliers
template <typename T>
struct ScanParams {
  const T* x;
  long long n;     // samples per signal
  long long ld_x;  // elements between signals
  T* out;          // transform output, or c for components
  T* out_s;        // s for components
  long long ld_out;      // elements (complex: complex elements) between signals
  long long ord_stride;  // components: elements between orders
  long long lo;          // first output position
  long long count;       // outputs per signal
  int K;
  int boundary;  // 0 zero, 1 clamp
  int accumulate;
  int vec_ok;  // output base/stride allow vector stores
  long long tiles_per_signal;
  long long warm_tiles;
  long long total_tiles;
  // ctrl[0] tile ticket, ctrl[1] finished-CTA count, ctrl[2] launch epoch. The last
  // CTA of a launch resets the ticket/count and bumps the epoch, so launches need no
  // host-side state (graph-capturable) and stale look-back flags are ignored.
  unsigned int* ctrl;
  unsigned long long* flags;
  double2* agg;
  double2* incl;
  const typename Vec2<T>::t* tab;
  const double2* tab_tile;
  T Dr, Di;
  OrdConst<T> oc[kMaxOrd];
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T load_ext(const T* __restrict__ xs, long long n, int bnd, long long j) {
  if (j >= 0 && j < n) return __ldg(xs + j);
  if (bnd == 0) return T(0);
  return __ldg(xs + (j < 0 ? 0 : n - 1));
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

template <typename T2>
__device__ __forceinline__ T2 make2(decltype(T2::x) a, decltype(T2::x) b) {
  T2 r;
  r.x = a;
  r.y = b;
  return r;
}

__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, d);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, d);
  }
  return v;
}

// Decoupled look-back (one warp). Publishes this tile's aggregate s_agg, resolves
// the exclusive carry (state at the end of the previous tile) from predecessors'
// aggregates / inclusive prefixes into s_run, then publishes this tile's inclusive
// prefix. Flags: (epoch << 32) | status, status 1 = aggregate, 2 = inclusive.
// Per-order state lives in shared memory so the hot loops keep their registers.
template <typename T, int NORD>
__device__ __forceinline__ void lookback(const ScanParams<T>& P, long long gt, long long first,
                                         unsigned int epoch, const double2* s_agg, double2* s_run,
                                         double2* s_scl, int lane) {
  const unsigned long long ep = static_cast<unsigned long long>(epoch) << 32;
  if (gt == first) {
    if (lane < NORD) {
      P.incl[gt * NORD + lane] = s_agg[lane];
      s_run[lane] = make_double2(0.0, 0.0);
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      st_release_u64(P.flags + gt, ep | 2ull);
    }
    __syncwarp();
    return;
  }
  if (lane < NORD) {
    P.agg[gt * NORD + lane] = s_agg[lane];
    s_run[lane] = make_double2(0.0, 0.0);
    s_scl[lane] = make_double2(1.0, 0.0);
  }
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    st_release_u64(P.flags + gt, ep | 1ull);
  }
  long long base = gt - 1;
  while (true) {
    const long long t = base - lane;
    int st = 3;  // 3: before the signal's first tile = inclusive zero
    if (t >= first) {
      do {
        const unsigned long long f = ld_acquire_u64(P.flags + t);
        st = (static_cast<unsigned int>(f >> 32) == epoch) ? static_cast<int>(f & 3ull) : 0;
      } while (st == 0);
    }
    __syncwarp();
    const unsigned inc = __ballot_sync(0xffffffffu, st >= 2);
    const int m = inc ? __ffs(inc) - 1 : 31;
    const bool take = lane <= m && st != 3;
    const double2* src = (st == 2) ? P.incl : P.agg;
#pragma unroll 1
    for (int p = 0; p < NORD; ++p) {
      double2 v = make_double2(0.0, 0.0);
      if (take) v = __ldcg(src + t * NORD + p);
      if (m == 0) {
        v.x = __shfl_sync(0xffffffffu, v.x, 0);
        v.y = __shfl_sync(0xffffffffu, v.y, 0);
      } else {
        v = warp_sum2(cmul(P.tab_tile[p * kTileTab + lane], v));
      }
      if (lane == 0) {
        const double2 sc = s_scl[p];
        s_run[p] = cadd(s_run[p], cmul(sc, v));
        s_scl[p] = cmul(sc, P.tab_tile[p * kTileTab + 32]);
      }
    }
    __syncwarp();
    if (inc) break;
    base -= 32;
  }
  if (lane < NORD) P.incl[gt * NORD + lane] = cadd(cmul(P.tab_tile[lane * kTileTab + 1], s_run[lane]), s_agg[lane]);
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    st_release_u64(P.flags + gt, ep | 2ull);
  }
  __syncwarp();
}

template <typename T, int NORD, int MODE, int L, int NT>
__global__ void __launch_bounds__(NT) sft_scan_kernel(const __grid_constant__ ScanParams<T> P) {
  using T2 = typename Vec2<T>::t;
  constexpr int TT = NT * L;
  constexpr int NW = NT / 32;
  constexpr int LOGNW = NW >= 16 ? 4 : NW >= 8 ? 3 : NW >= 4 ? 2 : NW >= 2 ? 1 : 0;
  constexpr int PAD = TT + TT / 32;
  static_assert(NORD >= 1 && NORD <= kMaxOrd, "order count");
  static_assert(NW <= 16, "at most 16 warps");

  __shared__ T s_lead[PAD];
  __shared__ T s_trail[PAD];
  __shared__ T2 s_w[NW][NORD];
  __shared__ double2 s_lb[3][NORD];  // tile aggregate, carry, scale
  __shared__ long long s_tile;
  __shared__ unsigned int s_epoch;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;

  if (tid == 0) {
    s_tile = static_cast<long long>(atomicAdd(P.ctrl, 1u));
    s_epoch = *reinterpret_cast<volatile unsigned int*>(P.ctrl + 2);
  }
  __syncthreads();
  const long long gt = s_tile;
  const unsigned int epoch = s_epoch;
  const long long sig = gt / P.tiles_per_signal;
  const long long first = sig * P.tiles_per_signal;
  const long long o0 = (gt - first - P.warm_tiles) * TT;  // first output index of this tile
  const T* __restrict__ xs = P.x + sig * P.ld_x;

  // ---- stage the leading (x[n+K]) and trailing (x[n-K]) samples, coalesced
  {
    const long long lead_min = P.lo - P.K;  // virtual zero before the warm start
#pragma unroll
    for (int k = 0; k < L; ++k) {
      const int e = tid + k * NT;
      const long long o = o0 + e;
      const long long pos = P.lo + o;
      const long long jl = pos + P.K;
      const int se = e + (e >> 5);
      s_lead[se] = (jl >= lead_min) ? load_ext(xs, P.n, P.boundary, jl) : T(0);
      s_trail[se] = (o >= 0) ? load_ext(xs, P.n, P.boundary, pos - P.K) : T(0);
    }
  }
  __syncthreads();
  T xl[L], xt[L];
#pragma unroll
  for (int i = 0; i < L; ++i) {
    const int e = tid * L + i;
    xl[i] = s_lead[e + (e >> 5)];
    xt[i] = s_trail[e + (e >> 5)];
  }

  // ---- phase 1: per-thread aggregate (zero state in), all orders
  T2 st[NORD];
#pragma unroll
  for (int p = 0; p < NORD; ++p) {
    const OrdConst<T>& c = P.oc[p];
    T vr = fma(-c.cr, xt[0], xl[0]);
    T vi = -c.ci * xt[0];
#pragma unroll
    for (int i = 1; i < L; ++i) {
      const T gr = fma(-c.cr, xt[i], xl[i]);
      const T gi = -c.ci * xt[i];
      const T nr = fma(c.zr, vr, fma(-c.zi, vi, gr));
      const T ni = fma(c.zr, vi, fma(c.zi, vr, gi));
      vr = nr;
      vi = ni;
    }
    st[p] = make2<T2>(vr, vi);
  }

  // ---- warp inclusive scan of (z^{L*d}, state) pairs
#pragma unroll
  for (int p = 0; p < NORD; ++p) {
    T2 v = st[p];
    const T2* tb = P.tab + p * kTabStride;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int d = 1 << k;
      const T ur = __shfl_up_sync(0xffffffffu, v.x, d);
      const T ui = __shfl_up_sync(0xffffffffu, v.y, d);
      if (lane >= d) {
        const T2 w = tb[32 + k];
        v.x = fma(w.x, ur, fma(-w.y, ui, v.x));
        v.y = fma(w.x, ui, fma(w.y, ur, v.y));
      }
    }
    st[p] = v;
  }
  if (lane == 31) {
#pragma unroll
    for (int p = 0; p < NORD; ++p) s_w[warp][p] = st[p];
  }
#pragma unroll
  for (int p = 0; p < NORD; ++p) {  // inclusive -> exclusive within the warp
    const T ur = __shfl_up_sync(0xffffffffu, st[p].x, 1);
    const T ui = __shfl_up_sync(0xffffffffu, st[p].y, 1);
    st[p] = lane ? make2<T2>(ur, ui) : make2<T2>(T(0), T(0));
  }
  __syncthreads();

  // ---- warp 0: inter-warp scan, tile aggregate, look-back, per-warp carries
  if (warp == 0) {
#pragma unroll 1
    for (int p = 0; p < NORD; ++p) {
      const T2* tb = P.tab + p * kTabStride;
      T2 v = lane < NW ? s_w[lane][p] : make2<T2>(T(0), T(0));
#pragma unroll
      for (int k = 0; k < LOGNW; ++k) {
        const int d = 1 << k;
        const T ur = __shfl_up_sync(0xffffffffu, v.x, d);
        const T ui = __shfl_up_sync(0xffffffffu, v.y, d);
        if (lane >= d) {
          const T2 w = tb[56 + k];
          v.x = fma(w.x, ur, fma(-w.y, ui, v.x));
          v.y = fma(w.x, ui, fma(w.y, ur, v.y));
        }
      }
      const T ur = __shfl_up_sync(0xffffffffu, v.x, 1);
      const T ui = __shfl_up_sync(0xffffffffu, v.y, 1);
      if (lane < NW) s_w[lane][p] = lane ? make2<T2>(ur, ui) : make2<T2>(T(0), T(0));  // exclusive
      if (lane == NW - 1) s_lb[0][p] = make_double2(static_cast<double>(v.x), static_cast<double>(v.y));
    }
    __syncwarp();
    lookback<T, NORD>(P, gt, first, epoch, s_lb[0], s_lb[1], s_lb[2], lane);
    if (lane < NW) {
#pragma unroll 1
      for (int p = 0; p < NORD; ++p) {
        const T2 w = P.tab[p * kTabStride + 40 + lane];
        const T cr = static_cast<T>(s_lb[1][p].x), ci = static_cast<T>(s_lb[1][p].y);
        const T2 ex = s_w[lane][p];
        s_w[lane][p] = make2<T2>(fma(w.x, cr, fma(-w.y, ci, ex.x)), fma(w.x, ci, fma(w.y, cr, ex.y)));
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    // every CTA has its ticket and has finished its look-back: the last one re-arms
    __threadfence();
    if (atomicAdd(P.ctrl + 1, 1u) == static_cast<unsigned int>(P.total_tiles - 1)) {
      atomicExch(P.ctrl, 0u);
      atomicExch(P.ctrl + 1, 0u);
      atomicAdd(P.ctrl + 2, 1u);
      __threadfence();
    }
  }

  if (o0 + TT <= 0) return;  // warm tile: no outputs

  // state entering this thread's segment: z^{L*lane} * Cw + in-warp exclusive
#pragma unroll
  for (int p = 0; p < NORD; ++p) {
    const T2 cw = s_w[warp][p];
    const T2 w = P.tab[p * kTabStride + lane];
    st[p] = make2<T2>(fma(w.x, cw.x, fma(-w.y, cw.y, st[p].x)), fma(w.x, cw.y, fma(w.y, cw.x, st[p].y)));
  }

  const long long ob = o0 + static_cast<long long>(tid) * L;  // first output of this thread
  if (ob >= P.count) return;
  const bool full = ob >= 0 && ob + L <= P.count;

  if constexpr (MODE == kModeComps) {
#pragma unroll
    for (int p = 0; p < NORD; ++p) {
      const OrdConst<T>& c = P.oc[p];
      T vr = st[p].x, vi = st[p].y;
      T* cptr = P.out + p * P.ord_stride + sig * P.ld_out;
      T* sptr = P.out_s + p * P.ord_stride + sig * P.ld_out;
#pragma unroll
      for (int i = 0; i < L; ++i) {
        const T gr = fma(-c.cr, xt[i], xl[i]);
        const T gi = -c.ci * xt[i];
        const T nr = fma(c.zr, vr, fma(-c.zi, vi, gr));
        const T ni = fma(c.zr, vi, fma(c.zi, vr, gi));
        vr = nr;
        vi = ni;
        const long long o = ob + i;
        if (o >= 0 && o < P.count) {
          cptr[o] = fma(c.k1, vr, fma(-c.k2, vi, c.k3 * xt[i]));
          sptr[o] = -fma(c.k2, vr, fma(c.k1, vi, c.k4 * xt[i]));
        }
      }
    }
  } else {
    constexpr bool CPLX = MODE == kModeComplex;
    T ar[L], ai[L];
#pragma unroll
    for (int i = 0; i < L; ++i) {
      ar[i] = P.Dr * xt[i];
      ai[i] = CPLX ? P.Di * xt[i] : T(0);
    }
#pragma unroll
    for (int p = 0; p < NORD; ++p) {
      const OrdConst<T>& c = P.oc[p];
      T vr = st[p].x, vi = st[p].y;
#pragma unroll
      for (int i = 0; i < L; ++i) {
        const T gr = fma(-c.cr, xt[i], xl[i]);
        const T gi = -c.ci * xt[i];
        const T nr = fma(c.zr, vr, fma(-c.zi, vi, gr));
        const T ni = fma(c.zr, vi, fma(c.zi, vr, gi));
        vr = nr;
        vi = ni;
        ar[i] = fma(c.k1, vr, fma(c.k2, vi, ar[i]));
        if (CPLX) ai[i] = fma(c.k3, vr, fma(c.k4, vi, ai[i]));
      }
    }
    if (CPLX) {
      T* optr = P.out + 2 * (sig * P.ld_out);
      if (full && P.vec_ok && !P.accumulate) {
        T2* o2 = reinterpret_cast<T2*>(optr) + ob;
#pragma unroll
        for (int i = 0; i < L; ++i) o2[i] = make2<T2>(ar[i], ai[i]);
      } else {
#pragma unroll
        for (int i = 0; i < L; ++i) {
          const long long o = ob + i;
          if (o >= 0 && o < P.count) {
            if (P.accumulate) {
              optr[2 * o] += ar[i];
              optr[2 * o + 1] += ai[i];
            } else {
              optr[2 * o] = ar[i];
              optr[2 * o + 1] = ai[i];
            }
          }
        }
      }
    } else {
      T* optr = P.out + sig * P.ld_out;
#pragma unroll
      for (int i = 0; i < L; ++i) {
        const long long o = ob + i;
        if (o >= 0 && o < P.count) {
          if (P.accumulate)
            optr[o] += ar[i];
          else
            optr[o] = ar[i];
        }
      }
    }
  }
}

}  // namespace sftk
