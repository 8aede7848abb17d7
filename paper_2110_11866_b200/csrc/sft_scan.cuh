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
//   V[n]  = sum_{j=n-K+1..n+K} x[j] z^{n+K-j}    (2K window: state bounded by the window)
//   V[n]  = z V[n-1] + g[n],  g[n] = x[n+K] - z^{2K} x[n-K]
//   y[n]  = z^{-K} V[n] + z^{K} x[n-K]
// For integer orders with beta = pi/K every order shares the real injection constant
// z^{2K} = e^{-2 alpha K}, so g is computed once per position for all orders (group
// mode 0); the multiplication method's real-frequency orders share one complex
// constant (group mode 1); anything else uses per-order injection (group mode 2).
// The combine sum_p wc_p c_p + ws_p s_p is folded into 4 real weights per order on
// (Re V, Im V) plus one complex weight D on x[n-K] shared by all orders.
//
// Parallel structure: a tile of TT = NT*L positions per CTA step; per thread the
// aggregate of its L positions is a dot product with precomputed z^{L-1-i} weights,
// then a warp shuffle scan, an inter-warp scan, and the tile carry. Two modes:
//   SEQ  one CTA owns a whole signal and walks its tiles with the carry in shared
//        memory (fp64) and the next tile's samples prefetched in registers — batched
//        workloads, no inter-CTA communication at all;
//   LB   one tile per CTA and a decoupled look-back over tiles (fp64 aggregates /
//        inclusive prefixes) — single long signals and small batches.
// The signal is consumed from a virtual zero state 2K positions before the first
// output ("warm tiles", phase 1 only), which makes the state at the first output exact.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace sftk {

#ifndef SFTK_SEQ_MINB
#define SFTK_SEQ_MINB 8
#endif
constexpr int kMaxOrd = 12;
constexpr int kMaxL = 16;
constexpr int kTabStride = 64;  // table entries per order (see layout below)
constexpr int kTabTileStride = 6;  // tile-table entries per order

enum Mode { kModeReal = 0, kModeComplex = 1, kModeComps = 2 };
// Injection group modes: 0 one real constant for all orders, 1 split (first NA orders
// real constant, the rest one complex constant), 2 per order, 3 one complex constant
// for all orders (host-side name; the kernel runs it as split with NA = 0).
enum GroupMode { kGroupShared = 0, kGroupSplit = 1, kGroupPerOrder = 2, kGroupSharedC = 3 };

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

// Hot per-order constants (kernel parameter space -> constant-bank operands).
// Transform modes: k1..k4 map (Re V, Im V) to (Re out, Im out).
// Components mode: k1 = Re a, k2 = Im a, k3 = Re b, k4 = Im b with a = z^{-K}, b = z^{K}.
// Stored as the packed pairs the fp32 path feeds to FFMA2 (fma.rn.f32x2):
//   zz = {zr, zr}, zx = {-zi, zi}, ka = {k1, k3}, kb = {k2, k4}, cc = {cr, ci},
//   w[i] = {Re, Im, -Im, Re} of z^{L-1-i}.
template <typename T>
struct OrdConst {
  T zz[2];
  T zx[2];
  T ka[2];
  T kb[2];
  T cc[2];  // z^{2K} (per-order injection, group mode 2)
  T w[kMaxL][4];
  T scan[5][4];   // z^{L 2^k}, warp-scan multipliers, as {re, re, -im, im}
  T wrot[4][4];   // z^{32 L w}, per-warp carry rotation (NW <= 4)
  T m32[4];       // z^{32 L}, inter-warp step
};

// Table layout per order (entries {re, re, -im, im}, stride kTabStride):
//   [ 0, 32)  z^{L*lane}
//   [32, 37)  z^{L*2^k}      warp-scan multipliers
//   [40, 56)  z^{32L*w}      per-warp carry rotation, w < NW
//   [56, 60)  z^{32L*2^k}    inter-warp scan multipliers
// Tile table (double2, per order, stride kTabTileStride): [0] z^{TT}, [1] z^{32 TT},
// [2 + g] z^{TT (cnt - min(cnt, (g + 1) ceil(cnt / G)))}: the LB window-carry segment
// scales (cnt = D + 1 predecessors, G = 4 lane groups for <= 8 orders, else 2).
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
  int vec_ok;  // output base and row stride allow 16-byte vector stores
  int na;  // group mode 1: orders [0, na) use injection A, [na, NORD) injection B
  long long tiles_per_signal;  // LB: per signal; SEQ: per chunk (warm tiles included)
  long long warm_tiles;
  long long total_tiles;  // LB: tiles in the grid
  long long chunk_len;    // SEQ: outputs per chunk (multiple of the tile), one CTA per chunk
  long long n_chunks;     // SEQ: chunks per signal
  int lb_D;               // LB: full tiles in the 2K window (2K = lb_D*TT + r)
  int lb_sfx;             // LB: first position of a tile's r-position suffix (TT if r == 0)
  // ctrl[0..1]: 64-bit count of LB CTAs ever started on this plan. Every launch adds
  // exactly total_tiles, so count / total_tiles numbers the launch (its epoch) without
  // host state (graph-capturable) or a re-arming CTA; stale look-back payloads carry an
  // older epoch.
  unsigned int* ctrl;
  unsigned long long* flags;
  double2* agg;
  double2* incl;
  const T* tab;  // [NORD][kTabStride][4] entries {re, re, -im, im}
  const double2* tab_tile;
  long long* trace;  // optional LB phase timestamps ([tile][8] globaltimer ns), tools/scan_trace.py
  T cAr, cAi, cBr, cBi;  // shared injection constants (group modes 0/1)
  T Dr, Di;
  OrdConst<T> oc[kMaxOrd];
};

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// fp32 plans publish look-back payloads without flags: every 8-byte word carries a launch
// tag in its low 4 bits. The payload doubles are converted from fp32, so those bits are
// zero and stripping the tag restores them exactly; each aligned 8-byte word is
// single-copy atomic, so a reader that sees the current tag sees that word's value
// (no release fence on the producer, no flag round trip on the consumer).
__device__ __forceinline__ unsigned long long pay_tag(unsigned int epoch) { return (epoch % 15u) + 1u; }
__device__ __forceinline__ unsigned long long tag_word(double v, unsigned long long tg) {
  return (static_cast<unsigned long long>(__double_as_longlong(v)) & ~15ull) | tg;
}
__device__ __forceinline__ double untag_word(unsigned long long w) {
  return __longlong_as_double(static_cast<long long>(w & ~15ull));
}
__device__ __forceinline__ void st_relaxed_v2(double2* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_relaxed_v2(const double2* p, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Leading samples are re-read 2K positions later as trailing samples: keep them in L2
// (evict_last policy); trailing reads are their last use and outputs are written once
// (streaming), so neither displaces the signal window still needed.
__device__ __forceinline__ unsigned long long l2_keep_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ float ld_keep(const float* p, unsigned long long pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_keep(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

template <typename T>
__device__ __forceinline__ T load_ext(const T* __restrict__ xs, long long n, int bnd, long long j) {
  if (j >= 0 && j < n) return __ldcs(xs + j);
  if (bnd == 0) return T(0);
  return __ldg(xs + (j < 0 ? 0 : n - 1));
}


__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, d);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, d);
  }
  return v;
}

template <typename T2>
__device__ __forceinline__ T2 make2(decltype(T2::x) a, decltype(T2::x) b) {
  T2 r;
  r.x = a;
  r.y = b;
  return r;
}

// ---- packed fp32 pairs (FFMA2). ptxas folds the half swaps / broadcasts into operand
// modifiers (.F32x2.LO_HI, .F32), so a complex multiply-add is two FFMA2.
using u64 = unsigned long long;
__device__ __forceinline__ u64 pk(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float plo(u64 v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return lo;
}
__device__ __forceinline__ float phi(u64 v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return hi;
}
__device__ __forceinline__ u64 pswap(u64 v) { return pk(phi(v), plo(v)); }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 ldp(const float* p) { return *reinterpret_cast<const u64*>(p); }
// v + w * u for complex w = (wr, wi) given as packed {wr, wi}
__device__ __forceinline__ u64 cmadd2(float wr, float wi, u64 u, u64 v) {
  return fma2(pk(-wi, wi), pswap(u), fma2(pk(wr, wr), u, v));
}

template <typename T, int NORD, int L, int NT, bool SEQ>
struct Smem {
  using T2 = typename Vec2<T>::t;
  static constexpr int TT = NT * L;
  static constexpr int PAD = TT + TT / 32;
  static constexpr int NW = NT / 32;
  static constexpr int NB = SEQ ? 2 : 1;  // SEQ double-buffers by tile parity
  T lead[NB][PAD];
  T trail[NB][PAD];
  T2 w[NW][NORD];         // warp totals, then per-warp carries
  double2 carry[NORD];    // state at the end of the previous tile (fp64)
  double2 tagg[NORD];     // this tile's aggregate (SEQ) / lead-only aggregate (LB)
  double2 tsfx[NORD];     // LB: lead-only aggregate of the tile's last r positions
  T2 wla[NW][NORD];       // LB: per-warp lead-only totals
  T2 wsa[NW][NORD];       // LB: per-warp lead-only suffix totals
  // The transposed-scan staging is dead once the scan's barrier has passed; the LB
  // window carry (warp 0, after that barrier) reuses it.
  union {
    T2 wscan[NW][NORD * 33];          // per-warp transposed scan staging (padded)
    double2 pay[SEQ ? 1 : (sizeof(T) == 8 ? 128 : 64)][NORD];  // LB window-carry staging (one round)
  };
  T2 wst[NW][NORD][4];              // per-warp segment starts of the transposed scan
  // powers for folding segment starts into thread states ({re, re, -im, im} entries):
  // [p][r] = z^{L r} (r < SEG), [p][SEG + g] = z^{L SEG g} (g < SEGS)
  static constexpr int SEG = NORD <= 8 ? 8 : 16;
  static constexpr int SEGS = 32 / SEG;
  T ptab[NORD][SEG + SEGS][4];
  long long tile;
  unsigned int epoch;
};

// LB phase timestamps for tools/scan_trace.py, compiled in only with -DSFTK_TRACE=1
// (SFTGPU_EXTRA_NVCC_FLAGS): 0 entry, 1 ticket, 2 staged, 3 published, 4 carry, 5 done,
// 6 lead-only sums, 7 window-carry start.
#ifndef SFTK_TRACE
#define SFTK_TRACE 0
#endif
template <typename T>
__device__ __forceinline__ void trace_ev(const ScanParams<T>& P, long long gt, int ev) {
  if constexpr (SFTK_TRACE) {
    if (P.trace && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      P.trace[gt * 8 + ev] = static_cast<long long>(t);
    }
  }
}

// LB-mode carry (warp 0). The window state depends only on the last 2K leading
// samples, V[n] = sum_{m=n-2K+1}^{n} z^{n-m} x[m+K], so the carry into tile t is the
// finite sum  sum_{d=1}^{D} z^{TT(d-1)} LA_{t-d} + z^{TT D} SA_{t-D-1}  of the
// predecessors' lead-only aggregates (LA: whole tile, SA: its last r positions).
// Every tile publishes (LA, SA) as soon as its samples are staged; nothing waits on a
// chain of inclusive prefixes. Flags: (epoch << 32) | 1, payload LA in `agg`, SA in
// `incl`. Staged 32 KS predecessors per round (KS per lane: 2 fp32, 4 fp64), Horner from
// the oldest (fp64).
template <typename T, int NORD, int L, int NT, bool SEQ>
__device__ __forceinline__ void window_carry(const ScanParams<T>& P, Smem<T, NORD, L, NT, SEQ>& S, long long gt,
                                             long long first, int lane) {
  double2 acc = make_double2(0.0, 0.0);
  const double2 zT = lane < NORD ? P.tab_tile[lane * kTabTileStride] : make_double2(1.0, 0.0);
  constexpr int KS = sizeof(T) == 8 ? 4 : 2, R = 32 * KS;  // predecessors per lane / round
  for (int hi = P.lb_D + 1; hi >= 1; hi -= R) {
    const int lo_d = hi - (R - 1) > 1 ? hi - (R - 1) : 1;
    const int cnt = hi - lo_d + 1;
    // Each lane stages predecessors j = lane + 32 k (k < KS) in two round trips: all its
    // flags polled together (relaxed), one acquire fence, then all payloads in flight
    // together (a poll + payload pair per predecessor would be 2 KS).
    const unsigned int ep = S.epoch;
    long long t[KS];
    bool live[KS];
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const int j = lane + 32 * k;
      t[k] = gt - (hi - j);
      live[k] = j < cnt && t[k] >= first;
    }
    if constexpr (sizeof(T) == 4) {
      // tagged payloads: one round trip when the predecessors have published
      const unsigned long long tg = pay_tag(ep);
      constexpr int KB = NORD <= 8 ? 2 : 1;  // predecessors in flight per lane (registers)
#pragma unroll
      for (int k0 = 0; k0 < KS; k0 += KB) {
        unsigned long long w[KB][NORD][2];
        auto load = [&](int kk) {
          const int k = k0 + kk;
          const double2* src = ((hi - (lane + 32 * k) == P.lb_D + 1) ? P.incl : P.agg) + t[k] * NORD;
#pragma unroll
          for (int p = 0; p < NORD; ++p) ld_relaxed_v2(src + p, w[kk][p][0], w[kk][p][1]);
        };
#pragma unroll
        for (int kk = 0; kk < KB; ++kk)
          if (live[k0 + kk]) load(kk);
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {
          if (!live[k0 + kk]) continue;
          for (;;) {
            bool ok = true;
#pragma unroll
            for (int p = 0; p < NORD; ++p) ok = ok && (w[kk][p][0] & 15ull) == tg && (w[kk][p][1] & 15ull) == tg;
            if (ok) break;
            load(kk);
          }
        }
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {
          const int j = lane + 32 * (k0 + kk);
          if (j < cnt) {
#pragma unroll
            for (int p = 0; p < NORD; ++p)
              S.pay[j][p] = live[k0 + kk] ? make_double2(untag_word(w[kk][p][0]), untag_word(w[kk][p][1]))
                                          : make_double2(0.0, 0.0);
          }
        }
      }
    } else {
      unsigned long long f[KS];
#pragma unroll
      for (int k = 0; k < KS; ++k) f[k] = live[k] ? ld_relaxed_u64(P.flags + t[k]) : 0ull;
#pragma unroll
      for (int k = 0; k < KS; ++k)
        if (live[k])
          while (static_cast<unsigned int>(f[k] >> 32) != ep) f[k] = ld_relaxed_u64(P.flags + t[k]);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      double2 v[KS][NORD];
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        const double2* src = (hi - (lane + 32 * k) == P.lb_D + 1) ? P.incl : P.agg;
#pragma unroll
        for (int p = 0; p < NORD; ++p) v[k][p] = live[k] ? __ldcg(src + t[k] * NORD + p) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int k = 0; k < KS; ++k)
        if (lane + 32 * k < cnt) {
#pragma unroll
          for (int p = 0; p < NORD; ++p) S.pay[lane + 32 * k][p] = v[k][p];
        }
    }
    __syncwarp();
    if (hi == P.lb_D + 1 && hi <= R) {
      // Single round (the common case, D + 1 <= R): G lane groups each Horner one
      // segment of the predecessors and scale it by z^{TT (cnt - segment end)} (host
      // table), then the groups are summed with shuffles: the fp64 dependency chain is
      // cnt / G long instead of cnt.
      constexpr int G = NORD <= 8 ? 4 : 2, WG = 32 / G;
      const int g = lane / WG, p = lane % WG;
      const int seg = (cnt + G - 1) / G;
      const int j0 = g * seg, j1 = min(cnt, j0 + seg);
      double2 part = make_double2(0.0, 0.0);
      if (p < NORD) {
        const double2 zp = P.tab_tile[p * kTabTileStride];
        for (int j = j0; j < j1; ++j) part = cadd(cmul(part, zp), S.pay[j][p]);
        part = cmul(part, P.tab_tile[p * kTabTileStride + 2 + g]);
      }
#pragma unroll
      for (int off = WG; off < 32; off <<= 1) {
        part.x += __shfl_xor_sync(0xffffffffu, part.x, off);
        part.y += __shfl_xor_sync(0xffffffffu, part.y, off);
      }
      acc = part;
    } else if (lane < NORD) {
      for (int j = 0; j < cnt; ++j) acc = cadd(cmul(acc, zT), S.pay[j][lane]);
    }
    __syncwarp();
  }
  if (lane < NORD) S.carry[lane] = acc;
  __syncwarp();
}

// ---- asynchronous staging (LDGSTS): global -> shared without holding registers
__device__ __forceinline__ unsigned long long l2_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <typename T>
__device__ __forceinline__ void cp_async(T* dst, const T* src, unsigned long long pol) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], %2, %3;"
               :: "r"(d), "l"(src), "n"(sizeof(T)), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Stages one stream of a tile (element e = tid + k*NT, coalesced) starting at signal
// index j0 into shared memory (padded index e + e/32). Samples before jmin are the
// virtual zeros ahead of the warm start; indices outside [0, n) follow the boundary
// policy. A segment lies inside the signal (asynchronous copies), entirely in one
// boundary region (uniform fill), or straddles an edge (per-element checks: at most
// two segments per signal and stream).
template <typename T, int L, int NT>
__device__ __forceinline__ void stage_stream(const ScanParams<T>& P, const T* __restrict__ xs, long long j0,
                                             long long jmin, int tid, unsigned long long pol, T* dst) {
  constexpr int TT = NT * L;
  const long long n = P.n;
  if (j0 >= jmin && j0 >= 0 && j0 + TT <= n) {
    const T* src = xs + j0;
#pragma unroll
    for (int k = 0; k < L; ++k) {
      const int e = tid + k * NT;
      cp_async(dst + e + (e >> 5), src + e, pol);
    }
    return;
  }
  if (j0 + TT <= jmin || (j0 >= jmin && (j0 >= n || j0 + TT <= 0))) {
    T v = T(0);
    if (j0 + TT > jmin && P.boundary != 0) v = __ldg(xs + (j0 >= n ? n - 1 : 0));
#pragma unroll
    for (int k = 0; k < L; ++k) {
      const int e = tid + k * NT;
      dst[e + (e >> 5)] = v;
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const int e = tid + k * NT;
    const long long j = j0 + e;
    dst[e + (e >> 5)] = j < jmin ? T(0) : load_ext(xs, n, P.boundary, j);
  }
}

// Register variant of stage_stream (same classification), for the one-tile LB path:
// both streams' loads are issued before any shared-memory store, so the two DRAM
// round trips overlap.
template <typename T, int L, int NT, bool KEEP>
__device__ __forceinline__ void fetch_stream(const ScanParams<T>& P, const T* __restrict__ xs, long long j0,
                                             long long jmin, int tid, unsigned long long pol, T (&f)[L]) {
  constexpr int TT = NT * L;
  const long long n = P.n;
  if (j0 >= jmin && j0 >= 0 && j0 + TT <= n) {
    const T* p = xs + j0 + tid;
#pragma unroll
    for (int k = 0; k < L; ++k) f[k] = KEEP ? ld_keep(p + k * NT, pol) : __ldcs(p + k * NT);
    return;
  }
  if (j0 + TT <= jmin || (j0 >= jmin && (j0 >= n || j0 + TT <= 0))) {
    T v = T(0);
    if (j0 + TT > jmin && P.boundary != 0) v = __ldg(xs + (j0 >= n ? n - 1 : 0));
#pragma unroll
    for (int k = 0; k < L; ++k) f[k] = v;
    return;
  }
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const long long j = j0 + tid + k * NT;
    f[k] = j < jmin ? T(0) : load_ext(xs, n, P.boundary, j);
  }
}

// Stages the tile starting at output index o0: output o reads lead x[lo+o+K] and trail
// x[lo+o-K]; both are zero before the warm start (o < -2K for the lead, o < 0 for the
// trail), i.e. below signal index lo - K in either stream. Leading samples are re-read
// 2K positions later as trailing samples (L2 evict_last); trailing reads are their last
// use (evict_first). Completion: cp_async_wait_all + barrier.
template <typename T, int L, int NT, bool ASYNC>
__device__ __forceinline__ void stage_tile(const ScanParams<T>& P, const T* __restrict__ xs, long long lo,
                                           long long o0, int tid, T* sl, T* stl) {
  const long long jmin = lo - P.K;
  if constexpr (ASYNC) {
    stage_stream<T, L, NT>(P, xs, lo + o0 + P.K, jmin, tid, l2_keep_policy(), sl);
    stage_stream<T, L, NT>(P, xs, lo + o0 - P.K, jmin, tid, l2_first_policy(), stl);
    cp_async_commit();
  } else {
    T fl[L], ft[L];
    fetch_stream<T, L, NT, true>(P, xs, lo + o0 + P.K, jmin, tid, l2_keep_policy(), fl);
    fetch_stream<T, L, NT, false>(P, xs, lo + o0 - P.K, jmin, tid, 0ull, ft);
#pragma unroll
    for (int k = 0; k < L; ++k) {
      const int e = tid + k * NT;
      sl[e + (e >> 5)] = fl[k];
      stl[e + (e >> 5)] = ft[k];
    }
  }
}

// Complex arithmetic on the recurrence state. fp32: packed pair {re, im} in one 64-bit
// register, every complex multiply-add = two FFMA2; fp64: scalar DFMA.
template <typename T>
struct Cx;

template <>
struct Cx<float> {
  using S = u64;
  using C = OrdConst<float>;
  static __device__ __forceinline__ S zero() { return 0ull; }
  static __device__ __forceinline__ S make(float a, float b) { return pk(a, b); }
  static __device__ __forceinline__ float re(S v) { return plo(v); }
  static __device__ __forceinline__ float im(S v) { return phi(v); }
  // v + w u, w packed as {wr, wr, -wi, wi}
  static __device__ __forceinline__ S madd(const float* w4, S u, S v) {
    return fma2(ldp(w4 + 2), pswap(u), fma2(ldp(w4), u, v));
  }
  // z V + g, g packed {gr, gi}
  static __device__ __forceinline__ S step(const C& c, S V, S g) {
    return fma2(ldp(c.zx), pswap(V), fma2(ldp(c.zz), V, g));
  }
  // acc + {k1 Vr + k2 Vi, k3 Vr + k4 Vi}
  static __device__ __forceinline__ S comb(const C& c, S V, S acc) {
    return fma2(ldp(c.kb), pk(im(V), im(V)), fma2(ldp(c.ka), pk(re(V), re(V)), acc));
  }
  static __device__ __forceinline__ float comb_re(const C& c, S V, float acc) {
    return fmaf(c.ka[0], re(V), fmaf(c.kb[0], im(V), acc));
  }
  // acc + z^{L-1-i} g for real g / complex g = {gr, gi}
  static __device__ __forceinline__ S agg_r(const C& c, int i, float g, S acc) {
    return fma2(ldp(&c.w[i][0]), pk(g, g), acc);
  }
  static __device__ __forceinline__ S agg_c(const C& c, int i, S g, S acc) {
    return fma2(ldp(&c.w[i][2]), pk(im(g), im(g)), fma2(ldp(&c.w[i][0]), pk(re(g), re(g)), acc));
  }
  static __device__ __forceinline__ S shfl(S v, int src) {
    return pk(__shfl_sync(0xffffffffu, re(v), src), __shfl_sync(0xffffffffu, im(v), src));
  }
  static __device__ __forceinline__ S warp_sum(S v) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) v = xor_add(v, d);
    return v;
  }
  static __device__ __forceinline__ S xor_add(S v, int d) {  // one butterfly level of warp_sum
    return fma2(pk(1.0f, 1.0f), pk(__shfl_xor_sync(0xffffffffu, re(v), d), __shfl_xor_sync(0xffffffffu, im(v), d)), v);
  }
};

template <>
struct Cx<double> {
  using S = double2;
  using C = OrdConst<double>;
  static __device__ __forceinline__ S zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ S make(double a, double b) { return make_double2(a, b); }
  static __device__ __forceinline__ double re(S v) { return v.x; }
  static __device__ __forceinline__ double im(S v) { return v.y; }
  static __device__ __forceinline__ S madd(const double* w4, S u, S v) {
    const double wr = w4[0], wi = w4[3];
    return make_double2(fma(wr, u.x, fma(-wi, u.y, v.x)), fma(wr, u.y, fma(wi, u.x, v.y)));
  }
  static __device__ __forceinline__ S step(const C& c, S V, S g) {
    const double zr = c.zz[0], zi = c.zx[1];
    return make_double2(fma(zr, V.x, fma(-zi, V.y, g.x)), fma(zr, V.y, fma(zi, V.x, g.y)));
  }
  static __device__ __forceinline__ S comb(const C& c, S V, S acc) {
    return make_double2(fma(c.ka[0], V.x, fma(c.kb[0], V.y, acc.x)), fma(c.ka[1], V.x, fma(c.kb[1], V.y, acc.y)));
  }
  static __device__ __forceinline__ double comb_re(const C& c, S V, double acc) {
    return fma(c.ka[0], V.x, fma(c.kb[0], V.y, acc));
  }
  static __device__ __forceinline__ S agg_r(const C& c, int i, double g, S acc) {
    return make_double2(fma(c.w[i][0], g, acc.x), fma(c.w[i][1], g, acc.y));
  }
  static __device__ __forceinline__ S agg_c(const C& c, int i, S g, S acc) {
    return make_double2(fma(c.w[i][0], g.x, fma(-c.w[i][1], g.y, acc.x)), fma(c.w[i][1], g.x, fma(c.w[i][0], g.y, acc.y)));
  }
  static __device__ __forceinline__ S shfl(S v, int src) {
    return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
  }
  static __device__ __forceinline__ S warp_sum(S v) { return warp_sum2(v); }
  static __device__ __forceinline__ S xor_add(S v, int d) {  // one butterfly level of warp_sum
    v.x += __shfl_xor_sync(0xffffffffu, v.x, d);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, d);
    return v;
  }
};

// One tile: stage samples, phase 1, scans, carry (SEQ: from smem; LB: look-back),
// phase 2, stores. `fl/ft` hold this tile's prefetched samples on entry and the next
// tile's on exit when `has_next`.
template <typename T, int NORD, int NA, int GM, int MODE, int L, int NT, bool SEQ>
__device__ __forceinline__ void do_tile(const ScanParams<T>& P, Smem<T, NORD, L, NT, SEQ>& S, long long sig,
                                        long long gt, long long first, long long lo, long long count,
                                        long long obase, long long o0, const T* __restrict__ xs,
                                        bool has_next) {
  using X = Cx<T>;
  using St = typename X::S;
  using T2 = typename Vec2<T>::t;
  constexpr int TT = NT * L;
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool warm = o0 + TT <= 0;
  // staging buffer parity: alternate per tile so the next tile's stores never race
  // this tile's reads (buffer b was last read two tiles ago, behind two barriers)
  const int b = SEQ ? static_cast<int>(((o0 / TT) % 2 + 2) % 2) : 0;
  T* const sl = S.lead[b];
  T* const stl = S.trail[b];

  if constexpr (SEQ) cp_async_wait_all();
  __syncthreads();  // this tile staged; the other buffer's last readers are done
  if constexpr (!SEQ) trace_ev(P, gt, 2);
  if constexpr (SEQ) {
    if (has_next) stage_tile<T, L, NT, true>(P, xs, lo, o0 + TT, tid, S.lead[b ^ 1], S.trail[b ^ 1]);
  }

  if constexpr (!SEQ) {
    // ---- lead-only aggregates (whole tile and its last r positions), published for
    // the successors' window carries. Samples are read once, and every order's two sums
    // go through the butterfly together (independent chains the scheduler interleaves;
    // the tile's publication waits on this block).
    {
      T xv[L];
#pragma unroll
      for (int i = 0; i < L; ++i) {
        const int e = tid * L + i;
        xv[i] = sl[e + (e >> 5)];
      }
      St la[NORD], sa[NORD];
#pragma unroll
      for (int p = 0; p < NORD; ++p) {
        const OrdConst<T>& c = P.oc[p];
        la[p] = X::zero();
        sa[p] = X::zero();
#pragma unroll
        for (int i = 0; i < L; ++i) {
          const int e = tid * L + i;
          la[p] = X::agg_r(c, i, xv[i], la[p]);
          sa[p] = X::agg_r(c, i, e >= P.lb_sfx ? xv[i] : T(0), sa[p]);
        }
        const T* rot = P.tab + (p * kTabStride + 31 - lane) * 4;  // z^{L(31-lane)} (prefetched)
        la[p] = X::madd(rot, la[p], X::zero());
        sa[p] = X::madd(rot, sa[p], X::zero());
      }
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) {
#pragma unroll
        for (int p = 0; p < NORD; ++p) {
          la[p] = X::xor_add(la[p], d);
          sa[p] = X::xor_add(sa[p], d);
        }
      }
      if (lane == 0) {
#pragma unroll
        for (int p = 0; p < NORD; ++p) {
          S.wla[warp][p] = make2<T2>(X::re(la[p]), X::im(la[p]));
          S.wsa[warp][p] = make2<T2>(X::re(sa[p]), X::im(sa[p]));
        }
      }
    }
    trace_ev(P, gt, 6);
    __syncthreads();
    if (tid < NORD) {
      const int p = tid;
      St a = X::zero(), b2 = X::zero();
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        a = X::madd(P.oc[p].m32, a, X::make(S.wla[w][p].x, S.wla[w][p].y));
        b2 = X::madd(P.oc[p].m32, b2, X::make(S.wsa[w][p].x, S.wsa[w][p].y));
      }
      S.tagg[p] = make_double2(static_cast<double>(X::re(a)), static_cast<double>(X::im(a)));
      S.tsfx[p] = make_double2(static_cast<double>(X::re(b2)), static_cast<double>(X::im(b2)));
      if constexpr (sizeof(T) == 4) {
        const unsigned long long tg = pay_tag(S.epoch);
        st_relaxed_v2(P.agg + gt * NORD + p, tag_word(S.tagg[p].x, tg), tag_word(S.tagg[p].y, tg));
        st_relaxed_v2(P.incl + gt * NORD + p, tag_word(S.tsfx[p].x, tg), tag_word(S.tsfx[p].y, tg));
      }
    }
    if constexpr (sizeof(T) == 4) {
      trace_ev(P, gt, 3);
    } else if (warp == 0) {
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int p = 0; p < NORD; ++p) {
          __stcg(P.agg + gt * NORD + p, S.tagg[p]);
          __stcg(P.incl + gt * NORD + p, S.tsfx[p]);
        }
        st_release_u64(P.flags + gt, (static_cast<unsigned long long>(S.epoch) << 32) | 1ull);
      }
      trace_ev(P, gt, 3);
    }
    if (warm) {
      trace_ev(P, gt, 5);
      return;  // warm tiles only feed their successors' windows
    }
  }

  // ---- injections, shared across orders where the group mode allows. Samples are
  // read from shared memory per position in both phases (no per-position registers).
  // gA = x[n+K] - cA x[n-K] (real), gB = x[n+K] - cB x[n-K] (complex, split modes).
  auto sample = [&](int i, T& xl, T& xt) {
    const int e = tid * L + i;
    xl = sl[e + (e >> 5)];
    xt = stl[e + (e >> 5)];
  };
  auto inj = [&](const OrdConst<T>& c, int p, T xl, T xt) -> St {
    if (GM == kGroupShared || (GM == kGroupSplit && p < NA)) return X::make(fma(-P.cAr, xt, xl), T(0));
    if constexpr (GM == kGroupSplit) return X::make(fma(-P.cBr, xt, xl), -P.cBi * xt);
    return X::make(fma(-c.cc[0], xt, xl), -c.cc[1] * xt);
  };

  // ---- phase 1: per-thread aggregate with zero state in (positions outer; each
  // order's sum runs over i in the same order as a per-order loop would)
  St st[NORD];
#pragma unroll
  for (int p = 0; p < NORD; ++p) st[p] = X::zero();
#pragma unroll
  for (int i = 0; i < L; ++i) {
    T xl, xt;
    sample(i, xl, xt);
#pragma unroll
    for (int p = 0; p < NORD; ++p) {
      const OrdConst<T>& c = P.oc[p];
      if (GM == kGroupShared || (GM == kGroupSplit && p < NA))
        st[p] = X::agg_r(c, i, fma(-P.cAr, xt, xl), st[p]);
      else
        st[p] = X::agg_c(c, i, inj(c, p, xl, xt), st[p]);
    }
  }

  // ---- warp-level exclusive scan, transposed and segmented: every thread parks its
  // per-order aggregates in shared memory (padded stride 33: conflict-free). The 32
  // aggregates of an order are cut into SEGS segments of SEG; lane (segment g, order p)
  // runs the SEG-step Horner chain of its segment, writing local exclusive prefixes in
  // place, and the segment totals are chained across lanes with SEGS-1 shuffles. The
  // segment start is folded into the per-thread state once the warp carry is known.
  constexpr int SEG = Smem<T, NORD, L, NT, SEQ>::SEG;
  constexpr int SEGS = Smem<T, NORD, L, NT, SEQ>::SEGS;
  {
    T2* wa = S.wscan[warp];
#pragma unroll
    for (int p = 0; p < NORD; ++p) wa[p * 33 + lane] = make2<T2>(X::re(st[p]), X::im(st[p]));
    __syncwarp();
    const int sp = lane % SEG, sg = lane / SEG;
    const bool act = sp < NORD;
    const int po = act ? sp : 0;
    St run = X::zero();
    if (act) {
      const T* zl = P.oc[sp].scan[0];  // z^L
#pragma unroll
      for (int j = 0; j < SEG; ++j) {
        const int idx = sp * 33 + sg * SEG + j;
        const T2 a = wa[idx];
        wa[idx] = make2<T2>(X::re(run), X::im(run));
        run = X::madd(zl, run, X::make(a.x, a.y));
      }
    }
    const T* zs = S.ptab[po][SEG + 1];  // z^{L SEG}
    St start = X::zero();
#pragma unroll
    for (int g = 0; g < SEGS - 1; ++g) {
      const St tg = X::shfl(run, sp + g * SEG);
      if (g < sg) start = X::madd(zs, start, tg);
    }
    if (act) {
      S.wst[warp][sp][sg] = make2<T2>(X::re(start), X::im(start));
      if (sg == SEGS - 1) {
        const St tot = X::madd(zs, start, run);
        S.w[warp][sp] = make2<T2>(X::re(tot), X::im(tot));
      }
    }
    __syncwarp();
#pragma unroll
    for (int p = 0; p < NORD; ++p) {
      const T2 e = wa[p * 33 + lane];
      st[p] = X::make(e.x, e.y);
    }
  }
  __syncthreads();

  // ---- one thread per order: inter-warp scan, tile aggregate, carry, per-warp carries
  if (tid < NORD) {
    const int p = tid;

    St ex[NW];
    St run = X::zero();
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      ex[w] = run;
      const T2 t = S.w[w][p];
      run = X::madd(P.oc[p].m32, run, X::make(t.x, t.y));  // z^{32L} run + total_w
    }
    if constexpr (SEQ) {
      S.tagg[p] = make_double2(static_cast<double>(X::re(run)), static_cast<double>(X::im(run)));
      const double2 c = S.carry[p];
      const St cs = X::make(static_cast<T>(c.x), static_cast<T>(c.y));
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const St r = X::madd(P.oc[p].wrot[w], cs, ex[w]);
        S.w[w][p] = make2<T2>(X::re(r), X::im(r));
      }
      S.carry[p] = cadd(cmul(P.tab_tile[p * kTabTileStride], c), S.tagg[p]);
    } else {
#pragma unroll
      for (int w = 0; w < NW; ++w) S.w[w][p] = make2<T2>(X::re(ex[w]), X::im(ex[w]));
    }
  }
  if constexpr (!SEQ) {
    if (warp == 0) {
      __syncwarp();
      trace_ev(P, gt, 7);
      window_carry<T, NORD, L, NT, SEQ>(P, S, gt, first, lane);
      trace_ev(P, gt, 4);
      if (tid < NORD) {
        const int p = tid;

        const St cs = X::make(static_cast<T>(S.carry[p].x), static_cast<T>(S.carry[p].y));
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const T2 e = S.w[w][p];
          const St r = X::madd(P.oc[p].wrot[w], cs, X::make(e.x, e.y));
          S.w[w][p] = make2<T2>(X::re(r), X::im(r));
        }
      }
    }
  }
  __syncthreads();
  if (warm) return;  // SEQ warm tile: phase 1 only (uniform per CTA)

  // state entering this thread's positions:
  //   z^{L lane} Cw + exclusive(lane) = e_local + z^{L r} (start_g + z^{L SEG g} Cw),
  // lane = g SEG + r, e_local its in-segment exclusive prefix
  {
    const int g = lane / SEG, r = lane % SEG;
#pragma unroll
    for (int p = 0; p < NORD; ++p) {
      const T2 cw = S.w[warp][p];
      const T2 s0 = S.wst[warp][p][g];
      const St adj = X::madd(S.ptab[p][SEG + g], X::make(cw.x, cw.y), X::make(s0.x, s0.y));
      st[p] = X::madd(S.ptab[p][r], adj, st[p]);
    }
  }

  // ---- phase 2: re-run the recurrence from the true state and combine
  const long long ob = o0 + static_cast<long long>(tid) * L;
  if constexpr (MODE == kModeComps) {
#pragma unroll
    for (int p = 0; p < NORD; ++p) {
      const OrdConst<T>& c = P.oc[p];
      St v = st[p];
      T* cptr = P.out + p * P.ord_stride + sig * P.ld_out + obase;
      T* sptr = P.out_s + p * P.ord_stride + sig * P.ld_out + obase;
#pragma unroll
      for (int i = 0; i < L; ++i) {
        T xl, xt;
        sample(i, xl, xt);
        v = X::step(c, v, inj(c, p, xl, xt));
        const long long o = ob + i;
        if (o < count) {
          // c = Re(a V + b x_t), s = -Im(a V + b x_t), a = (k1, k2), b = (k3, k4) = (ka[1], kb[1])
          const T vr = X::re(v), vi = X::im(v);
          cptr[o] = fma(c.ka[0], vr, fma(-c.kb[0], vi, c.ka[1] * xt));
          sptr[o] = -fma(c.kb[0], vr, fma(c.ka[0], vi, c.kb[1] * xt));
        }
      }
    }
  } else {
    constexpr bool CPLX = MODE == kModeComplex;
    constexpr int CW = CPLX ? 2 : 1;    // T words per output
    constexpr int VW = 16 / sizeof(T);  // T words per 16-byte vector
    constexpr int VP = VW / CW;         // outputs per vector
    static_assert(L % VP == 0, "positions per thread must fill whole vectors");
    constexpr int CH = VP;  // outputs computed per store batch
    T* const optr = P.out + CW * (sig * P.ld_out + obase);
    const bool vec = P.vec_ok && !P.accumulate && ob + L <= count;
    // positions outer, orders inner: NORD independent recurrence chains per position
#pragma unroll
    for (int i0 = 0; i0 < L; i0 += CH) {
      T buf[CH * CW];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        T xl, xt;
        sample(i0 + j, xl, xt);
        St acc = X::make(P.Dr * xt, CPLX ? P.Di * xt : T(0));
        T accr = P.Dr * xt;
#pragma unroll
        for (int p = 0; p < NORD; ++p) {
          const OrdConst<T>& c = P.oc[p];
          st[p] = X::step(c, st[p], inj(c, p, xl, xt));
          if constexpr (CPLX)
            acc = X::comb(c, st[p], acc);
          else
            accr = X::comb_re(c, st[p], accr);
        }
        if constexpr (CPLX) {
          buf[2 * j] = X::re(acc);
          buf[2 * j + 1] = X::im(acc);
        } else {
          buf[j] = accr;
        }
      }
      if (vec) {
        T* dst = optr + (ob + i0) * CW;
#pragma unroll
        for (int v = 0; v < CH * CW / VW; ++v) {
          if constexpr (sizeof(T) == 4)
            __stcs(reinterpret_cast<float4*>(dst) + v,
                   make_float4(buf[4 * v], buf[4 * v + 1], buf[4 * v + 2], buf[4 * v + 3]));
          else
            __stcs(reinterpret_cast<double2*>(dst) + v, make_double2(buf[2 * v], buf[2 * v + 1]));
        }
      } else {
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const long long o = ob + i0 + j;
          if (o < count) {
#pragma unroll
            for (int w = 0; w < CW; ++w) {
              if (P.accumulate)
                optr[o * CW + w] += buf[j * CW + w];
              else
                optr[o * CW + w] = buf[j * CW + w];
            }
          }
        }
      }
    }
  }
}

template <typename T, int NORD, int NA, int GM, int MODE, int L, int NT, bool SEQ>
__global__ void __launch_bounds__(NT, (sizeof(T) == 4 ? (SEQ ? (L >= 16 ? 5 : (NORD <= 8 ? SFTK_SEQ_MINB : 6)) : 4) : 2)) sft_scan_kernel(const __grid_constant__ ScanParams<T> P) {
  static_assert(NORD >= 1 && NORD <= kMaxOrd, "order count");
  static_assert(L <= kMaxL, "positions per thread");
  constexpr int TT = NT * L;
  extern __shared__ __align__(16) unsigned char smem_raw[];  // sized by the launcher
  Smem<T, NORD, L, NT, SEQ>& S = *reinterpret_cast<Smem<T, NORD, L, NT, SEQ>*>(smem_raw);
  const int tid = threadIdx.x;
  // LB: count this CTA in; the result (the launch's epoch) is first needed when the
  // tile publishes, so the round trip overlaps the table and sample staging
  unsigned long long started = 0;
  unsigned long long t_entry = 0;
  if constexpr (!SEQ) {
    if constexpr (SFTK_TRACE) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_entry));
    if (tid == 0) started = atomicAdd(reinterpret_cast<unsigned long long*>(P.ctrl), 1ull);
  }
  if constexpr (!SEQ) {
    // tables read later on the tile's chain (lead-only warp sums, window carry): start
    // their fetch now, without waiting on it
    // (one warp: every CTA of the launch reads the same few table lines at once)
    if (tid < 32) {
#pragma unroll
      for (int p = 0; p < NORD; ++p)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(P.tab + (p * kTabStride + 31 - tid) * 4));
      if (tid < NORD) asm volatile("prefetch.global.L1 [%0];" ::"l"(P.tab_tile + tid * kTabTileStride));
    }
  }
  // segment-power table: every load issued now, stored after the tile's sample loads
  // are in flight too (LB), so the two round trips overlap
  using Sm = Smem<T, NORD, L, NT, SEQ>;
  constexpr int E = Sm::SEG + Sm::SEGS;
  constexpr int NQ = (NORD * E * 4 + NT - 1) / NT;
  T ptv[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) {
    const int q = tid + k * NT;
    if (q < NORD * E * 4) {
      const int p = q / (E * 4), j = (q / 4) % E, w = q % 4;
      const int src = j < Sm::SEG ? j : Sm::SEG * (j - Sm::SEG);
      ptv[k] = P.tab[(p * kTabStride + src) * 4 + w];
    }
  }
  auto store_ptab = [&]() {
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const int q = tid + k * NT;
      if (q < NORD * E * 4) (&S.ptab[0][0][0])[q] = ptv[k];
    }
  };

  if constexpr (SEQ) {
    // one CTA per (signal, chunk): tiles in order from the chunk's own warm start,
    // carry in shared memory
    const long long sig = blockIdx.x / P.n_chunks;
    const long long ch = blockIdx.x - sig * P.n_chunks;
    const long long obase = ch * P.chunk_len;
    const long long lo = P.lo + obase;
    const long long count = P.count - obase < P.chunk_len ? P.count - obase : P.chunk_len;
    const long long tiles = P.warm_tiles + (count + TT - 1) / TT;
    const T* __restrict__ xs = P.x + sig * P.ld_x;
    if (tid < NORD) S.carry[tid] = make_double2(0.0, 0.0);
    const long long o_first = -P.warm_tiles * TT;
    const int b0 = static_cast<int>(((o_first / TT) % 2 + 2) % 2);
    stage_tile<T, L, NT, true>(P, xs, lo, o_first, tid, S.lead[b0], S.trail[b0]);
    store_ptab();  // read after do_tile's first barrier
    for (long long t = 0; t < tiles; ++t)
      do_tile<T, NORD, NA, GM, MODE, L, NT, true>(P, S, sig, 0, 0, lo, count, obase, o_first + t * TT, xs,
                                                  t + 1 < tiles);
  } else {
    // tiles in block order: a tile only waits on tiles of lower index, so staging starts
    // at once. Forward progress assumes the hardware starts a grid's CTAs in blockIdx
    // order (as CUB's single-pass scan does): a spinning CTA's predecessors have then all
    // started and never wait on it. This holds with other kernels running concurrently
    // (the scalogram's streams): they only delay when this grid's next CTA starts.
    const long long gt = blockIdx.x;
    if constexpr (SFTK_TRACE) {
      if (P.trace && tid == 0) P.trace[gt * 8] = static_cast<long long>(t_entry);
    }
    trace_ev(P, gt, 1);
    const long long sig = gt / P.tiles_per_signal;
    const long long first = sig * P.tiles_per_signal;
    const long long o0 = (gt - first - P.warm_tiles) * TT;
    const T* __restrict__ xs = P.x + sig * P.ld_x;
    stage_tile<T, L, NT, false>(P, xs, P.lo, o0, tid, S.lead[0], S.trail[0]);
    store_ptab();  // read after do_tile's first barrier
    // epoch >= 1 (read after do_tile's barrier). The plan zeroes its flags and payloads:
    // flag epoch 0 and payload tag 0 never match a live launch.
    if (tid == 0) S.epoch = static_cast<unsigned int>(started / static_cast<unsigned long long>(P.total_tiles)) + 1u;
    do_tile<T, NORD, NA, GM, MODE, L, NT, false>(P, S, sig, gt, first, P.lo, P.count, 0, o0, xs, false);
    if (o0 + TT > 0) trace_ev(P, gt, 5);
  }
}

}  // namespace sftk
