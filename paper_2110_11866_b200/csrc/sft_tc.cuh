// K4 — tensor-core chunked SFT/ASFT transform (tcgen05, 3xTF32), sm_100a.
//
// Same transform as K1 (sft_scan.cuh; reference proj/src/transforms.cpp:279-428 over
// proj/src/engine.cpp:53-219), re-associated so the per-sample work runs on the
// tensor cores instead of the FP32 pipe. With chunks of Q = 32 positions (chunk c of a
// 4096-position tile, position i, o = o0 + 32 c + i), every order's 2K-window state
// V_p obeys
//   V_p[o0+32c+i] = z^{i+1} S_p[c] + sum_{m<=i} z^{i-m} (xl[m] - c_inj xt[m])
//   S_p[c+1]      = z^{32} S_p[c] + A_p[c],  A_p[c] = sum_m z^{31-m} (xl[m] - c_inj xt[m])
// and the combined output sum_p K_p(V_p) + D xt is, per chunk,
//   out[c, :] = xl[c, :] HL^T + xt[c, :] HT^T + S[c, :] CS^T          (GEMM2, N = 2Q or Q)
//   A[c, :]   = xl[c, :] AL^T + xt[c, :] AT^T                          (GEMM1, N = 16)
// HL/HT are lower-triangular Toeplitz blocks of the effective kernel, CS maps the chunk
// start states to the outputs, AL/AT produce the chunk aggregates; all are built on
// the host in fp64 (sftgpu_api.cu, build_tc_image). The chunk-state scan
// S[c] = z^{32} S[c-1] + A[c-1] runs on CUDA cores (warp shuffles, fp64 tile carry).
//
// Precision: operands are split x = hi + lo with hi the TF32 head; each product is
// hi*hi + lo*hi + hi*lo (3xTF32), fp32 accumulation in TMEM (~1e-6 relative).
//
// Roles (one persistent CTA per SM, 448 threads):
//   warps 0-3   chunk-state scan (thread = chunk = TMEM lane); warm-up tiles only reduce
//               their aggregates into the fp64 tile carry
//   warps 4-7   epilogue: TMEM -> registers -> swizzled staging -> coalesced 16-byte stores
//   warps 8-11  loader: cp.async (LDGSTS) of the raw samples straight into the SW128 hi
//               tiles (the MMA reads them as TF32 heads), then the fp32 remainders into
//               the lo tiles; boundary segments by value
//   warps 12-13 MMA issuers (GEMM1 of every tile / GEMM2 of every output tile)
// Pipelines (mbarriers): X tiles double-buffered, GEMM1/GEMM2 accumulators
// double-buffered in TMEM, chunk-state operand single-buffered, tile carry
// double-buffered.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "sft_tc_launch.h"
#include "umma.cuh"

namespace tck {

struct Misc {
  uint64_t xfull[2], xfree[2], g1done[2], d1free[2], g2done[2], d2free[2], ssfull;
  uint32_t tmem;
  double2 cy[2][kMaxOrd];     // tile carry (state entering the tile), fp64, by tile parity
  float2 wtot[2][4][kMaxOrd]; // per-warp chunk-aggregate totals (by tile parity)
};

// (item, tile) walk shared by every role
struct Walk {
  long long item, t, ntiles, obase, cnt, sig;
  bool valid;
  __device__ void setup(const TcParams& P) {
    valid = item < P.n_items;
    if (!valid) return;
    sig = item / P.n_chunks;
    const long long ch = item - sig * P.n_chunks;
    obase = ch * P.chunk_len;
    cnt = P.count - obase < P.chunk_len ? P.count - obase : P.chunk_len;
    ntiles = P.warm_tiles + (cnt + kTile - 1) / kTile;
    t = 0;
  }
  __device__ void begin(const TcParams& P) {
    item = blockIdx.x;
    setup(P);
  }
  __device__ void advance(const TcParams& P) {
    if (++t < ntiles) return;
    item += gridDim.x;
    setup(P);
  }
  __device__ bool warm(const TcParams& P) const { return t < P.warm_tiles; }
  __device__ long long o0(const TcParams& P) const { return (t - P.warm_tiles) * kTile; }
  __device__ bool last(const TcParams& P) const { return t + 1 == ntiles; }
};


__device__ __forceinline__ float tf32_lo(float v) { return v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

__device__ __forceinline__ void cp_async4(uint32_t dst, const float* src, unsigned long long pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "l"(pol)
               : "memory");
}

// Stage one stream of a tile: element e = lt + 128 r (warp-coalesced) -> (row e / 32,
// column e % 32) of the SW128 hi/lo tiles. Returns true when the samples are in flight
// (cp.async into the hi tile; lo tile pending), false when both tiles were written.
// Segment classes as in K1's stage_stream: inside the signal, one uniform boundary
// value (before the warm start: zeros; clamp region: the edge sample), or straddling.
__device__ __forceinline__ bool stage_stream(const TcParams& P, const float* xs, long long j0, long long jmin, int lt,
                                             unsigned long long pol, unsigned char* hi, unsigned char* lo) {
  const long long n = P.n;
  const uint32_t hs = umma::smem_u32(hi);
  if (j0 >= jmin && j0 >= 0 && j0 + kTile <= n) {
    const float* p = xs + j0 + lt;
#pragma unroll
    for (int r = 0; r < 32; ++r)
      cp_async4(hs + umma::sw128_off(static_cast<uint32_t>((lt >> 5) + 4 * r), static_cast<uint32_t>(lt & 31)),
                p + 128 * r, pol);
    return true;
  }
  if (j0 + kTile <= jmin || (j0 >= jmin && (j0 >= n || j0 + kTile <= 0))) {
    float v = 0.f;
    if (j0 + kTile > jmin && P.boundary != 0) v = __ldg(xs + (j0 >= n ? n - 1 : 0));
    const float l = tf32_lo(v);
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const uint32_t off = umma::sw128_off(static_cast<uint32_t>((lt >> 5) + 4 * r), static_cast<uint32_t>(lt & 31));
      *reinterpret_cast<float*>(hi + off) = v;
      *reinterpret_cast<float*>(lo + off) = l;
    }
    return false;
  }
  float v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const long long j = j0 + lt + 128 * r;
    const long long jc = j < 0 ? 0 : (j >= n ? n - 1 : j);
    v[r] = __ldg(xs + jc);
  }
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const long long j = j0 + lt + 128 * r;
    if (j < jmin || (P.boundary == 0 && (j < 0 || j >= n))) v[r] = 0.f;
    const uint32_t off = umma::sw128_off(static_cast<uint32_t>((lt >> 5) + 4 * r), static_cast<uint32_t>(lt & 31));
    *reinterpret_cast<float*>(hi + off) = v[r];
    *reinterpret_cast<float*>(lo + off) = tf32_lo(v[r]);
  }
  return false;
}

// bulk L2 prefetch of the 16 KB a tile stream reads (clipped to the signal, 16-B aligned)
__device__ __forceinline__ void prefetch_l2(const float* xs, long long j0, long long n) {
  long long a = j0 < 0 ? 0 : j0, e = j0 + kTile > n ? n : j0 + kTile;
  if (e <= a) return;
  const uintptr_t pa = reinterpret_cast<uintptr_t>(xs + a) & ~uintptr_t(15);
  const uintptr_t pe = (reinterpret_cast<uintptr_t>(xs + e) + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pa), "r"(static_cast<uint32_t>(pe - pa))
               : "memory");
}

// lo tile from the landed hi tile (this thread's own elements; all loads before the
// stores, so they overlap instead of serialising on possible aliasing)
__device__ __forceinline__ void finish_lo(const unsigned char* hi, unsigned char* lo, int lt) {
  float v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r)
    v[r] = *reinterpret_cast<const float*>(
        hi + umma::sw128_off(static_cast<uint32_t>((lt >> 5) + 4 * r), static_cast<uint32_t>(lt & 31)));
#pragma unroll
  for (int r = 0; r < 32; ++r)
    *reinterpret_cast<float*>(lo + umma::sw128_off(static_cast<uint32_t>((lt >> 5) + 4 * r),
                                                   static_cast<uint32_t>(lt & 31))) = tf32_lo(v[r]);
}

__device__ __forceinline__ void trace_ev(const TcParams& P, long long gt, int ev) {
  if (P.trace && blockIdx.x == 0 && gt < 64) P.trace[gt * 16 + ev] = clock64();
}

__device__ __forceinline__ void bar_scan() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void bar_epi() { asm volatile("bar.sync 2, 128;" ::: "memory"); }

__device__ __forceinline__ float2 cmla(float2 z, float2 t, float2 a) {  // a + z t
  return make_float2(fmaf(z.x, t.x, fmaf(-z.y, t.y, a.x)), fmaf(z.x, t.y, fmaf(z.y, t.x, a.y)));
}

template <int B, int K>
__device__ __forceinline__ void gemm1_k(uint64_t db, uint32_t d, uint32_t id, bool trail) {
  constexpr uint32_t x0 = kX + B * 4 * kXT, ko = 32 * K;
  umma::mma_tf32_off<x0 + ko, kALh + ko>(d, db, id, K > 0);
  umma::mma_tf32_off<x0 + kXT + ko, kALh + ko>(d, db, id, 1);
  umma::mma_tf32_off<x0 + ko, kALl + ko>(d, db, id, 1);
  if (trail) {
    umma::mma_tf32_off<x0 + 2 * kXT + ko, kATh + ko>(d, db, id, 1);
    umma::mma_tf32_off<x0 + 3 * kXT + ko, kATh + ko>(d, db, id, 1);
    umma::mma_tf32_off<x0 + 2 * kXT + ko, kATl + ko>(d, db, id, 1);
  }
}

template <int B>
__device__ __forceinline__ void gemm1(uint64_t db, uint32_t tmem, bool trail) {
  const uint32_t d = tmem + 128 + 32 * B;
  constexpr uint32_t id = umma::idesc_tf32(128, 16);
  gemm1_k<B, 0>(db, d, id, trail);
  gemm1_k<B, 1>(db, d, id, trail);
  gemm1_k<B, 2>(db, d, id, trail);
  gemm1_k<B, 3>(db, d, id, trail);
}

template <int B, int K>
__device__ __forceinline__ void gemm2_k(uint64_t db, uint32_t d, uint32_t id) {
  constexpr uint32_t x0 = kX + B * 4 * kXT, ko = 32 * K;
  umma::mma_tf32_off<x0 + ko, kHLh + ko>(d, db, id, K > 0);
  umma::mma_tf32_off<x0 + kXT + ko, kHLh + ko>(d, db, id, 1);
  umma::mma_tf32_off<x0 + ko, kHLl + ko>(d, db, id, 1);
  umma::mma_tf32_off<x0 + 2 * kXT + ko, kHTh + ko>(d, db, id, 1);
  umma::mma_tf32_off<x0 + 3 * kXT + ko, kHTh + ko>(d, db, id, 1);
  umma::mma_tf32_off<x0 + 2 * kXT + ko, kHTl + ko>(d, db, id, 1);
  umma::mma_tf32_off<kSS + ko, kBC1 + ko>(d, db, id, 1);
  if (K < 2) umma::mma_tf32_off<kSS + ko, kBC2 + ko>(d, db, id, 1);
}

template <int B, int D2>
__device__ __forceinline__ void gemm2(uint64_t db, uint32_t tmem, int cplx) {
  const uint32_t d = tmem + 64 * D2;
  const uint32_t id = cplx ? umma::idesc_tf32(128, 64) : umma::idesc_tf32(128, 32);
  gemm2_k<B, 0>(db, d, id);
  gemm2_k<B, 1>(db, d, id);
  gemm2_k<B, 2>(db, d, id);
  gemm2_k<B, 3>(db, d, id);
}

template <int NORD>
__global__ void __launch_bounds__(kThreads, 1) sft_tc_kernel(const __grid_constant__ TcParams P) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  Misc& M = *reinterpret_cast<Misc*>(sm + kMisc);
  const int tid = threadIdx.x, lane = tid & 31;
  // warp index as a provably warp-uniform value: role branches become uniform branches
  // and the MMA issuers keep descriptors on the uniform datapath
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);

  // ---- setup: operand image, barriers, TMEM (256 columns: D2 x2 at 0/64, D1 x2 at 128/160)
  {
    uint4* dst = reinterpret_cast<uint4*>(sm);
    for (int i = tid; i < static_cast<int>(kImage / 16); i += kThreads) dst[i] = __ldg(P.image + i);
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&M.xfull[b], 128);
      umma::mbar_init(&M.xfree[b], 1);
      umma::mbar_init(&M.g1done[b], 1);
      umma::mbar_init(&M.d1free[b], 128);
      umma::mbar_init(&M.g2done[b], 1);
      umma::mbar_init(&M.d2free[b], 128);
    }
    umma::mbar_init(&M.ssfull, 128);
    umma::mbar_fence_init();
  }
  if (tid < kMaxOrd) M.cy[0][tid] = make_double2(0.0, 0.0);
  if (warp == 0) umma::tmem_alloc(&M.tmem, 256);
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, M.tmem, 0);  // warp-uniform
  constexpr int nord = NORD;

  if (warp >= 8 && warp < 12) {
    // ================= loader: complete tile gt-1 (lo tiles, xfull), then stage tile gt
    // into its buffer once GEMM2 of tile gt-2 has released it, and prefetch tile gt+1's
    // samples into L2 so its copies hit L2
    const int lt = tid - 256;
    unsigned long long keep, first;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(first));
    Walk w;
    w.begin(P);
    bool pend_l = false, pend_t = false;  // previous tile's streams still in flight
    long long gt = 0;
    for (; w.valid; ++gt) {
      const int b = static_cast<int>(gt & 1);
      if (gt >= 1) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        if (lt == 0) trace_ev(P, gt - 1, 14);
        unsigned char* pb = sm + kX + (b ^ 1) * 4 * kXT;
        if (pend_l) finish_lo(pb, pb + kXT, lt);
        if (pend_t) finish_lo(pb + 2 * kXT, pb + 3 * kXT, lt);
        umma::fence_proxy_async();
        umma::mbar_arrive(&M.xfull[b ^ 1]);
        if (lt == 0) trace_ev(P, gt - 1, 1);
      }
      Walk nx = w;
      nx.advance(P);
      if (lt == 0 && nx.valid) {
        const float* xs = P.x + nx.sig * P.ld_x;
        const long long lo = P.lo + nx.obase, o0 = nx.o0(P);
        prefetch_l2(xs, lo + o0 + P.K, P.n);
        if (!nx.warm(P)) prefetch_l2(xs, lo + o0 - P.K, P.n);
      }
      if (gt >= 2) umma::mbar_wait(&M.xfree[b], static_cast<uint32_t>(((gt >> 1) - 1) & 1));
      if (lt == 0) trace_ev(P, gt, 0);
      unsigned char* xb = sm + kX + b * 4 * kXT;
      const float* xs = P.x + w.sig * P.ld_x;
      const long long lo = P.lo + w.obase, o0 = w.o0(P), jmin = lo - P.K;
      pend_l = stage_stream(P, xs, lo + o0 + P.K, jmin, lt, keep, xb, xb + kXT);
      pend_t = !w.warm(P) && stage_stream(P, xs, lo + o0 - P.K, jmin, lt, first, xb + 2 * kXT, xb + 3 * kXT);
      asm volatile("cp.async.commit_group;" ::: "memory");
      w = nx;
    }
    if (gt >= 1) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      const int b = static_cast<int>((gt - 1) & 1);
      unsigned char* pb = sm + kX + b * 4 * kXT;
      if (pend_l) finish_lo(pb, pb + kXT, lt);
      if (pend_t) finish_lo(pb + 2 * kXT, pb + 3 * kXT, lt);
      umma::fence_proxy_async();
      umma::mbar_arrive(&M.xfull[b]);
    }
  } else if (warp >= 12) {
    // ================= MMA issuers (warp-uniform control flow, one elected lane issues):
    // warp 12 runs GEMM1 of every tile as soon as its samples are staged; warp 13 runs
    // GEMM2 of every output tile as soon as its chunk states are. All operand addresses
    // are compile-time offsets from one descriptor base per (stage, accumulator buffer).
    const uint64_t dbase = umma::desc_sw128(umma::smem_u32(sm));
    Walk w;
    w.begin(P);
    if (warp == 12) {
      for (long long g = 0; w.valid; ++g, w.advance(P)) {
        const int b = static_cast<int>(g & 1);
        umma::mbar_wait(&M.xfull[b], static_cast<uint32_t>((g >> 1) & 1));
        if (g >= 2) umma::mbar_wait(&M.d1free[b], static_cast<uint32_t>(((g >> 1) - 1) & 1));
        __syncwarp();
        umma::fence_after();
        const bool trail = !w.warm(P);
        if (b == 0)
          gemm1<0>(dbase, tmem, trail);
        else
          gemm1<1>(dbase, tmem, trail);
        umma::commit_elect(&M.g1done[b]);
        if (!trail) umma::commit_elect(&M.xfree[b]);
        if (lane == 0) trace_ev(P, g, 2);
      }
    } else {
      long long u = 0;
      for (long long g = 0; w.valid; ++g, w.advance(P)) {
        if (w.warm(P)) continue;
        const int b2 = static_cast<int>(u & 1);
        umma::mbar_wait(&M.ssfull, static_cast<uint32_t>(u & 1));
        if (lane == 0) trace_ev(P, g, 15);
        if (u >= 2) umma::mbar_wait(&M.d2free[b2], static_cast<uint32_t>(((u >> 1) - 1) & 1));
        __syncwarp();
        umma::fence_after();
        const int sel = static_cast<int>(g & 1) * 2 + b2;
        if (sel == 0)
          gemm2<0, 0>(dbase, tmem, P.cplx);
        else if (sel == 1)
          gemm2<0, 1>(dbase, tmem, P.cplx);
        else if (sel == 2)
          gemm2<1, 0>(dbase, tmem, P.cplx);
        else
          gemm2<1, 1>(dbase, tmem, P.cplx);
        umma::commit_elect(&M.g2done[b2]);
        umma::commit_elect(&M.xfree[g & 1]);
        if (lane == 0) trace_ev(P, g, 5);
        ++u;
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue (non-warm tiles): thread = chunk = TMEM lane
    const int c = tid - 128;
    const uint32_t lrow = static_cast<uint32_t>((warp - 4) * 32) << 16;
    unsigned char* const stg = sm + kStage;
    const int ew = warp - 4;
    const int halves = P.cplx ? 2 : 1;
    const int cw = P.cplx ? 2 : 1;
    Walk w;
    w.begin(P);
    long long u = 0, gt = -1;
    for (; w.valid; w.advance(P)) {
      ++gt;
      if (w.warm(P)) continue;
      const int b2 = static_cast<int>(u & 1);
      umma::mbar_wait(&M.g2done[b2], static_cast<uint32_t>((u >> 1) & 1));
      if (c == 0) trace_ev(P, gt, 6);
      __syncwarp();
      umma::fence_after();
      uint32_t v[64];
      if (halves == 2) {
        umma::tmem_ld32(tmem + lrow + 64 * b2, v);
        umma::tmem_ld32(tmem + lrow + 64 * b2 + 32, v + 32);
      } else {
        umma::tmem_ld32(tmem + lrow + 64 * b2, v);
      }
      umma::tmem_wait_ld();
      umma::fence_before();
      umma::mbar_arrive(&M.d2free[b2]);
      ++u;
      const long long o0 = w.o0(P), cnt = w.cnt;
      float* const orow = P.out + (w.sig * P.ld_out + w.obase) * cw;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h < halves) {
          // row c of the staging area: 8 chunks of 16 B, chunk q at q ^ (c & 7)
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<uint4*>(stg + c * 128 + ((q ^ (c & 7)) << 4)) =
                make_uint4(v[32 * h + 4 * q], v[32 * h + 4 * q + 1], v[32 * h + 4 * q + 2], v[32 * h + 4 * q + 3]);
          bar_epi();
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const int row = ew * 32 + r * 4 + (lane >> 3), q = lane & 7;
            const float4 val = *reinterpret_cast<const float4*>(stg + row * 128 + ((q ^ (row & 7)) << 4));
            const long long pos = o0 + row * 32 + (P.cplx ? 16 * h + 2 * q : 4 * q);
            float* dst = orow + (o0 + row * 32) * cw + 32 * h + 4 * q;
            const int per = P.cplx ? 2 : 4;
            if (P.vec_ok && pos + per <= cnt) {
              __stcs(reinterpret_cast<float4*>(dst), val);
            } else {
              const float e[4] = {val.x, val.y, val.z, val.w};
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if (pos + j / cw < cnt) dst[j] = e[j];
            }
          }
          bar_epi();
        }
      }
      if (c == 0) trace_ev(P, gt, 7);
    }
  } else {
    // ================= chunk-state scan: thread = chunk = TMEM lane
    const float2* zl = reinterpret_cast<const float2*>(sm + kZl);
    const uint32_t lrow = static_cast<uint32_t>(warp * 32) << 16;
    unsigned char* const ss = sm + kSS;
    const int c = tid;
    Walk w;
    w.begin(P);
    long long u = 0;
    for (long long gt = 0; w.valid; ++gt) {
      const int b = static_cast<int>(gt & 1);
      umma::mbar_wait(&M.g1done[b], static_cast<uint32_t>((gt >> 1) & 1));
      if (tid == 0) trace_ev(P, gt, 3);
      if (tid == 96) trace_ev(P, gt, 8);
      __syncwarp();
      umma::fence_after();
      uint32_t a16[16];
      umma::tmem_ld16(tmem + lrow + 128 + 32 * b, a16);
      umma::tmem_wait_ld();
      umma::fence_before();
      umma::mbar_arrive(&M.d1free[b]);
      const bool warm = w.warm(P);
      float2 inc[kMaxOrd];
      if (warm) {
        // only the tile total is needed: sum_l z^{32 (31 - l)} A[l] per warp
#pragma unroll
        for (int p = 0; p < kMaxOrd; ++p) {
          if (p < nord) {
            const float2 a = make_float2(__uint_as_float(a16[2 * p]), __uint_as_float(a16[2 * p + 1]));
            float2 s = cmla(zl[p * 32 + 31 - lane], a, make_float2(0.f, 0.f));
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) {
              s.x += __shfl_xor_sync(0xffffffffu, s.x, d);
              s.y += __shfl_xor_sync(0xffffffffu, s.y, d);
            }
            if (lane == 0) M.wtot[b][warp][p] = s;
          }
        }
      } else {
        // inclusive warp scan over chunks: I[l] = sum_{l' <= l} z^{32 (l - l')} A[l']
        // (steps outer, orders inner: the orders' shuffle chains overlap)
#pragma unroll
        for (int p = 0; p < kMaxOrd; ++p)
          if (p < nord) inc[p] = make_float2(__uint_as_float(a16[2 * p]), __uint_as_float(a16[2 * p + 1]));
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int d = 1 << k;
          float2 t[kMaxOrd];
#pragma unroll
          for (int p = 0; p < kMaxOrd; ++p)
            if (p < nord)
              t[p] = make_float2(__shfl_up_sync(0xffffffffu, inc[p].x, d), __shfl_up_sync(0xffffffffu, inc[p].y, d));
#pragma unroll
          for (int p = 0; p < kMaxOrd; ++p)
            if (p < nord && lane >= d) inc[p] = cmla(P.zs[p][k], t[p], inc[p]);
        }
        if (lane == 31) {
#pragma unroll
          for (int p = 0; p < kMaxOrd; ++p)
            if (p < nord) M.wtot[b][warp][p] = inc[p];
        }
      }
      if (tid == 0) trace_ev(P, gt, 9);
      if (tid == 96) trace_ev(P, gt, 10);
      bar_scan();
      if (tid == 0) trace_ev(P, gt, 11);
      const double2* cyin = M.cy[b];
      if (!warm) {
        // state entering chunk c: S = excl + z^{32 lane} W_warp. Lane p < nord derives
        // W_warp for order p from the fp64 tile carry and the earlier warps' totals.
        float2 Wp = make_float2(0.f, 0.f);
        if (lane < nord) {
          const double2 z = P.z1024[lane];
          double2 Wd = cyin[lane];
          for (int w2 = 0; w2 < warp; ++w2) {
            const float2 t = M.wtot[b][w2][lane];
            Wd = make_double2(fma(z.x, Wd.x, fma(-z.y, Wd.y, static_cast<double>(t.x))),
                              fma(z.x, Wd.y, fma(z.y, Wd.x, static_cast<double>(t.y))));
          }
          Wp = make_float2(static_cast<float>(Wd.x), static_cast<float>(Wd.y));
        }
        float sv[2 * kMaxOrd];
#pragma unroll
        for (int p = 0; p < kMaxOrd; ++p) {
          float2 s = make_float2(0.f, 0.f);
          if (p < nord) {
            const float2 W = make_float2(__shfl_sync(0xffffffffu, Wp.x, p), __shfl_sync(0xffffffffu, Wp.y, p));
            float2 e = make_float2(__shfl_up_sync(0xffffffffu, inc[p].x, 1), __shfl_up_sync(0xffffffffu, inc[p].y, 1));
            if (lane == 0) e = make_float2(0.f, 0.f);
            s = cmla(zl[p * 32 + lane], W, e);
          }
          sv[2 * p] = s.x;
          sv[2 * p + 1] = s.y;
        }
        // the chunk-state operand is free once GEMM2 of the previous tile is done
        if (u >= 1) umma::mbar_wait(&M.g2done[(u - 1) & 1], static_cast<uint32_t>(((u - 1) >> 1) & 1));
        if (tid == 0) trace_ev(P, gt, 12);
        // hi = the raw value (the MMA reads its TF32 head), lo = the remainder
#pragma unroll
        for (int k = 0; k < 2 * kMaxOrd; ++k) {
          *reinterpret_cast<float*>(ss + umma::sw128_off(c, k)) = sv[k];
          *reinterpret_cast<float*>(ss + umma::sw128_off(c, 16 + k)) = tf32_lo(sv[k]);
        }
        umma::fence_proxy_async();
        umma::mbar_arrive(&M.ssfull);
        if (tid == 0) trace_ev(P, gt, 4);
        if (tid == 96) trace_ev(P, gt, 13);
        ++u;
      }
      if (tid < nord) {
        // carry into the next tile (fp64): z^{4096} C + sum_w z^{1024 (3 - w)} T_w
        const int p = tid;
        const double2 z = P.z1024[p], zt = P.zT[p];
        double2 T = make_double2(0.0, 0.0);
        for (int w2 = 0; w2 < 4; ++w2) {
          const float2 t = M.wtot[b][w2][p];
          T = make_double2(fma(z.x, T.x, fma(-z.y, T.y, static_cast<double>(t.x))),
                           fma(z.x, T.y, fma(z.y, T.x, static_cast<double>(t.y))));
        }
        const double2 cy = cyin[p];
        M.cy[b ^ 1][p] = w.last(P) ? make_double2(0.0, 0.0)
                                   : make_double2(fma(zt.x, cy.x, fma(-zt.y, cy.y, T.x)),
                                                  fma(zt.x, cy.y, fma(zt.y, cy.x, T.y)));
      }
      w.advance(P);
    }
  }

  umma::fence_before();
  __syncthreads();
  if (warp == 0) {
    umma::fence_after();
    umma::tmem_free(tmem, 256);
  }
}

}  // namespace tck
