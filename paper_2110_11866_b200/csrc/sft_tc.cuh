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
// Operand placement: the signal tiles and the chunk states are A operands held in TMEM
// (lane = chunk, column = position), so shared memory only feeds the small coefficient
// B operands; GEMM1 rides along GEMM2 as 16 extra N columns (B rows [outputs ;
// aggregates]), and the chunk-state product is a second short MMA chain into the same
// accumulator once the scan has produced the states.
//
// Roles (one persistent CTA per SM, 512 threads):
//   warps 0-7   chunk-state scan (thread = chunk = TMEM lane; warps 0-3 take the first
//               half of the orders, warps 4-7 the rest) -> states into TMEM, then warp 0
//               issues the chunk-state GEMM; warm-up tiles only reduce their aggregates
//               into the fp64 tile carry
//   warps 8-11  epilogue: TMEM -> swizzled staging (accumulator released) -> coalesced
//               16-byte stores
//   warps 12-15 loader: coalesced cp.async into a ring of padded staging rows; each
//               thread then reads its chunk row, splits it (TF32 head / remainder) and
//               tcgen05.st's it; warp 12 then issues the merged GEMM of the tile
// Pipelines (mbarriers): TMEM X operands, chunk states and accumulators double-buffered;
// loader staging ring; tile carry double-buffered.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "sft_tc_launch.h"
#include "umma.cuh"

namespace tck {

struct Misc {
  uint64_t xfree[2], g1done[2], dfree[2], g2done[2];
  uint32_t tmem;
  double2 cy[2][kMaxOrd];      // tile carry (state entering the tile), fp64, by tile parity
  float2 wtot[2][4][kMaxOrd];  // per-warp chunk-aggregate totals (by tile parity)
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
    t = ch == 0 ? P.skip0 : 0;  // skipped constant warm-up tiles (carry in closed form)
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

// fp64 state entering the first processed tile of `item` for order p: the closed-form
// contribution of the skipped constant warm-up tiles (0 when none are skipped)
__device__ __forceinline__ double2 item_carry(const TcParams& P, long long item, int p) {
  if (item >= P.n_items || P.skip0 == 0 || P.boundary == 0) return make_double2(0.0, 0.0);
  const long long sig = item / P.n_chunks;
  if (item - sig * P.n_chunks != 0) return make_double2(0.0, 0.0);
  const double v = static_cast<double>(__ldg(P.x + sig * P.ld_x));
  return make_double2(v * P.g0[p].x, v * P.g0[p].y);
}

// Per-tile event clocks of CTA 0 for tools/tc_trace.py. Compiled in only with
// -DTCK_TRACE=1 (SFTGPU_EXTRA_NVCC_FLAGS): the checks cost issue slots in every role.
#ifndef TCK_TRACE
#define TCK_TRACE 0
#endif
__device__ __forceinline__ void trace_ev(const TcParams& P, long long gt, int ev) {
  if constexpr (TCK_TRACE) {
    if (P.trace && blockIdx.x == 0 && gt < 64) P.trace[gt * 16 + ev] = clock64();
  }
}

__device__ __forceinline__ float tf32_lo(float v) { return v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

__device__ __forceinline__ void cp_async4(uint32_t dst, const float* src, unsigned long long pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "l"(pol)
               : "memory");
}

// bulk L2 prefetch of the samples a tile stream reads (clipped to the signal, 16-B aligned)
__device__ __forceinline__ void prefetch_l2(const float* xs, long long j0, long long n) {
  long long a = j0 < 0 ? 0 : j0, e = j0 + kTile > n ? n : j0 + kTile;
  if (e <= a) return;
  const uintptr_t pa = reinterpret_cast<uintptr_t>(xs + a) & ~uintptr_t(15);
  const uintptr_t pe = (reinterpret_cast<uintptr_t>(xs + e) + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pa), "r"(static_cast<uint32_t>(pe - pa))
               : "memory");
}

// Boundary segments of stage_rows (kept out of line: cold code, small hot loop)
__device__ __noinline__ void stage_rows_edge(const TcParams& P, const float* xs, long long j0, long long jmin,
                                             int lane, float* stg) {
  const long long n = P.n;
  constexpr int kSeg = 32 * kQ;
  if (j0 + kSeg <= jmin || (j0 >= jmin && (j0 >= n || j0 + kSeg <= 0))) {
    float v = 0.f;
    if (j0 + kSeg > jmin && P.boundary != 0) v = __ldg(xs + (j0 >= n ? n - 1 : 0));
    for (int r = 0; r < 32; ++r) stg[r * kStgRow + lane] = v;
    return;
  }
  float v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const long long j = j0 + kQ * r + lane;
    v[r] = __ldg(xs + (j < 0 ? 0 : (j >= n ? n - 1 : j)));
  }
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const long long j = j0 + kQ * r + lane;
    if (j < jmin || (P.boundary == 0 && (j < 0 || j >= n))) v[r] = 0.f;
    stg[r * kStgRow + lane] = v[r];
  }
}

// Stage one stream of this warp's 32 chunk rows: row r = samples j0 + 32 r + [0, 32),
// lane l loads column l (warp-coalesced) into the padded staging rows. Segment classes as
// in K1's stage_stream: inside the signal (cp.async), or a boundary segment (uniform
// boundary value, or straddling an edge / the warm start: per element).
__device__ __forceinline__ void stage_rows(const TcParams& P, const float* xs, long long j0, long long jmin, int lane,
                                           unsigned long long pol, float* stg) {
  constexpr int kSeg = 32 * kQ;
  if (j0 >= jmin && j0 >= 0 && j0 + kSeg <= P.n) {
    const uint32_t s0 = umma::smem_u32(stg) + 4u * static_cast<uint32_t>(lane);
    const float* p = xs + j0 + lane;
#pragma unroll
    for (int r = 0; r < 32; ++r) cp_async4(s0 + r * kStgRow * 4, p + kQ * r, pol);
    return;
  }
  stage_rows_edge(P, xs, j0, jmin, lane, stg);
}

// this thread's chunk row from staging -> TMEM: head columns [col, +32), remainder [col+32, +32)
__device__ __forceinline__ void row_to_tmem(const float* stg, int lane, uint32_t taddr) {
  uint32_t h[32], l[32];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 v = *reinterpret_cast<const float4*>(stg + lane * kStgRow + 4 * j);
    h[4 * j] = __float_as_uint(v.x);
    h[4 * j + 1] = __float_as_uint(v.y);
    h[4 * j + 2] = __float_as_uint(v.z);
    h[4 * j + 3] = __float_as_uint(v.w);
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) l[i] = __float_as_uint(tf32_lo(__uint_as_float(h[i])));
  umma::tmem_st32(taddr, h);
  umma::tmem_st32(taddr + 32, l);
}

__device__ __noinline__ void store_masked(float* dst, float4 val, long long pos, long long cnt, int cw) {
  const float e[4] = {val.x, val.y, val.z, val.w};
  for (int j = 0; j < 4; ++j)
    if (pos + j / cw < cnt) dst[j] = e[j];
}

// named barriers: scan order-sets (1, 2), epilogue (3), loader (4), all scan warps (5)
__device__ __forceinline__ void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ float2 cmla(float2 z, float2 t, float2 a) {  // a + z t
  return make_float2(fmaf(z.x, t.x, fmaf(-z.y, t.y, a.x)), fmaf(z.x, t.y, fmaf(z.y, t.x, a.y)));
}

// ---- MMA chains (warp-uniform; B at compile-time offsets from the descriptor base)
// Merged GEMM1 + GEMM2a of an output tile: D[:, 0:NO+16) = X . [B_out ; B_agg]^T (3xTF32)
template <int K>
__device__ __forceinline__ void merged_k(uint64_t db, uint32_t d, uint32_t x, uint32_t id) {
  constexpr uint32_t ko = 32 * K;
  umma::mma_tf32_ts<kBLh + ko>(d, x + 8 * K, db, id, K > 0);        // xl_h . BL_h
  umma::mma_tf32_ts<kBLh + ko>(d, x + 32 + 8 * K, db, id, 1);       // xl_l . BL_h
  umma::mma_tf32_ts<kBLl + ko>(d, x + 8 * K, db, id, 1);            // xl_h . BL_l
  umma::mma_tf32_ts<kBTh + ko>(d, x + 64 + 8 * K, db, id, 1);       // xt_h . BT_h
  umma::mma_tf32_ts<kBTh + ko>(d, x + 96 + 8 * K, db, id, 1);       // xt_l . BT_h
  umma::mma_tf32_ts<kBTl + ko>(d, x + 64 + 8 * K, db, id, 1);       // xt_h . BT_l
}
// Warm-up tile: aggregates only (lead stream; the trail is before the warm start)
template <int K, uint32_t NO>
__device__ __forceinline__ void warm_k(uint64_t db, uint32_t d, uint32_t x, uint32_t id) {
  constexpr uint32_t ko = 32 * K, ro = NO * 128;
  umma::mma_tf32_ts<kBLh + ro + ko>(d, x + 8 * K, db, id, K > 0);
  umma::mma_tf32_ts<kBLh + ro + ko>(d, x + 32 + 8 * K, db, id, 1);
  umma::mma_tf32_ts<kBLl + ro + ko>(d, x + 8 * K, db, id, 1);
}

template <int NORD>
__global__ void __launch_bounds__(kThreads, 1) sft_tc_kernel(const __grid_constant__ TcParams P) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  Misc& M = *reinterpret_cast<Misc*>(sm + kMisc);
  const int tid = threadIdx.x, lane = tid & 31;
  // warp index as a provably warp-uniform value: role branches become uniform branches
  // and the MMA issuer keeps descriptors on the uniform datapath
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int NO = P.cplx ? 2 * kQ : kQ;  // output columns of the accumulator

  // ---- setup: operand image, barriers, TMEM (512 columns)
  {
    uint4* dst = reinterpret_cast<uint4*>(sm);
    for (int i = tid; i < static_cast<int>(kImage / 16); i += kThreads) dst[i] = __ldg(P.image + i);
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&M.xfree[b], 1);
      umma::mbar_init(&M.g1done[b], 1);
      umma::mbar_init(&M.dfree[b], 128);
      umma::mbar_init(&M.g2done[b], 1);
    }
    umma::mbar_fence_init();
  }
  if (tid < kMaxOrd) M.cy[0][tid] = item_carry(P, blockIdx.x, tid);
  if (warp == 0) umma::tmem_alloc(&M.tmem, 512);
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, M.tmem, 0);  // warp-uniform
  constexpr int nord = NORD;
  const uint64_t dbase = umma::desc_sw128(umma::smem_u32(sm));

  if (warp >= 12) {
    // ================= loader: warp q owns chunk rows [32 q, +32) = TMEM lanes of warp q
    const int q = warp - 12;
    const uint32_t lrow = static_cast<uint32_t>(q * 32) << 16;
    float* const stg = reinterpret_cast<float*>(sm + kLStage + q * kStgWarp);
    unsigned long long keep, first;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(first));
    const uint32_t idm = umma::idesc_tf32(128, NO + 16), ida = umma::idesc_tf32(128, 16);
    auto issue = [&](const Walk& w, int buf) {
      if (w.valid) {
        const float* xs = P.x + w.sig * P.ld_x;
        const long long lo = P.lo + w.obase, o0 = w.o0(P) + 32LL * kQ * q, jmin = lo - P.K;
        float* sb = stg + buf * 2 * 32 * kStgRow;
        stage_rows(P, xs, lo + o0 + P.K, jmin, lane, keep, sb);
        if (!w.warm(P)) stage_rows(P, xs, lo + o0 - P.K, jmin, lane, first, sb + 32 * kStgRow);
        if (lane == 0) {
          Walk nx = w;
          nx.advance(P);
          if (nx.valid) {
            const float* xn = P.x + nx.sig * P.ld_x;
            const long long ln = P.lo + nx.obase, on = nx.o0(P) + 32LL * kQ * q;
            prefetch_l2(xn, ln + on + P.K, P.n);
            if (!nx.warm(P)) prefetch_l2(xn, ln + on - P.K, P.n);
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");  // one group per tile (possibly empty)
    };
    // staging ring of kLoadAhead + 1 tiles: tile gt + kLoadAhead is issued before tile gt
    // is moved into TMEM
    Walk wi, w;
    wi.begin(P);
    w.begin(P);
    for (int k = 0; k < kLoadAhead; ++k) {
      issue(wi, k);
      if (wi.valid) wi.advance(P);
    }
    for (long long gt = 0; w.valid; ++gt) {
      issue(wi, static_cast<int>((gt + kLoadAhead) % (kLoadAhead + 1)));
      if (wi.valid) wi.advance(P);
      asm volatile("cp.async.wait_group %0;" ::"n"(kLoadAhead) : "memory");
      __syncwarp();
      const int b = static_cast<int>(gt & 1);
      if (gt >= 2) umma::mbar_wait(&M.xfree[b], static_cast<uint32_t>(((gt >> 1) - 1) & 1));
      __syncwarp();
      umma::fence_after();
      if (lane == 0) trace_ev(P, gt, 0);
      const float* sb = stg + static_cast<int>(gt % (kLoadAhead + 1)) * 2 * 32 * kStgRow;
      const uint32_t tx = tmem + lrow + kTX + 128 * b;
      const bool warm = w.warm(P);
      row_to_tmem(sb, lane, tx);
      if (!warm) row_to_tmem(sb + 32 * kStgRow, lane, tx + 64);
      umma::tmem_wait_st();
      umma::fence_before();
      bar_named(4, 128);  // all four lane quarters of the tile are in TMEM
      if (lane == 0) trace_ev(P, gt, 1);
      if (q == 0) {
        // merged GEMM (outputs + aggregates; warm tiles: aggregates of the lead stream)
        // into accumulator b once the epilogue / scan have released it
        if (gt >= 2) umma::mbar_wait(&M.dfree[b], static_cast<uint32_t>(((gt >> 1) - 1) & 1));
        __syncwarp();
        umma::fence_after();
        const uint32_t d = tmem + (b ? kTD1 : kTD0), x = tmem + kTX + 128 * b;
        if (!warm) {
          merged_k<0>(dbase, d, x, idm);
          merged_k<1>(dbase, d, x, idm);
          merged_k<2>(dbase, d, x, idm);
          merged_k<3>(dbase, d, x, idm);
        } else if (NO == 64) {
          warm_k<0, 64>(dbase, d + 64, x, ida);
          warm_k<1, 64>(dbase, d + 64, x, ida);
          warm_k<2, 64>(dbase, d + 64, x, ida);
          warm_k<3, 64>(dbase, d + 64, x, ida);
        } else {
          warm_k<0, 32>(dbase, d + 32, x, ida);
          warm_k<1, 32>(dbase, d + 32, x, ida);
          warm_k<2, 32>(dbase, d + 32, x, ida);
          warm_k<3, 32>(dbase, d + 32, x, ida);
        }
        umma::commit_elect(&M.g1done[b]);
        umma::commit_elect(&M.xfree[b]);
        if (lane == 0) trace_ev(P, gt, 2);
      }
      __syncwarp();  // every lane has read its row before the ring slot is refilled
      w.advance(P);
    }
  } else if (warp >= 8) {
    // ================= epilogue (non-warm tiles): thread = chunk = TMEM lane
    const int c = tid - 256;
    const int ew = warp - 8;
    const uint32_t lrow = static_cast<uint32_t>(ew * 32) << 16;
    unsigned char* const stgo = sm + kStage;
    const int halves = P.cplx ? 2 : 1;
    const int cw = P.cplx ? 2 : 1;
    Walk w;
    w.begin(P);
    long long u = 0;
    for (long long gt = 0; w.valid; w.advance(P), ++gt) {
      if (w.warm(P)) continue;
      const int s = static_cast<int>(u & 1);
      umma::mbar_wait(&M.g2done[s], static_cast<uint32_t>((u >> 1) & 1));
      if (c == 0) trace_ev(P, gt, 6);
      __syncwarp();
      umma::fence_after();
      const uint32_t dcol = (gt & 1) ? kTD1 : kTD0;
      // the previous tile's TMA stores must have read the staging area
      if (c == 0 && P.use_tma) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      bar_named(3, 128);
      // accumulator -> staging (row c: 8 chunks of 16 B per half, chunk q at q ^ (c & 7):
      // the TMA SWIZZLE_128B layout of a [128 rows][32 floats] box)
      for (int h = 0; h < halves; ++h) {
        uint32_t v[32];
        umma::tmem_ld32(tmem + lrow + dcol + 32 * h, v);
        umma::tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<uint4*>(stgo + h * 16384 + c * 128 + ((q ^ (c & 7)) << 4)) =
              make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
      umma::fence_before();
      umma::mbar_arrive(&M.dfree[gt & 1]);
      if (c == 0) trace_ev(P, gt, 14);
      ++u;
      const long long o0 = w.o0(P), cnt = w.cnt;
      if (P.use_tma) {
        // one thread hands the tile to the TMA engine: 128 rows x 32 floats per half
        umma::fence_proxy_async();
        bar_named(3, 128);
        if (c == 0) {
          const int row0 = static_cast<int>((w.obase + o0) / kQ), sg = static_cast<int>(w.sig);
          for (int h = 0; h < halves; ++h) {
            const uint32_t src = umma::smem_u32(stgo + h * 16384);
            if (P.cplx)
              asm volatile(
                  "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                      reinterpret_cast<uint64_t>(&P.out_map)),
                  "r"(0), "r"(h), "r"(row0), "r"(sg), "r"(src)
                  : "memory");
            else
              asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                               reinterpret_cast<uint64_t>(&P.out_map)),
                           "r"(0), "r"(row0), "r"(sg), "r"(src)
                           : "memory");
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (c == 0) trace_ev(P, gt, 7);
        continue;
      }
      bar_named(3, 128);
      float* const orow = P.out + (w.sig * P.ld_out + w.obase) * cw;
      for (int h = 0; h < halves; ++h) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int row = ew * 32 + r * 4 + (lane >> 3), q = lane & 7;
          const float4 val = *reinterpret_cast<const float4*>(stgo + h * 16384 + row * 128 + ((q ^ (row & 7)) << 4));
          const long long pos = o0 + row * 32 + (P.cplx ? 16 * h + 2 * q : 4 * q);
          float* dst = orow + (o0 + row * 32) * cw + 32 * h + 4 * q;
          if (P.vec_ok && pos + (P.cplx ? 2 : 4) <= cnt)
            __stcs(reinterpret_cast<float4*>(dst), val);
          else
            store_masked(dst, val, pos, cnt, cw);
        }
      }
      if (c == 0) trace_ev(P, gt, 7);
    }
    if (c == 0 && P.use_tma) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else {
    // ================= chunk-state scan: thread = chunk = TMEM lane; order set `os`
    constexpr int hA = 4;  // set 0: orders [0, 4) (state columns 0-7), set 1: [4, 8) (8-15)
    const int os = warp >> 2;
    const int sw = warp & 3;   // lane quarter
    const int p0 = os ? hA : 0;
    const int st = tid & 127;
    const float2* zl = reinterpret_cast<const float2*>(sm + kZl);
    const uint32_t lrow = static_cast<uint32_t>(sw * 32) << 16;
    Walk w;
    w.begin(P);
    long long u = 0;
    for (long long gt = 0; w.valid; ++gt) {
      const int b = static_cast<int>(gt & 1);
      umma::mbar_wait(&M.g1done[b], static_cast<uint32_t>((gt >> 1) & 1));
      if (tid == 0) trace_ev(P, gt, 3);
      __syncwarp();
      umma::fence_after();
      const bool warm = w.warm(P);
      uint32_t a8[8];
      umma::tmem_ld8(tmem + lrow + (b ? kTD1 : kTD0) + NO + 2 * p0, a8);  // this set's orders
      umma::tmem_wait_ld();
      if (tid == 0) trace_ev(P, gt, 8);
      if (warm) {
        // nothing else reads this accumulator: hand it back once both sets have read it
        umma::fence_before();
        bar_named(5, 256);
        if (warp == 0) {
          __syncwarp();
          if (lane == 0) umma::mbar_arrive_cnt(&M.dfree[b], 128);
        }
      }
      float2 inc[4];
      if (warm) {
        // only the tile total is needed: sum_l z^{32 (31 - l)} A[l] per warp
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int p = p0 + j;
          if (j < hA && p < nord) {
            const float2 a = make_float2(__uint_as_float(a8[2 * j]), __uint_as_float(a8[2 * j + 1]));
            float2 s = cmla(zl[p * 32 + 31 - lane], a, make_float2(0.f, 0.f));
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) {
              s.x += __shfl_xor_sync(0xffffffffu, s.x, d);
              s.y += __shfl_xor_sync(0xffffffffu, s.y, d);
            }
            if (lane == 0) M.wtot[b][sw][p] = s;
          }
        }
      } else {
        // inclusive warp scan over chunks: I[l] = sum_{l' <= l} z^{32 (l - l')} A[l']
#pragma unroll
        for (int j = 0; j < 4; ++j) inc[j] = make_float2(__uint_as_float(a8[2 * j]), __uint_as_float(a8[2 * j + 1]));
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int d = 1 << k;
          float2 t[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j < hA && p0 + j < nord)
              t[j] = make_float2(__shfl_up_sync(0xffffffffu, inc[j].x, d), __shfl_up_sync(0xffffffffu, inc[j].y, d));
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j < hA && p0 + j < nord && lane >= d) inc[j] = cmla(P.zs[p0 + j][k], t[j], inc[j]);
        }
        if (lane == 31) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j < hA && p0 + j < nord) M.wtot[b][sw][p0 + j] = inc[j];
        }
      }
      if (tid == 0) trace_ev(P, gt, 9);
      bar_named(1 + os, 128);
      if (tid == 0) trace_ev(P, gt, 11);
      const double2* cyin = M.cy[b];
      if (!warm) {
        // state entering chunk c: S = excl + z^{32 lane} W_warp. Lane j < set size derives
        // W_warp for order p0 + j from the fp64 tile carry and the earlier warps' totals.
        float2 Wp = make_float2(0.f, 0.f);
        if (lane < hA && p0 + lane < nord) {
          const int p = p0 + lane;
          const double2 z = P.z1024[p];
          double2 Wd = cyin[p];
          for (int w2 = 0; w2 < sw; ++w2) {
            const float2 t = M.wtot[b][w2][p];
            Wd = make_double2(fma(z.x, Wd.x, fma(-z.y, Wd.y, static_cast<double>(t.x))),
                              fma(z.x, Wd.y, fma(z.y, Wd.x, static_cast<double>(t.y))));
          }
          Wp = make_float2(static_cast<float>(Wd.x), static_cast<float>(Wd.y));
        }
        uint32_t sh[8], sl[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 s = make_float2(0.f, 0.f);
          if (j < hA && p0 + j < nord) {
            const float2 W = make_float2(__shfl_sync(0xffffffffu, Wp.x, j), __shfl_sync(0xffffffffu, Wp.y, j));
            float2 e = make_float2(__shfl_up_sync(0xffffffffu, inc[j].x, 1), __shfl_up_sync(0xffffffffu, inc[j].y, 1));
            if (lane == 0) e = make_float2(0.f, 0.f);
            s = cmla(zl[(p0 + j) * 32 + lane], W, e);
          }
          // head = the raw value (the MMA reads its TF32 head), remainder separately
          sh[2 * j] = __float_as_uint(s.x);
          sh[2 * j + 1] = __float_as_uint(s.y);
          sl[2 * j] = __float_as_uint(tf32_lo(s.x));
          sl[2 * j + 1] = __float_as_uint(tf32_lo(s.y));
        }
        if (tid == 0) trace_ev(P, gt, 12);
        // this state buffer is free once the chunk-state GEMM of output tile u-2 is done
        const int s = static_cast<int>(u & 1);
        if (u >= 2) umma::mbar_wait(&M.g2done[s], static_cast<uint32_t>(((u >> 1) - 1) & 1));
        __syncwarp();
        umma::fence_after();
        const uint32_t ts = tmem + lrow + kTSS + 32 * s + 2 * p0;
        umma::tmem_st8(ts, sh);
        umma::tmem_st8(ts + 16, sl);
        umma::tmem_wait_st();
        umma::fence_before();
        bar_named(5, 256);  // both order sets' states are in TMEM
        if (tid == 0) trace_ev(P, gt, 4);
        if (warp == 0) {
          // chunk-state GEMM: D[:, 0:NO) += S . C^T (3xTF32)
          umma::fence_after();
          const uint32_t d = tmem + (b ? kTD1 : kTD0), a = tmem + kTSS + 32 * s;
          const uint32_t ids = umma::idesc_tf32(128, NO);
          umma::mma_tf32_ts<kBC>(d, a, dbase, ids, 1);  // S_h . C_h
          umma::mma_tf32_ts<kBC + 32>(d, a + 8, dbase, ids, 1);
          umma::mma_tf32_ts<kBC>(d, a + 16, dbase, ids, 1);  // S_l . C_h
          umma::mma_tf32_ts<kBC + 32>(d, a + 24, dbase, ids, 1);
          umma::mma_tf32_ts<kBC + 64>(d, a, dbase, ids, 1);  // S_h . C_l
          umma::mma_tf32_ts<kBC + 96>(d, a + 8, dbase, ids, 1);
          umma::commit_elect(&M.g2done[s]);
          if (lane == 0) trace_ev(P, gt, 5);
        }
        ++u;
      }
      if (st < hA && p0 + st < nord && sw == 0) {
        // carry into the next tile (fp64): z^{4096} C + sum_w z^{1024 (3 - w)} T_w
        const int p = p0 + st;
        const double2 z = P.z1024[p], zt = P.zT[p];
        double2 T = make_double2(0.0, 0.0);
        for (int w2 = 0; w2 < 4; ++w2) {
          const float2 t = M.wtot[b][w2][p];
          T = make_double2(fma(z.x, T.x, fma(-z.y, T.y, static_cast<double>(t.x))),
                           fma(z.x, T.y, fma(z.y, T.x, static_cast<double>(t.y))));
        }
        const double2 cy = cyin[p];
        M.cy[b ^ 1][p] = w.last(P) ? item_carry(P, w.item + gridDim.x, p)
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
    umma::tmem_free(tmem, 512);
  }
}

}  // namespace tck
