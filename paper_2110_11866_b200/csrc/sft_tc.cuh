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
//   warps 12-15 loader: one thread stages each tile's lead and trail streams with two TMA
//               boxes (SW128 rows of 32 samples) into a 3-slot ring; every thread then
//               reads its chunk row (shifted by the plan's sub-16-byte stream offset),
//               splits it (TF32 head / remainder) and tcgen05.st's it; warp 12 then
//               issues the merged GEMM of the tile
// Pipelines (mbarriers): TMEM X operands, chunk states and accumulators double-buffered;
// loader staging ring; tile carry double-buffered.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "sft_tc_launch.h"
#include "umma.cuh"

namespace tck {

struct Misc {
  uint64_t xfull[2], xfree[2], g1done[2], dfree[2], sready[2], g2done[2];
  uint64_t fullL[kLoadAhead + 1], fullT[kTrailAhead + 1];  // loader ring slots landed (lead, trail)
  uint64_t drain, scandone, imgbar;  // scale switch: MMAs done, scans done, new image landed
  uint32_t tmem;
  double2 cy[2][kMaxOrd];  // tile carry (state entering the tile), fp64, by tile parity
  float2 tot[kMaxOrd];     // tile total of the order's chunk scan (lane 31 of phase 2)
};
static_assert(sizeof(Misc) <= 512, "Misc region");

// Work of one CTA: a contiguous range [c, cend) of the global chunk sequence. Units
// u = scale * nsig + sig are cut into fixed chunks (TcGeom); chunks are ordered scale-major
// and partitioned over the CTAs by cost (warm-up + output tiles), so a CTA meets few
// scales. A chunk (segment) is its warm-up tiles (from its own warm start, 2K positions
// before its first output; leading constant ones of a unit's first chunk skipped)
// followed by its output tiles.
__device__ __forceinline__ int scale_of_chunk(const TcParams& P, int c) {
  int lo = 0, hi = P.n_scales - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (P.geo[mid].cbase <= c) lo = mid; else hi = mid - 1;
  }
  return lo;
}
// tiles of all chunks before chunk c
__device__ __forceinline__ int chunk_prefix(const TcParams& P, int c) {
  if (c >= P.total_chunks) return P.total_cost;
  const int s = scale_of_chunk(P, c);
  const TcGeom& G = P.geo[s];
  const int rem = c - G.cbase, u = rem / G.nc, k = rem - u * G.nc;
  const int unit_cost = P.tiles_unit + G.nc * G.warm - G.skip0;
  return G.wbase + u * unit_cost + k * (G.L + G.warm) - (k > 0 ? G.skip0 : 0);
}
// first chunk of CTA j: the smallest c with chunk_prefix(c) >= j * total_cost / grid
__device__ __forceinline__ int cta_first_chunk(const TcParams& P, int j) {
  const int target = static_cast<int>((static_cast<long long>(j) * P.total_cost) / gridDim.x);
  int lo = 0, hi = P.total_chunks;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (chunk_prefix(P, mid) >= target) hi = mid; else lo = mid + 1;
  }
  return lo;
}

struct Walk {
  int c, cend;       // current chunk; range end
  int sig, scale;
  int l0, nout;      // first output tile of the chunk within its unit; output tiles
  int W, t;          // warm-up tiles of the chunk's scale; tile cursor
  bool valid;
  __device__ void setup(const TcParams& P) {
    valid = c < cend;
    if (!valid) return;
    scale = scale_of_chunk(P, c);
    const TcGeom& G = P.geo[scale];
    const int rem = c - G.cbase, u = rem / G.nc, k = rem - u * G.nc;
    sig = u;
    l0 = k * G.L;
    const int room = P.tiles_unit - l0;
    nout = G.L < room ? G.L : room;
    W = G.warm;
    t = l0 == 0 ? G.skip0 : 0;  // skipped constant warm-up tiles
  }
  __device__ void begin(const TcParams& P) {
    c = cta_first_chunk(P, blockIdx.x);
    cend = cta_first_chunk(P, blockIdx.x + 1);
    setup(P);
  }
  __device__ void advance(const TcParams& P) {
    if (++t < W + nout) return;
    ++c;
    setup(P);
  }
  __device__ int unit(const TcParams& P) const { return scale * P.nsig + sig; }
  __device__ bool warm(const TcParams&) const { return t < W; }
  __device__ long long obase() const { return static_cast<long long>(l0) * kTile; }
  __device__ long long o0(const TcParams&) const { return static_cast<long long>(t - W) * kTile; }
  __device__ long long cnt(const TcParams& P) const {
    const long long cc = P.count - obase(), e = static_cast<long long>(nout) * kTile;
    return cc < e ? cc : e;
  }
  __device__ bool last(const TcParams&) const { return t + 1 == W + nout; }
};

// fp64 state entering the first processed tile of segment w for order p: the closed-form
// contribution of the skipped constant warm-up tiles (0 when none are skipped)
__device__ __forceinline__ const unsigned char* scale_image(const TcParams& P, int s) {
  return reinterpret_cast<const unsigned char*>(
      __ldg(reinterpret_cast<const unsigned long long*>(&P.scales[s].image)));
}

__device__ __forceinline__ double2 seg_carry(const TcParams& P, const Walk& w, int p) {
  if (!w.valid || w.l0 != 0 || P.boundary == 0) return make_double2(0.0, 0.0);
  if (P.geo[w.scale].skip0 == 0) return make_double2(0.0, 0.0);
  const TcScale* S = P.scales + w.scale;
  const double v = static_cast<double>(__ldg(P.x + w.sig * P.ld_x));
  const double2 g0 = __ldg(&S->g0[p]);
  return make_double2(v * g0.x, v * g0.y);
}

// Per-tile event clocks of CTA 0 for tools/tc_trace.py. Compiled in only with
// -DTCK_TRACE=1 (SFTGPU_EXTRA_NVCC_FLAGS): the checks cost issue slots in every role.
#ifndef TCK_TRACE
#define TCK_TRACE 0
#endif
#ifndef TCK_SCANPROBE
#define TCK_SCANPROBE 0
#endif
__device__ __forceinline__ void trace_ev(const TcParams& P, long long gt, int ev) {
  if constexpr (TCK_TRACE) {
    if (P.trace && blockIdx.x == 0 && gt < 64) P.trace[gt * 16 + ev] = clock64();
  }
}

__device__ __forceinline__ float tf32_lo(float v) { return v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

// 4-byte cp.async (zero-filled when `zero`: nothing is read) and 16-byte cp.async
__device__ __forceinline__ void cp_async4(uint32_t dst, const float* src, bool zero) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(zero ? 0 : 4) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// the mbarrier counts one arrival once all of this thread's earlier cp.async have landed
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(umma::smem_u32(bar)) : "memory");
}

// How a tile stream is staged (uniform over the loader threads; j0 = its first sample used,
// a = j0 rounded down to 16 bytes):
//  - kTma: the lead stream of an interior segment, one TMA box (the TMA engine carries
//    only lead boxes and output stores: it moves ~32 B/clk per SM, tools/tma_lat.cu);
//  - kCp: an interior trail segment (an L2 hit), 16-byte cp.async;
//  - kZero / kFirst / kLast: one value everywhere (before the warm start, or the boundary
//    value outside [0, n)): the reader writes it to TMEM directly;
//  - kMixed: segments that straddle an edge or the warm start, or an input that is not
//    16-byte aligned: per sample.
enum StreamKind { kTma = 0, kCp = 1, kZero = 2, kFirst = 3, kLast = 4, kMixed = 5 };
__device__ __forceinline__ int stream_kind(const TcParams& P, long long a, long long j0, long long jmin, bool lead) {
  if (P.use_tma_in && a >= 0 && a >= jmin && a + kBoxRows * 32 <= P.n) {
    if ((lead || TCK_TRAIL_TMA) && (a >> 5) + kBoxRows <= P.in_rows) return kTma;
    return kCp;
  }
  const long long j1 = j0 + kTile;
  if (j1 <= jmin) return kZero;
  if (j0 >= jmin && j1 <= 0) return P.boundary != 0 ? kFirst : kZero;
  if (j0 >= jmin && j0 >= P.n) return P.boundary != 0 ? kLast : kZero;
  return kMixed;
}
constexpr uint32_t kValOff = kBoxBytes;  // per-stream words after the rows: x[0], x[n - 1]

// A non-TMA stream of a tile, staged by the 128 loader threads t with cp.async only, so
// that no thread waits on a global load here; the caller then arrives on the slot's
// mbarrier with cp.async.mbarrier.arrive (completion tracked by the barrier):
//  - kCp: the 129 SW128 rows, 16-byte copies;
//  - kFirst / kLast / kMixed: thread 0 copies the boundary values x[0], x[n - 1] to the
//    words at kValOff; kMixed also copies its in-signal samples (flat sample f = 32 rho + i
//    of the slot is x[a + f]), 4-byte copies; fill_mixed stores the rest once they have
//    landed: no copy ever reads a clamped address, which would serialise thousands of
//    copies on one line.
__device__ __forceinline__ void stage_stream(const TcParams& P, const float* xs, long long a, long long jmin, int kind,
                                             int t, unsigned char* slot) {
  const uint32_t s0 = umma::smem_u32(slot);
  if (kind == kCp) {
    for (int i = t; i < static_cast<int>(kBoxRows * 8); i += 128) {
      const int row = i >> 3, pc = i & 7;
      cp_async16(s0 + row * 128 + ((pc ^ (row & 7)) << 4), xs + a + 4 * i);
    }
    return;
  }
  if (kind == kZero) return;
  const long long n = P.n;
  if (t == 0) {
    cp_async4(s0 + kValOff, xs, false);
    cp_async4(s0 + kValOff + 4, xs + n - 1, false);
  }
  if (kind != kMixed) return;
  const long long lo = (jmin > 0 ? jmin : 0) - a, hi = n - a;
  const int f0 = static_cast<int>(lo < 0 ? 0 : lo);
  const int f1 = static_cast<int>(hi > kBoxRows * 32 ? kBoxRows * 32 : (hi < 0 ? 0 : hi));
  for (int f = f0 + t; f < f1; f += 128)
    cp_async4(s0 + umma::sw128_off(static_cast<uint32_t>(f >> 5), static_cast<uint32_t>(f & 31)), xs + a + f, false);
}

// a uniform stream row: the same value in every TMEM column (head and remainder)
__device__ __forceinline__ void uniform_to_tmem(float v, uint32_t taddr) {
  uint32_t h[16], l[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    h[i] = __float_as_uint(v);
    l[i] = __float_as_uint(tf32_lo(v));
  }
  umma::tmem_st16(taddr, h);
  umma::tmem_st16(taddr + 16, h);
  umma::tmem_st16(taddr + 32, l);
  umma::tmem_st16(taddr + 48, l);
}

// Chunk row c of a staged stream, R samples past its box start (flat samples
// 32 c + R + [0, 32)), split into the TF32 head (the raw value: the MMA reads its head)
// and the fp32 remainder -> TMEM columns [0, 32) head and [32, 64) remainder of taddr.
// SW128 rows make the 16-byte row reads of 8 consecutive threads conflict-free.
template <int R>
__device__ __forceinline__ void row_to_tmem_r(const unsigned char* slot, int c, uint32_t taddr) {
#pragma unroll
  for (int qq = 0; qq < 4; ++qq) {  // quarters of 8 columns keep the live registers low
    float f[12];
#pragma unroll
    for (int k = 0; k < (R ? 3 : 2); ++k) {
      const int p = 2 * qq + k, row = c + (p >> 3), pc = p & 7;
      const float4 v = *reinterpret_cast<const float4*>(slot + row * 128 + ((pc ^ (row & 7)) << 4));
      f[4 * k] = v.x;
      f[4 * k + 1] = v.y;
      f[4 * k + 2] = v.z;
      f[4 * k + 3] = v.w;
    }
    uint32_t h[8], l[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float v = f[R + i];
      h[i] = __float_as_uint(v);
      l[i] = __float_as_uint(tf32_lo(v));
    }
    umma::tmem_st8(taddr + 8 * qq, h);
    umma::tmem_st8(taddr + 32 + 8 * qq, l);
  }
}
__device__ __forceinline__ void row_to_tmem(const unsigned char* slot, int r, int c, uint32_t taddr) {
  switch (r) {  // plan-uniform
    case 0: row_to_tmem_r<0>(slot, c, taddr); break;
    case 1: row_to_tmem_r<1>(slot, c, taddr); break;
    case 2: row_to_tmem_r<2>(slot, c, taddr); break;
    default: row_to_tmem_r<3>(slot, c, taddr); break;
  }
}
// kMixed stream staged from a: once its in-signal samples have landed, the loader
// threads t store the rest of the slot (zeros before the warm start, the boundary policy
// outside [0, n)) so that the regular row reader applies. Cold path, out of line: the
// slot comes in as a shared-window address (a generic pointer would make every store a
// generic one).
__device__ __noinline__ void fill_mixed(long long n, int boundary, uint32_t slot, int t, long long a, long long jmin) {
  auto clip = [](long long v) {
    return static_cast<int>(v < 0 ? 0 : (v > kBoxRows * 32 ? kBoxRows * 32 : v));
  };
  const int fj = clip(jmin - a), f0 = clip(-a), fn = clip(n - a);
  float v0 = 0.f, vn = 0.f;
  if (boundary != 0) {
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v0) : "r"(slot + kValOff));
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(vn) : "r"(slot + kValOff + 4));
  }
  auto put = [&](int f, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(slot + umma::sw128_off(static_cast<uint32_t>(f >> 5),
                                                                       static_cast<uint32_t>(f & 31))),
                 "f"(v)
                 : "memory");
  };
  const int fz = fj > f0 ? fj : f0;  // [0, fj) zeros (warm start), then [fj, f0) x[0]
  for (int f = t; f < fz; f += 128) put(f, f < fj ? 0.f : v0);
  for (int f = fn + t; f < static_cast<int>(kBoxRows * 32); f += 128) put(f, vn);
}

__device__ __noinline__ void store_masked(float* dst, float4 val, long long pos, long long cnt, int cw) {
  const float e[4] = {val.x, val.y, val.z, val.w};
  for (int j = 0; j < 4; ++j)
    if (pos + j / cw < cnt) dst[j] = e[j];
}

// named barriers: epilogue (3), lead loaders (4), scan warps (5), trail loaders (6)
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
// timing probe (dbg 32): the hi . hi products only (wrong results)
template <int K>
__device__ __forceinline__ void merged_hh(uint64_t db, uint32_t d, uint32_t x, uint32_t id) {
  constexpr uint32_t ko = 32 * K;
  umma::mma_tf32_ts<kBLh + ko>(d, x + 8 * K, db, id, K > 0);
  umma::mma_tf32_ts<kBTh + ko>(d, x + 64 + 8 * K, db, id, 1);
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
  // 1024-byte aligned base, derived by pointer arithmetic on the shared array so that the
  // compiler keeps every access in the shared window (LDS/STS, not generic LD/ST)
  unsigned char* sm = smraw + ((1024u - (umma::smem_u32(smraw) & 1023u)) & 1023u);
  Misc& M = *reinterpret_cast<Misc*>(sm + kMisc);
  const int tid = threadIdx.x, lane = tid & 31;
  // warp index as a provably warp-uniform value: role branches become uniform branches
  // and the MMA issuer keeps descriptors on the uniform datapath
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int NO = P.cplx ? 2 * kQ : kQ;  // output columns of the accumulator

  // ---- setup: operand image, barriers, TMEM (512 columns)
  Walk w0;  // this CTA's first segment: its scale's operand image is loaded first
  w0.begin(P);
  if (!w0.valid) return;
  {
    uint4* dst = reinterpret_cast<uint4*>(sm);
    const uint4* src = reinterpret_cast<const uint4*>(scale_image(P, w0.scale));
    for (int i = tid; i < static_cast<int>(kImage / 16); i += kThreads) dst[i] = __ldg(src + i);
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&M.xfull[b], 256);  // both stream groups
      umma::mbar_init(&M.xfree[b], 1);
      umma::mbar_init(&M.g1done[b], 1);
      umma::mbar_init(&M.dfree[b], 128);
      umma::mbar_init(&M.sready[b], 256);
      umma::mbar_init(&M.g2done[b], 1);
    }
    umma::mbar_init(&M.drain, 1);
    umma::mbar_init(&M.scandone, 256);
    umma::mbar_init(&M.imgbar, 1);
    for (int k = 0; k <= kLoadAhead; ++k) umma::mbar_init(&M.fullL[k], 129);  // TMA issuer + 128 cp.async arrivals
    for (int k = 0; k <= kTrailAhead; ++k) umma::mbar_init(&M.fullT[k], TCK_TRAIL_TMA ? 129 : 128);
    umma::mbar_fence_init();
  }
  __syncthreads();  // image (g0) in shared memory
  if (tid < kMaxOrd) M.cy[0][tid] = seg_carry(P, w0, tid);
  if (warp == 0) umma::tmem_alloc(&M.tmem, 512);
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, M.tmem, 0);  // warp-uniform
  constexpr int nord = NORD;

  if (warp == 20) {
    // ================= MMA issuer: merged GEMM of tile gt, then the chunk-state GEMM of
    // the previous output tile (issued after it so that it overlaps that tile's scan)
    const uint64_t dbase = umma::desc_sw128(umma::smem_u32(sm));
    const uint32_t idm = umma::idesc_tf32(128, NO + 16), ida = umma::idesc_tf32(128, 16);
    const uint32_t ids = umma::idesc_tf32(128, NO);
    long long u = 0;       // output tiles whose state GEMM has been issued
    int pend = -1;         // accumulator of the output tile whose state GEMM is pending
    auto state_gemm = [&]() {
      const int s = static_cast<int>(u & 1);
      umma::mbar_wait(&M.sready[s], static_cast<uint32_t>((u >> 1) & 1));
      umma::fence_after();
      const uint32_t d = tmem + (pend ? kTD1 : kTD0), a = tmem + kTSS + 32 * s;
      umma::mma_tf32_ts<kBC>(d, a, dbase, ids, 1);  // S_h . C_h
      umma::mma_tf32_ts<kBC + 32>(d, a + 8, dbase, ids, 1);
      umma::mma_tf32_ts<kBC>(d, a + 16, dbase, ids, 1);  // S_l . C_h
      umma::mma_tf32_ts<kBC + 32>(d, a + 24, dbase, ids, 1);
      umma::mma_tf32_ts<kBC + 64>(d, a, dbase, ids, 1);  // S_h . C_l
      umma::mma_tf32_ts<kBC + 96>(d, a + 8, dbase, ids, 1);
      umma::commit_elect(&M.g2done[s]);
      ++u;
      pend = -1;
    };
    Walk w;
    w.begin(P);
    int cur = w.scale, sw = 0;  // scale whose operand image is in shared memory; switches
    for (long long gt = 0; w.valid; ++gt) {
      const int b = static_cast<int>(gt & 1);
      const bool warm = w.warm(P);
      if (w.scale != cur) {
        // scale switch: every MMA and every scan of the old scale must be done with the
        // image before the new one is copied over it (at most a few per CTA)
        if (pend >= 0) state_gemm();
        umma::commit_elect(&M.drain);
        umma::mbar_wait(&M.drain, static_cast<uint32_t>(sw & 1));
        umma::mbar_wait(&M.scandone, static_cast<uint32_t>(sw & 1));
        if (lane == 0) {
          umma::mbar_arrive_tx(&M.imgbar, kImage);
          const unsigned char* src = scale_image(P, w.scale);
          for (uint32_t o = 0; o < kImage; o += 16384)
            umma::bulk_g2s(umma::smem_u32(sm) + o, src + o, kImage - o < 16384 ? kImage - o : 16384, &M.imgbar);
        }
        __syncwarp();
        umma::mbar_wait(&M.imgbar, static_cast<uint32_t>(sw & 1));
        cur = w.scale;
        ++sw;
      }
      const uint32_t xph = static_cast<uint32_t>((gt >> 1) & 1), dph = static_cast<uint32_t>(((gt >> 1) - 1) & 1);
      if (pend >= 0) {
        // the previous output tile's state GEMM goes first if its states are ready before
        // this tile's operands (it gates that tile's epilogue and accumulator release)
        const int s = static_cast<int>(u & 1);
        const uint32_t sph = static_cast<uint32_t>((u >> 1) & 1);
        bool xok = false;
        for (;;) {
          if (umma::mbar_test(&M.sready[s], sph)) {
            state_gemm();
            if (lane == 0) trace_ev(P, gt - 1, 5);
            break;
          }
          if (!xok) xok = umma::mbar_test(&M.xfull[b], xph) && (gt < 2 || umma::mbar_test(&M.dfree[b], dph));
          if (xok) break;
        }
      }
      umma::mbar_wait(&M.xfull[b], xph);
      if (gt >= 2) umma::mbar_wait(&M.dfree[b], dph);
      umma::fence_after();
      if (lane == 0) trace_ev(P, gt, 1);
      const uint32_t d = tmem + (b ? kTD1 : kTD0), x = tmem + kTX + 128 * b;
      if (!warm) {
        // the whole merged GEMM goes in first; the pending state GEMM follows it (below).
        // Slotting the state GEMM in between k-steps as soon as its states were ready
        // measured 2-4% slower (configs 4 and 5, same box): it delays this tile's
        // aggregates, which start the next scan
        if (P.dbg & 32) {
          merged_hh<0>(dbase, d, x, idm);
          merged_hh<1>(dbase, d, x, idm);
          merged_hh<2>(dbase, d, x, idm);
          merged_hh<3>(dbase, d, x, idm);
        } else {
          merged_k<0>(dbase, d, x, idm);
          merged_k<1>(dbase, d, x, idm);
          merged_k<2>(dbase, d, x, idm);
          merged_k<3>(dbase, d, x, idm);
        }
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
      if (pend >= 0) {
        state_gemm();
        if (lane == 0) trace_ev(P, gt - 1, 5);
      }
      if (!warm) pend = b;
      w.advance(P);
    }
    if (pend >= 0) state_gemm();
  } else if (warp >= 12) {
    // ================= loader: two groups of four warps, one per stream (warps 12-15 the
    // lead, 16-19 the trail); in each, thread t = chunk row t = TMEM lane t (warp w: lanes
    // [32 (w % 4), +32)). Each group stages its stream `ahead` tiles ahead into its ring
    // (TMA boxes inside the signal, boundary segments by cp.async), then moves its rows into
    // the X operand in TMEM.
    const bool lead = warp < 16;
    const int t = tid - (lead ? 384 : 512);
    const uint32_t lrow = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int bar_id = lead ? 4 : 6;
    unsigned char* const ring = sm + (lead ? kLStage : kTrail);
    const uint32_t stride = lead ? kLeadBytes : kTrailBytes;
    uint64_t* const full = lead ? M.fullL : M.fullT;
    // lead lines are read again 2K positions later as the trail, which is their last use
    unsigned long long keep;
    if (lead)
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    else
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(keep));
    if (P.dbg & 2) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(keep));
    const int ahead = lead ? kLoadAhead : kTrailAhead;
    // this group's stream of a tile: x[n + K] (lead) or x[n - K] (trail) from n = lo + o0,
    // its start rounded down to 16 bytes (r samples before the first one used), its kind
    auto stream = [&](const Walk& w, long long& a, long long& jmin, int& r) {
      const TcGeom& G = P.geo[w.scale];
      const int K = G.K;
      r = lead ? G.rl : G.rt;
      const long long lo = G.lo + w.obase(), o0 = w.o0(P);
      jmin = lo - K;
      a = lo + o0 + (lead ? K : -K) - r;
      if (!lead && w.warm(P)) return static_cast<int>(kZero);  // warm tiles: no trail operand
      return stream_kind(P, a, a + r, jmin, lead);
    };
    // stage tile w into ring slot `slot`: a box by TMA (one thread, transaction bytes on
    // full[slot]), everything else by cp.async from the group's 128 threads, each of which
    // then arrives on the slot's barrier once its copies have landed
    auto issue = [&](const Walk& w, int slot, long long gtrace) {
      if (!w.valid) return;
      long long a, jmin;
      int r;
      const int k = stream(w, a, jmin, r);
      unsigned char* const sl = ring + slot * stride;
      if ((lead || TCK_TRAIL_TMA) && t == 0) {
        if (lead && !TCK_SCANPROBE) trace_ev(P, gtrace, 13);
        const bool box = k == kTma && !(P.dbg & 8);  // dbg 8: timing probe without input boxes
        umma::mbar_arrive_tx(&full[slot], box ? kBoxBytes : 0u);
        if (box)
          umma::tma_load_3d(umma::smem_u32(sl), &P.in_map, &full[slot], static_cast<int>(a & 31),
                            static_cast<int>(a >> 5), w.sig, keep);
      }
      if (k != kTma) stage_stream(P, P.x + w.sig * P.ld_x, a, jmin, k, t, sl);
      cp_async_arrive(&full[slot]);
    };
    // ring of ahead + 1 tiles: tile gt + ahead is issued before tile gt is moved into TMEM
    // (its slot was last read by tile gt - 1, before the group's barrier)
    uint32_t fph = 0;  // full[] phase bits
    Walk wi, w;
    wi.begin(P);
    w.begin(P);
    for (int k = 0; k < ahead; ++k) {
      issue(wi, k, k);
      if (wi.valid) wi.advance(P);
    }
    int slot = 0, islot = ahead;  // ring slots of tile gt and of tile gt + ahead
    for (long long gt = 0; w.valid; ++gt) {
      issue(wi, islot, gt + ahead);
      if (wi.valid) wi.advance(P);
      if (!lead && t == 0 && !TCK_SCANPROBE) trace_ev(P, gt + ahead, 11);  // trail tile gt + ahead issued
      long long a, jmin;
      int r;
      const int k = stream(w, a, jmin, r);
      umma::mbar_wait(&full[slot], (fph >> slot) & 1u);
      fph ^= 1u << slot;
      umma::fence_proxy_async();  // the cp.async writes precede a later TMA box in this slot
      if (t == 0) trace_ev(P, gt, lead ? 10 : 15);  // slot landed (lead / trail group)
      const int b = static_cast<int>(gt & 1);
      if (gt >= 2) umma::mbar_wait(&M.xfree[b], static_cast<uint32_t>(((gt >> 1) - 1) & 1));
      __syncwarp();
      umma::fence_after();
      if (lead && t == 0) trace_ev(P, gt, 0);
      const unsigned char* sl = ring + slot * stride;
      const uint32_t tx = tmem + lrow + kTX + 128 * b + (lead ? 0 : 64);
      if (k == kMixed) {
        fill_mixed(P.n, P.boundary, umma::smem_u32(sl), t, a, jmin);
        bar_named(bar_id, 128);
      }
      if (P.dbg & 128) {  // dbg 128: timing probe without the X operand stores
      } else if (k == kTma || k == kCp || k == kMixed)
        row_to_tmem(sl, r, t, tx);
      else if (lead || !w.warm(P))  // uniform: zero, x[0] (kFirst) or x[n - 1] (kLast)
        uniform_to_tmem(k == kZero ? 0.f : *reinterpret_cast<const float*>(sl + kValOff + (k == kLast ? 4 : 0)), tx);
      if (!lead && t == 0 && !TCK_SCANPROBE) trace_ev(P, gt, 12);  // trail group: rows written
      umma::tmem_wait_st();
      umma::fence_before();
      umma::mbar_arrive(&M.xfull[b]);
      bar_named(bar_id, 128);  // every row of the slot has been read: it may be refilled
      w.advance(P);
      slot = slot == ahead ? 0 : slot + 1;
      islot = islot == ahead ? 0 : islot + 1;
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
      // accumulator -> registers, then release it at once (it gates the merged GEMM two
      // tiles on); then registers -> staging (row c: 8 chunks of 16 B per half, chunk q at
      // q ^ (c & 7): the TMA SWIZZLE_128B layout of a [128 rows][32 floats] box)
      uint32_t v[2][32];
      if (!(P.dbg & 64)) {  // dbg 64: timing probe without the accumulator load
        umma::tmem_ld32(tmem + lrow + dcol, v[0]);
        if (halves == 2) umma::tmem_ld32(tmem + lrow + dcol + 32, v[1]);
        umma::tmem_wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[0][i] = v[1][i] = static_cast<uint32_t>(c + i);
      }
      umma::fence_before();
      umma::mbar_arrive(&M.dfree[gt & 1]);
      if (c == 0) trace_ev(P, gt, 14);
      // the previous tile's TMA stores must have read the staging area
      if (c == 0 && P.use_tma) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      bar_named(3, 128);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h < halves) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<uint4*>(stgo + h * 16384 + c * 128 + ((q ^ (c & 7)) << 4)) =
                make_uint4(v[h][4 * q], v[h][4 * q + 1], v[h][4 * q + 2], v[h][4 * q + 3]);
        }
      }
      ++u;
      const long long o0 = w.o0(P), cnt = w.cnt(P);
      if (P.use_tma) {
        // one thread hands the tile to the TMA engine: 128 rows x 32 floats per half
        umma::fence_proxy_async();
        bar_named(3, 128);
        if (c == 0) {
          const int row0 = static_cast<int>((w.obase() + o0) / kQ), sg = w.unit(P);
          unsigned long long spol;
          asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(spol));
          for (int h = 0; h < ((P.dbg & 16) ? 0 : halves); ++h) {  // dbg 16: timing probe without stores
            const uint32_t src = umma::smem_u32(stgo + h * 16384);
            if (P.cplx && (P.dbg & 4))
              asm volatile(
                  "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3, %4}], [%5], %6;" ::"l"(
                      reinterpret_cast<uint64_t>(&P.out_map)),
                  "r"(0), "r"(h), "r"(row0), "r"(sg), "r"(src), "l"(spol)
                  : "memory");
            else if (P.cplx)
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
      float* const orow = P.out + (static_cast<long long>(w.unit(P)) * P.ld_out + w.obase()) * cw;
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
    // ================= chunk-state scan (warps 0-7), in three phases per tile:
    //  (1) chunk threads (thread = chunk = TMEM lane; warps 0-3 orders 0-3, warps 4-7
    //      orders 4-7) copy the chunk aggregates A_p[c] from the accumulator into shared
    //      memory, order-major;
    //  (2) warp p scans order p over the tile's 128 chunks: lane t owns chunks 4t..4t+3
    //      (a serial 4-step recurrence), plus one 5-step warp scan with multiplier
    //      z^128 (12 shuffles per order and tile instead of a 5-step scan per chunk);
    //      lane 31 also advances the fp64 tile carry;
    //  (3) chunk threads move their states (TF32 head / remainder) into TMEM and signal
    //      the MMA issuer (sready), which runs the chunk-state GEMM.
    const int os = warp >> 2;
    const int sw = warp & 3;  // lane quarter
    const int p0 = os * 4;
    const int c = sw * 32 + lane;  // chunk of phases (1) and (3)
    const uint32_t lrow = static_cast<uint32_t>(sw * 32) << 16;
    // [order][128]: aggregates, overwritten in place by the states (phase 2: each lane
    // reads its four chunks' aggregates before it writes their states)
    float2* const At = reinterpret_cast<float2*>(sm + kScr);
    float2* const St = At;
    const float2* const zs = reinterpret_cast<const float2*>(sm + kZs);     // [order][8]
    const double2* const zd = reinterpret_cast<const double2*>(sm + kZd);   // z^4096 [order], g0
    const float2* const z128 = reinterpret_cast<const float2*>(sm + kZ128);  // [order][32]
    const int p = warp;  // order of phase (2)
    Walk w;
    w.begin(P);
    long long u = 0;
    int cur = w.scale, nsw = 0;  // scale whose tables are in shared memory; switches
    for (long long gt = 0; w.valid; ++gt) {
      const int b = static_cast<int>(gt & 1);
      if (w.scale != cur) {  // the MMA issuer has copied the new scale's image
        umma::mbar_wait(&M.imgbar, static_cast<uint32_t>(nsw & 1));
        cur = w.scale;
        ++nsw;
      }
      umma::mbar_wait(&M.g1done[b], static_cast<uint32_t>((gt >> 1) & 1));
      if (tid == 0) trace_ev(P, gt, 3);
      __syncwarp();
      umma::fence_after();
      const bool warm = w.warm(P);
      {
        uint32_t a8[8];
        umma::tmem_ld8(tmem + lrow + (b ? kTD1 : kTD0) + NO + 2 * p0, a8);  // this set's orders
        umma::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (p0 + j < nord) At[(p0 + j) * kNC + c] = make_float2(__uint_as_float(a8[2 * j]), __uint_as_float(a8[2 * j + 1]));
      }
      umma::fence_before();
      bar_named(5, 256);
      if (tid == 0) trace_ev(P, gt, 8);
      if (warm && tid == 0) umma::mbar_arrive_cnt(&M.dfree[b], 128);  // nothing else reads it
      if (p < nord) {
        float2 zk[6];  // this order's multipliers: z^32, z^{128 2^k} (k < 5)
#pragma unroll
        for (int k = 0; k < 6; ++k) zk[k] = zs[p * 8 + k];
        const float2 zc = z128[p * 32 + lane];
        const float2 z32 = zk[0];
        const float4 a01 = *reinterpret_cast<const float4*>(At + p * kNC + 4 * lane);
        const float4 a23 = *reinterpret_cast<const float4*>(At + p * kNC + 4 * lane + 2);
        const float2 a0 = make_float2(a01.x, a01.y), a1 = make_float2(a01.z, a01.w);
        const float2 a2 = make_float2(a23.x, a23.y), a3 = make_float2(a23.z, a23.w);
        // group total: sum_j z^{32 (3 - j)} a_j
        float2 g = cmla(z32, cmla(z32, cmla(z32, a0, a1), a2), a3);
        if (TCK_SCANPROBE && p == 0 && lane == 0) trace_ev(P, gt, 13);
        // inclusive warp scan over groups, multiplier z^{128 2^k}
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int d = 1 << k;
          const float2 tt = make_float2(__shfl_up_sync(0xffffffffu, g.x, d), __shfl_up_sync(0xffffffffu, g.y, d));
          if (lane >= d) g = cmla(zk[1 + k], tt, g);
        }
        if (TCK_SCANPROBE && p == 0 && lane == 0) trace_ev(P, gt, 11);
        // fp64 tile carry C (state entering the tile); state entering chunk 4t:
        // sum of the earlier groups (exclusive scan) + z^{128 t} C
        const double2 C = M.cy[b][p];
        float2 e = make_float2(__shfl_up_sync(0xffffffffu, g.x, 1), __shfl_up_sync(0xffffffffu, g.y, 1));
        if (lane == 0) e = make_float2(0.f, 0.f);
        if (!warm) {
          const float2 cf = make_float2(static_cast<float>(C.x), static_cast<float>(C.y));
          const float2 cz = cmla(zc, cf, make_float2(0.f, 0.f));
          const float2 s0 = make_float2(e.x + cz.x, e.y + cz.y);
          const float2 s1 = cmla(z32, s0, a0), s2 = cmla(z32, s1, a1), s3 = cmla(z32, s2, a2);
          *reinterpret_cast<float4*>(St + p * kNC + 4 * lane) = make_float4(s0.x, s0.y, s1.x, s1.y);
          *reinterpret_cast<float4*>(St + p * kNC + 4 * lane + 2) = make_float4(s2.x, s2.y, s3.x, s3.y);
        }
        if (lane == 31) M.tot[p] = g;
      }
      bar_named(5, 256);  // states in shared memory; At / St free for the next tile after phase 3
      if (tid == 0) trace_ev(P, gt, 9);
      if (!warm) {
        uint32_t sh[8], sl[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 s = make_float2(0.f, 0.f);
          if (p0 + j < nord) s = St[(p0 + j) * kNC + c];
          // head = the raw value (the MMA reads its TF32 head), remainder separately
          sh[2 * j] = __float_as_uint(s.x);
          sh[2 * j + 1] = __float_as_uint(s.y);
          sl[2 * j] = __float_as_uint(tf32_lo(s.x));
          sl[2 * j + 1] = __float_as_uint(tf32_lo(s.y));
        }
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
        umma::mbar_arrive(&M.sready[s]);
        if (tid == 0) trace_ev(P, gt, 4);
        ++u;
      }
      // carry into the next tile (fp64): z^{4096} C + (tile total), off the state GEMM's
      // path (read by the next tile's phase 2, after its phase-1 barrier)
      if (p < nord && lane == 31) {
        const double2 zt = zd[p], Cin = M.cy[b][p];
        const float2 gtot = M.tot[p];
        Walk nx = w;
        if (w.last(P)) nx.advance(P);
        M.cy[b ^ 1][p] = w.last(P) ? seg_carry(P, nx, p)
                                   : make_double2(fma(zt.x, Cin.x, fma(-zt.y, Cin.y, static_cast<double>(gtot.x))),
                                                  fma(zt.x, Cin.y, fma(zt.y, Cin.x, static_cast<double>(gtot.y))));
        if (TCK_SCANPROBE && p == 0) trace_ev(P, gt, 12);
      }
      if (w.last(P)) {
        Walk nx = w;
        nx.advance(P);
        if (nx.valid && nx.scale != w.scale) umma::mbar_arrive(&M.scandone);  // done with this image
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
