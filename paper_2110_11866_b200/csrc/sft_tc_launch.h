// Host-visible declarations of K4 (tensor-core chunked transform): parameter block
// layout constants shared by the plan builder (sftgpu_api.cu) and the kernel.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tck {

constexpr int kQ = 32;           // positions per chunk (GEMM K per stream)
constexpr int kNC = 128;         // chunks per tile (GEMM M)
constexpr int kTile = kQ * kNC;  // 4096 positions
constexpr int kMaxOrd = 8;       // 2 * orders <= 16 aggregate columns
constexpr int kThreads = 512;    // 16 warps: scan (2 order sets), epilogue, loader

// shared-memory image (bytes; SW128 K-major B operands, 1024-aligned regions).
// BL/BT: [output rows (NO = 64 complex / 32 real) ; 16 aggregate rows] x 32 positions for
// the lead / trail streams, TF32 head (h) and remainder (l); BC: chunk-state -> output,
// columns [C head (16) | C remainder (16)].
constexpr uint32_t kBLh = 0, kBLl = 10240, kBTh = 20480, kBTl = 30720, kBC = 40960;
constexpr uint32_t kZl = 49152;     // float2 [kMaxOrd][32]: z^{32 l}
constexpr uint32_t kImage = 51200;  // bytes copied from the plan's device image
constexpr uint32_t kStgRow = 36;    // padded staging row (floats): conflict-free row reads
constexpr int kLoadAhead = 2;       // loader lookahead (tiles in flight ahead of the one stored)
constexpr uint32_t kStgWarp = (kLoadAhead + 1) * 2 * 32 * kStgRow * 4;  // [ring slot][stream][32 rows]
constexpr uint32_t kLStage = kImage;                     // loader staging, 4 warps
constexpr uint32_t kStage = kLStage + 4 * kStgWarp;      // epilogue staging (128 rows x 128 B)
constexpr uint32_t kMisc = kStage + 32768;  // epilogue staging: two halves
constexpr uint32_t kSmemBytes = kMisc + 1024 + 1024;  // misc + alignment slack
// TMEM columns (512 allocated): X operands [stage][xl_h, xl_l, xt_h, xt_l] x 32,
// chunk states [2][S_h (16) | S_l (16)], accumulators [2][outputs | aggregates]
constexpr uint32_t kTX = 0, kTSS = 256, kTD0 = 320, kTD1 = 416;

struct TcParams {
  CUtensorMap out_map;  // TMA view of the output (see run_tc); valid when use_tma
  const float* x;
  float* out;
  long long n, ld_x, ld_out;  // ld_out in outputs (complex outputs count once)
  long long lo, count;        // first output position, outputs per signal
  long long chunk_len, n_chunks, n_items, warm_tiles;
  int K, boundary, nord, cplx, vec_ok, use_tma;
  const uint4* image;  // kImage bytes
  long long* trace;    // optional: per-tile event clocks of CTA 0 ([64][8]), tools/tc_trace.py
  float2 zs[kMaxOrd][6];  // z^{32 * 2^k} (k < 5), z^{1024}
  double2 z1024[kMaxOrd];
  double2 zT[kMaxOrd];  // z^{4096}
  // Leading warm-up tiles of a signal's first chunk whose lead samples all lie in the
  // uniform boundary region (before sample 0) are not processed: the state they build is
  // v * g0[p], v = x[0] (clamp) or 0 (zero boundary), g0 = sum_{e < E} z^e (host, fp64).
  int skip0;
  double2 g0[kMaxOrd];
};

cudaError_t launch_tc(const TcParams& p, int grid, cudaStream_t s);

}  // namespace tck
