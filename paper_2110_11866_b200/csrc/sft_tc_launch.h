// Host-visible declarations of K4 (tensor-core chunked transform): parameter block
// layout constants shared by the plan builder (sftgpu_api.cu) and the kernel.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tck {

constexpr int kQ = 32;           // positions per chunk (GEMM K per stream)
constexpr int kNC = 128;         // chunks per tile (GEMM M)
constexpr int kTile = kQ * kNC;  // 4096 positions
constexpr int kMaxOrd = 8;       // 2 * orders <= 16 = GEMM1 N
constexpr int kThreads = 448;  // 14 warps: scan, epilogue, loader, 2 MMA issuers

// shared-memory image (bytes; SW128 regions 1024-aligned)
constexpr uint32_t kHLh = 0, kHLl = 8192, kHTh = 16384, kHTl = 24576, kBC1 = 32768, kBC2 = 40960;
constexpr uint32_t kALh = 49152, kALl = 51200, kATh = 53248, kATl = 55296;
constexpr uint32_t kZl = 57344;        // float2 [kMaxOrd][32]: z^{32 l}
constexpr uint32_t kImage = 59392;     // bytes copied from the plan's device image
constexpr uint32_t kX = kImage;        // [2 stages][XLh, XLl, XTh, XTl] x 16 KB
constexpr uint32_t kXT = 16384;
constexpr uint32_t kSS = kX + 2 * 4 * kXT;  // chunk-state operand [S_hi | S_lo]
constexpr uint32_t kStage = kSS + kXT;      // epilogue staging (128 rows x 128 B)
constexpr uint32_t kMisc = kStage + kXT;
constexpr uint32_t kSmemBytes = kMisc + 1024 + 1024;  // misc + alignment slack

struct TcParams {
  const float* x;
  float* out;
  long long n, ld_x, ld_out;  // ld_out in outputs (complex outputs count once)
  long long lo, count;        // first output position, outputs per signal
  long long chunk_len, n_chunks, n_items, warm_tiles;
  int K, boundary, nord, cplx, vec_ok;
  const uint4* image;  // kImage bytes
  long long* trace;    // optional: per-tile event clocks of CTA 0 ([64][8]), tools/tc_trace.py
  float2 zs[kMaxOrd][6];  // z^{32 * 2^k} (k < 5), z^{1024}
  double2 z1024[kMaxOrd];
  double2 zT[kMaxOrd];  // z^{4096}
};

cudaError_t launch_tc(const TcParams& p, int grid, cudaStream_t s);

}  // namespace tck
