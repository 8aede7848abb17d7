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
constexpr int kThreads = 672;    // 21 warps: scan (8), epilogue (4), loaders (4 lead + 4 trail), MMA issuer

// shared-memory image (bytes; SW128 K-major B operands, 1024-aligned regions).
// BL/BT: [output rows (NO = 64 complex / 32 real) ; 16 aggregate rows] x 32 positions for
// the lead / trail streams, TF32 head (h) and remainder (l); BC: chunk-state -> output,
// columns [C head (16) | C remainder (16)].
constexpr uint32_t kBLh = 0, kBLl = 10240, kBTh = 20480, kBTl = 30720, kBC = 40960;
// Per-order scan constants in shared memory (the scan indexes them by order / lane):
constexpr uint32_t kZ128 = 49152;   // float2 [kMaxOrd][32]: z^{128 t}
constexpr uint32_t kZs = 51200;     // float2 [kMaxOrd][8]: z^{32}, z^{128 * 2^k} (k < 5)
constexpr uint32_t kZd = 51712;     // double2 [3][kMaxOrd]: z^{4096}, (unused), g0
constexpr uint32_t kImage = 52096;  // bytes copied from the plan's device image
// Loader staging: one ring per stream, kLoadAhead + 1 (lead) / kTrailAhead + 1 (trail)
// tiles. Each tile stream is 129 SW128 rows of 32 samples (row rho, column i = sample
// a + 32 rho + i, a = the stream's first sample rounded down to 16 bytes; the 129th row
// carries the <= 3 samples a misaligned stream spills past 4096), followed by one word for a
// uniform stream's value. Both streams are TMA boxes inside the signal (1024-aligned
// destinations); the trail reads lines the lead brought into L2 2K samples earlier, so it
// runs fewer tiles ahead. TCK_TRAIL_TMA=0 restores the round-2 16-byte cp.async trail.
#ifndef TCK_TRAIL_TMA
#define TCK_TRAIL_TMA 1
#endif
#ifndef TCK_LEAD_AHEAD
#define TCK_LEAD_AHEAD 3
#endif
#ifndef TCK_TRAIL_AHEAD
#define TCK_TRAIL_AHEAD (TCK_TRAIL_TMA ? 2 : 3)
#endif
constexpr int kLoadAhead = TCK_LEAD_AHEAD;       // lead tiles in flight ahead of the one moved to TMEM
constexpr int kTrailAhead = TCK_TRAIL_AHEAD;     // trail tiles in flight
constexpr uint32_t kBoxRows = kNC + 1;           // 129 rows per stream
constexpr uint32_t kBoxBytes = kBoxRows * 128;   // 16512 bytes of TMA transaction per box
constexpr uint32_t kLeadBytes = 17408;           // lead stride (1024-aligned)
constexpr uint32_t kTrailBytes = TCK_TRAIL_TMA ? 17408 : 16640;  // trail stride (1024- / 128-aligned)
constexpr uint32_t kLStage = (kImage + 1023) / 1024 * 1024;                 // lead ring
constexpr uint32_t kTrail = kLStage + (kLoadAhead + 1) * kLeadBytes;       // trail ring
constexpr uint32_t kStage = kTrail + (kTrailAhead + 1) * kTrailBytes;       // epilogue staging (SW128)
constexpr uint32_t kScr = kStage + 32768;  // epilogue staging: two halves; then the scan's
                                           // aggregates / states [order][chunk] (aliased)
constexpr uint32_t kMisc = kScr + kMaxOrd * kNC * 8;
constexpr uint32_t kSmemBytes = kMisc + 512 + 1024;  // misc + alignment slack
static_assert(kStage % 1024 == 0 && kLStage % 1024 == 0, "SW128 regions need 1024-byte alignment");
static_assert(kSmemBytes <= 232448, "shared memory budget (227 KB)");
// TMEM columns (512 allocated): X operands [stage][xl_h, xl_l, xt_h, xt_l] x 32,
// chunk states [2][S_h (16) | S_l (16)], accumulators [2][outputs | aggregates]
constexpr uint32_t kTX = 0, kTSS = 256, kTD0 = 320, kTD1 = 416;

// One scale (spec) of a K4 launch: its operand image and stream geometry. A launch walks
// units u = scale * nsig + sig; plans over one spec have one scale.
struct TcScale {
  const uint4* image;  // kImage bytes (operands and scan tables of this spec)
  long long lo;        // first output position of the plan (n0 shift applied)
  int K;               // half-width
  int rl, rt;          // (lo + K) mod 4, (lo - K) mod 4: sample offsets of the lead / trail
                       // streams from their 16-byte aligned starts
  int warm_tiles;      // ceil(2K / 4096)
  // Leading warm-up tiles of a unit's first segment whose lead samples all lie in the
  // uniform boundary region (before sample 0) are not processed: the state they build is
  // v * g0[p], v = x[0] (clamp) or 0 (zero boundary), g0 = sum_{e < E} z^e (host, fp64).
  int skip0;
  int pad;
  double2 g0[kMaxOrd];
};

// Per-scale stream geometry in the parameter block (uniform, constant-cached reads on the
// loaders' per-tile path); the rest of a scale lives in TcScale.
constexpr int kMaxScales = 128;  // scales per launch (larger sets launch in groups)
struct TcGeom {
  int lo;                             // first output position (n0 shift applied)
  int K;                              // half-width
  unsigned char rl, rt, warm, skip0;  // see TcScale
  // Units of this scale are cut into nc fixed chunks of L output tiles (the last one
  // shorter); the cut depends only on the spec and the output count, never on the batch
  // or the GPU, so results are reproducible bit for bit across batchings and devices.
  int nc, L;
  int cbase;  // global index of the scale's first chunk
  int wbase;  // tiles (warm-up + output) of all earlier scales' chunks
};

struct TcParams {
  CUtensorMap out_map;  // TMA view of the output (see run_tc); valid when use_tma
  // TMA view of the input for the loader: [signal][row][64 samples], rows 32 samples
  // (128 B) apart, so a box of 32 samples may start at any 16-byte aligned sample
  // (overlapping rows); valid when use_tma_in
  CUtensorMap in_map;
  long long in_rows;  // rows of in_map (row r + 1 of a box must lie below in_rows)
  const float* x;
  float* out;
  long long n, ld_x, ld_out;  // ld_out in outputs (complex outputs count once); out row = unit
  long long count;            // outputs per unit
  int tiles_unit;             // output tiles per unit, ceil(count / 4096)
  int total_chunks;           // chunks of all units
  int total_cost;             // tiles (warm-up + output) of all chunks (< 2^31)
  int nsig, n_scales;
  const TcScale* scales;  // [n_scales], device memory
  TcGeom geo[kMaxScales];
  int boundary, nord, cplx, vec_ok, use_tma, use_tma_in;
  long long* trace;  // optional: per-tile event clocks of CTA 0 ([64][16]), tools/tc_trace.py
  int dbg;           // experiment switches (SFTGPU_TC_DBG): 2 no lead L2 hint, 4 evict-first output stores;
                     // timing probes (wrong results): 8 no input boxes, 16 no output stores, 32 hi.hi MMAs only,
                     // 64 no accumulator load in the epilogue, 128 no X operand stores by the loaders
};

cudaError_t launch_tc(const TcParams& p, int grid, cudaStream_t s);

}  // namespace tck
