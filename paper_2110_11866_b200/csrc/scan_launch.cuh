// Launch dispatch for K1. Instantiated per (precision, mode, SEQ) in scan_inst_*.cu so
// the kernel variants compile in parallel; sftgpu_api.cu only sees the declarations.
#pragma once

#include "device_util.cuh"
#include "sft_scan.cuh"

namespace sftk {

// Tile geometry: NT threads x L positions. SEQ (batched) uses long tiles; LB (one
// tile per CTA) uses shorter tiles so a single signal still spreads over the SMs.
constexpr int kThreads = 128;
constexpr int kLSeqF32 = 16, kLSeqF64 = 4;
constexpr int kLLbF32 = 8, kLLbF64 = 4;

template <typename T, bool SEQ>
constexpr int lanes_per_thread() {
  return sizeof(T) == 4 ? (SEQ ? kLSeqF32 : kLLbF32) : (SEQ ? kLSeqF64 : kLLbF64);
}

// Group mode 1 (split injection) is instantiated for the multiplication method's layout:
// NORD = 3P+2 orders of which the first P+1 (kappa terms) use the real constant.
constexpr int split_na(int nord) { return (nord % 3 == 2) ? (nord + 1) / 3 : -1; }
// Group mode 3 (one complex injection constant) is instantiated for 2P+1 orders: the
// multiplication method once its kappa terms are below fp64 resolution (ξ ≳ 9).
constexpr bool has_shared_complex(int nord) { return nord % 2 == 1; }

struct LaunchKey {
  int nord, gm, mode, seq;
};

// Forward-progress assumption of the LB (look-back) launches: tile = blockIdx.x and a tile
// waits only on lower tiles, so progress relies on blocks being dispatched in index order
// with every earlier block already resident or finished (the assumption CUB's single-pass
// scan makes too). A plan's LB launches are serialised (sftgpu_api.cu, lb_order_begin);
// running LB plans concurrently with other kernels that occupy every SM (e.g. under MPS)
// can delay lower tiles but not deadlock as long as started blocks run to completion.
template <typename T, int MODE, bool SEQ>
void launch_scan(const LaunchKey& key, const ScanParams<T>& p, long long grid, cudaStream_t s);

#ifdef SFTK_INSTANTIATE
template <typename T, int NORD, int GM, int MODE, bool SEQ>
static void launch_fixed(const ScanParams<T>& p, long long grid, cudaStream_t s) {
  constexpr int L = lanes_per_thread<T, SEQ>();
  constexpr int NA = GM == kGroupShared ? NORD : (GM == kGroupSplit ? split_na(NORD) : 0);
  constexpr int KGM = GM == kGroupSharedC ? kGroupSplit : GM;
  constexpr size_t smem = sizeof(Smem<T, NORD, L, kThreads, SEQ>);
  auto* kern = &sft_scan_kernel<T, NORD, NA, KGM, MODE, L, kThreads, SEQ>;
  if constexpr (smem > 48 * 1024) {
    // once per device (if it failed, the launch below fails and run_groups reports it)
    static std::atomic<unsigned long long> opted{0};
    (void)smem_opt_in(kern, static_cast<int>(smem), opted);
  }
  kern<<<grid, kThreads, smem, s>>>(p);
}

template <typename T, int NORD, int MODE, bool SEQ>
static void launch_gm(int gm, const ScanParams<T>& p, long long grid, cudaStream_t s) {
  if constexpr (MODE == kModeComplex && split_na(NORD) > 0) {
    if (gm == kGroupSplit) return launch_fixed<T, NORD, kGroupSplit, MODE, SEQ>(p, grid, s);
  }
  if constexpr (MODE == kModeComplex && has_shared_complex(NORD)) {
    if (gm == kGroupSharedC) return launch_fixed<T, NORD, kGroupSharedC, MODE, SEQ>(p, grid, s);
  }
  if (gm == kGroupShared) return launch_fixed<T, NORD, kGroupShared, MODE, SEQ>(p, grid, s);
  launch_fixed<T, NORD, kGroupPerOrder, MODE, SEQ>(p, grid, s);
}

template <typename T, int MODE, bool SEQ>
void launch_scan(const LaunchKey& key, const ScanParams<T>& p, long long grid, cudaStream_t s) {
  switch (key.nord) {
    case 1: launch_gm<T, 1, MODE, SEQ>(key.gm, p, grid, s); break;
    case 2: launch_gm<T, 2, MODE, SEQ>(key.gm, p, grid, s); break;
    case 3: launch_gm<T, 3, MODE, SEQ>(key.gm, p, grid, s); break;
    case 4: launch_gm<T, 4, MODE, SEQ>(key.gm, p, grid, s); break;
    case 5: launch_gm<T, 5, MODE, SEQ>(key.gm, p, grid, s); break;
    case 6: launch_gm<T, 6, MODE, SEQ>(key.gm, p, grid, s); break;
    case 7: launch_gm<T, 7, MODE, SEQ>(key.gm, p, grid, s); break;
    case 8: launch_gm<T, 8, MODE, SEQ>(key.gm, p, grid, s); break;
    case 9: launch_gm<T, 9, MODE, SEQ>(key.gm, p, grid, s); break;
    case 10: launch_gm<T, 10, MODE, SEQ>(key.gm, p, grid, s); break;
    case 11: launch_gm<T, 11, MODE, SEQ>(key.gm, p, grid, s); break;
    default: launch_gm<T, 12, MODE, SEQ>(key.gm, p, grid, s); break;
  }
}
#endif

}  // namespace sftk
