// Launch dispatch for K1. Instantiated per (precision, mode) in scan_inst_*.cu so the
// 72 kernel variants compile in parallel; sftgpu_api.cu only sees the declarations.
#pragma once

#include "sft_scan.cuh"

namespace sftk {

template <typename T, int MODE>
void launch_scan(int L, int nord, const ScanParams<T>& p, long long grid, cudaStream_t s);

#ifdef SFTK_INSTANTIATE
template <typename T, int NORD, int MODE>
static void launch_fixed(int L, const ScanParams<T>& p, long long grid, cudaStream_t s) {
  if constexpr (sizeof(T) == 4) {
    if (L == 8) {
      sft_scan_kernel<T, NORD, MODE, 8, 256><<<grid, 256, 0, s>>>(p);
      return;
    }
  }
  sft_scan_kernel<T, NORD, MODE, 4, 256><<<grid, 256, 0, s>>>(p);
}

template <typename T, int MODE>
void launch_scan(int L, int nord, const ScanParams<T>& p, long long grid, cudaStream_t s) {
  switch (nord) {
    case 1: launch_fixed<T, 1, MODE>(L, p, grid, s); break;
    case 2: launch_fixed<T, 2, MODE>(L, p, grid, s); break;
    case 3: launch_fixed<T, 3, MODE>(L, p, grid, s); break;
    case 4: launch_fixed<T, 4, MODE>(L, p, grid, s); break;
    case 5: launch_fixed<T, 5, MODE>(L, p, grid, s); break;
    case 6: launch_fixed<T, 6, MODE>(L, p, grid, s); break;
    case 7: launch_fixed<T, 7, MODE>(L, p, grid, s); break;
    case 8: launch_fixed<T, 8, MODE>(L, p, grid, s); break;
    case 9: launch_fixed<T, 9, MODE>(L, p, grid, s); break;
    case 10: launch_fixed<T, 10, MODE>(L, p, grid, s); break;
    case 11: launch_fixed<T, 11, MODE>(L, p, grid, s); break;
    default: launch_fixed<T, 12, MODE>(L, p, grid, s); break;
  }
}
#endif

}  // namespace sftk
