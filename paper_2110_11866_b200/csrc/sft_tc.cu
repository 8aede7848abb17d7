// K4 launch (tensor-core chunked transform). The kernel lives in sft_tc.cuh; the
// operand image and the per-order constants are built by the plan (sftgpu_api.cu).
#include "device_util.cuh"
#include "sft_tc.cuh"
#include "sft_tc_launch.h"

namespace tck {

template <int NORD>
static cudaError_t launch_n(const TcParams& p, int grid, cudaStream_t s) {
  static std::atomic<unsigned long long> opted{0};  // once per device
  const cudaError_t opt_in = sftk::smem_opt_in(sft_tc_kernel<NORD>, static_cast<int>(kSmemBytes), opted);
  if (opt_in != cudaSuccess) return opt_in;
  sft_tc_kernel<NORD><<<grid, kThreads, kSmemBytes, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_tc(const TcParams& p, int grid, cudaStream_t s) {
  switch (p.nord) {
    case 1: return launch_n<1>(p, grid, s);
    case 2: return launch_n<2>(p, grid, s);
    case 3: return launch_n<3>(p, grid, s);
    case 4: return launch_n<4>(p, grid, s);
    case 5: return launch_n<5>(p, grid, s);
    case 6: return launch_n<6>(p, grid, s);
    case 7: return launch_n<7>(p, grid, s);
    default: return launch_n<8>(p, grid, s);
  }
}

}  // namespace tck
