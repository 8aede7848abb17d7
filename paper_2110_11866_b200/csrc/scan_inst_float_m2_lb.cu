// Explicit instantiation of the K1 launcher: T=float, mode=2, SEQ=false (see scan_launch.cuh).
#define SFTK_INSTANTIATE
#include "scan_launch.cuh"
template void sftk::launch_scan<float, 2, false>(const sftk::LaunchKey&, const sftk::ScanParams<float>&, long long,
                                                  cudaStream_t);
