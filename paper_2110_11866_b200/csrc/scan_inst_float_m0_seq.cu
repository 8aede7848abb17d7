// Explicit instantiation of the K1 launcher: T=float, mode=0, SEQ=true (see scan_launch.cuh).
#define SFTK_INSTANTIATE
#include "scan_launch.cuh"
template void sftk::launch_scan<float, 0, true>(const sftk::LaunchKey&, const sftk::ScanParams<float>&, long long,
                                                  cudaStream_t);
