// Explicit instantiation of the K1 launcher: T=double, mode=1, SEQ=true (see scan_launch.cuh).
#define SFTK_INSTANTIATE
#include "scan_launch.cuh"
template void sftk::launch_scan<double, 1, true>(const sftk::LaunchKey&, const sftk::ScanParams<double>&, long long,
                                                  cudaStream_t);
