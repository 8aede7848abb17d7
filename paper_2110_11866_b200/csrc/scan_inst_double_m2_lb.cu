// Explicit instantiation of the K1 launcher: T=double, mode=2, SEQ=false (see scan_launch.cuh).
#define SFTK_INSTANTIATE
#include "scan_launch.cuh"
template void sftk::launch_scan<double, 2, false>(const sftk::LaunchKey&, const sftk::ScanParams<double>&, long long,
                                                  cudaStream_t);
