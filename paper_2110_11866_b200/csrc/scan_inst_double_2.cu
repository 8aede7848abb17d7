// Explicit instantiation of the K1 launcher for T=double, mode=2 (see scan_launch.cuh).
#define SFTK_INSTANTIATE
#include "scan_launch.cuh"
template void sftk::launch_scan<double, 2>(int, int, const sftk::ScanParams<double>&, long long, cudaStream_t);
