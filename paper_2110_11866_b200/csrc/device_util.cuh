// Per-device host helpers shared by the launchers: the SM count (grid sizing) and the
// dynamic shared-memory opt-in. Both are per device, so a process that drives several
// GPUs (one plan per device) gets each device's own value / attribute.
#pragma once

#include <cuda_runtime.h>

#include <atomic>

namespace sftk {

constexpr int kMaxDevices = 64;

// Multiprocessor count of the current device (cached per device; 148 on B200).
inline int sm_count() {
  static std::atomic<int> cache[kMaxDevices] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 148;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1) v = 148;
  cache[dev].store(v, std::memory_order_relaxed);
  return v;
}

// Opts `kern` into `bytes` of dynamic shared memory on the current device, once per
// device (`done` is one bit per device, owned by the caller's kernel instantiation).
template <typename Kern>
inline cudaError_t smem_opt_in(Kern* kern, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
  return e;
}

}  // namespace sftk
