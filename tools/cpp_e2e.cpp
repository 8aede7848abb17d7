// End-to-end timing through the drop-in C++ API with the reference's signature
// (sft::morlet_direct_transform(sig, spec), proj/include/sft/transforms.hpp:86-102) at
// BASELINE config 3 (MDS5P6 fp32 ASFT, N=102400, sigma=8192, xi=10): every call takes
// the fp64 host signal and returns the fp64 complex result (H2D, kernel, D2H and the
// fp64<->fp32 conversion inside), plan cached by the library.
// Build: g++ -std=c++17 -O2 -I include tools/cpp_e2e.cpp -o tools/cpp_e2e -L paper_2110_11866_b200 -lsftgpu -Wl,-rpath,$PWD/paper_2110_11866_b200
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "sft_b200/sft.hpp"

int main(int argc, char** argv) {
  const int steps = argc > 1 ? std::atoi(argv[1]) : 200;
  sft::TransformOptions o;
  o.precision = sft::Precision::Single;
  const sft::TransformSpec spec = sft::make_transform_spec("MDS5P6", 8192.0, 10.0, o);
  const sft::Signal sig = sft::make_test_signal(sft::TestSignalKind::SeededNoise, 102400, 1234);
  for (int i = 0; i < 5; ++i) sft::morlet_direct_transform(sig, spec);
  std::vector<double> us;
  double sink = 0;
  for (int i = 0; i < steps; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    const sft::TransformResult r = sft::morlet_direct_transform(sig, spec);
    const auto t1 = std::chrono::steady_clock::now();
    sink += r.values[12345].real();
    us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
  }
  std::sort(us.begin(), us.end());
  const double med = us[us.size() / 2];
  // the same C ABI call into a reused (already faulted-in) result buffer: what the library
  // itself costs per call, without the page faults of a fresh 1.6 MB result array
  const sftgpu_spec raw = spec.synced();
  std::vector<double> out(2 * 102400);
  int cplx = 0;
  std::vector<double> us2;
  for (int i = 0; i < steps; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    sftgpu_transform_oneshot(&raw, 102400, 1, sig.samples.data(), out.data(), &cplx);
    const auto t1 = std::chrono::steady_clock::now();
    us2.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
  }
  std::sort(us2.begin(), us2.end());
  // the synchronous plan path on pinned fp32 buffers (sftgpu_transform_execute_host)
  sftgpu_plan* pl = nullptr;
  sftgpu_transform_plan_create(&raw, 102400, 1, 1, &pl);
  float *hx = nullptr, *ho = nullptr;
  cudaHostAlloc(reinterpret_cast<void**>(&hx), 102400 * 4, 0);
  cudaHostAlloc(reinterpret_cast<void**>(&ho), 2 * 102400 * 4, 0);
  for (int i = 0; i < 102400; ++i) hx[i] = static_cast<float>(sig.samples[i]);
  std::vector<double> us3;
  for (int i = 0; i < steps + 5; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    sftgpu_transform_execute_host(pl, hx, ho, nullptr);
    const auto t1 = std::chrono::steady_clock::now();
    if (i >= 5) us3.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
  }
  std::sort(us3.begin(), us3.end());
  sftgpu_plan_destroy(pl);
  std::printf("{\"path\": \"sft::morlet_direct_transform(sig, spec) (C++ drop-in, library plan cache)\", "
              "\"us_per_call_median\": %.2f, \"us_per_call_min\": %.2f, \"value\": %.1f, "
              "\"unit\": \"Msamples*scales/s\", \"calls\": %d, \"check\": %.6f, "
              "\"oneshot_reused_buffer_us_median\": %.2f, \"execute_host_pinned_fp32_us_median\": %.2f}\n",
              med, us.front(), 102400.0 / med, steps, sink / steps, us2[us2.size() / 2], us3[us3.size() / 2]);
  return 0;
}
