// libsftgpu C ABI: plans, launch dispatch, workspace, host transfers, and the
// C wrappers of the host precompute (fits / spec factories). See include/sftgpu.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <thread>
#include <cstdlib>
#include <type_traits>
#include <cmath>
#include <complex>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sftgpu.h"
#include "aux_kernels.cuh"
#include "host_fit.hpp"
#include "scan_launch.cuh"
#include "sft_tc_launch.h"

namespace {
using cd = std::complex<double>;
}  // namespace
thread_local std::string g_err;
namespace {

struct ApiError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& m) { throw ApiError{code, m}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(SFTGPU_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return SFTGPU_OK;
  } catch (const ApiError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const sftb::FitDegenerate& e) {
    g_err = e.what();
    return SFTGPU_EDEGENERATE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return SFTGPU_EINVAL;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return SFTGPU_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SFTGPU_EINTERNAL;
  }
}

void require_device() {
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    fail(SFTGPU_ECUDA, "no CUDA device available (libsftgpu has no CPU fallback)");
}

// z^m for z = e^{-alpha - i omega} (m may be negative).
cd zpow(double alpha, double omega, double m) {
  const double mag = std::exp(-alpha * m);
  const double ang = omega * m;
  return cd(mag * std::cos(ang), -mag * std::sin(ang));
}

// One component sequence of the lowered transform: frequency + combine weights on
// (c, s) as in the reference combine loops (wc * c + ws * s, complex weights).
struct Order {
  double omega;
  cd wc, ws;
};

struct Lowered {
  std::vector<Order> orders;
  double alpha = 0.0;
  double prefactor = 1.0;
  bool complex_out = false;
  int K = 1;
};

// Group of <= kMaxOrd orders executed by one kernel launch.
struct Group {
  int nord = 0;
  int gm = sftk::kGroupPerOrder;
  sftk::ScanParams<float> pf{};
  sftk::ScanParams<double> pd{};
  void* d_tab = nullptr;
  double2* d_tab_tile = nullptr;
};

}  // namespace

struct sftgpu_plan {
  int is_components = 0;
  int precision = SFTGPU_DOUBLE;
  int mode = sftk::kModeReal;
  int conv = 0;  // GCT3/MCT3 direct convolution plan
  long long n = 0, batch = 0, lo = 0, count = 0;
  long long in_batch = -1;  // input signals when not `batch` (multi-scale plans: 1 signal, batch = scales)
  int K = 1, boundary = SFTGPU_BOUNDARY_CLAMP;
  int L = 8, NT = 128;
  int seq = 0;  // 1: one CTA walks a whole (signal, chunk), no look-back workspace
  int mode_hint = 0;  // 0 auto, 1 force SEQ (chunked), 2 force LB
  long long n_chunks = 1, chunk_len = 0;
  long long TT = 1024, tiles_per_signal = 0, warm_tiles = 0, total_tiles = 0;
  std::vector<Group> groups;
  int max_nord = 1;
  unsigned int* d_ctrl = nullptr;  // LB: 64-bit count of CTAs ever started (launch epochs)
  // LB launches of one plan share the workspace and number themselves from d_ctrl, so
  // they must never overlap: each launch waits on the event the previous one recorded
  // when it was issued on a different stream (same stream: already ordered)
  cudaEvent_t ev_lb = nullptr;
  cudaStream_t lb_stream = nullptr;
  bool lb_recorded = false;
  unsigned long long* d_flags = nullptr;
  double2* d_agg = nullptr;
  double2* d_incl = nullptr;
  // direct-convolution plans
  double2* d_taps = nullptr;
  long long n_taps = 0, tap_lo = 0;
  double2* d_conv_tmp = nullptr;
  // host-transfer staging
  void* d_x = nullptr;
  void* d_out = nullptr;
  size_t cap_x = 0, cap_out = 0;
  int device = 0;
  // K4 (tensor-core chunked transform): operand image + parameter block
  int tc = 0;
  void* d_tc_image = nullptr;            // [scales][kImage] operand images
  tck::TcScale* d_tc_scales = nullptr;  // [scales] descriptors
  tck::TcParams tcp{};
  int tc_grid = 0, tc_warm = 0;
  const void* tc_map_out = nullptr;  // output buffer the cached TMA map describes
  long long tc_map_ld = -1;
  const void* tc_map_in = nullptr;  // input buffer the cached loader map describes
  long long tc_map_in_ld = -1;
  // pipelined host execution: internal copy-in / compute / copy-out streams and a ring
  // of staging slots, so the transfers of neighbouring calls overlap this call's kernel
  struct Slot {
    void* d_x = nullptr;
    void* d_out = nullptr;
    cudaEvent_t ev_in = nullptr, ev_comp = nullptr, ev_out = nullptr;
  };
  static constexpr int kSlots = 3;
  Slot slots[kSlots];
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
  cudaEvent_t ev_entry = nullptr;
  int next_slot = 0;
  // sub-batched synchronous host execution (large K4 plans): two device staging slots
  void* sb_x[2] = {nullptr, nullptr};
  void* sb_out[2] = {nullptr, nullptr};
  size_t sb_cap_x[2] = {0, 0}, sb_cap_out[2] = {0, 0};

  ~sftgpu_plan() {
    if (s_in) {
      cudaStreamSynchronize(s_in);
      cudaStreamSynchronize(s_comp);
      cudaStreamSynchronize(s_out);
      for (Slot& sl : slots) {
        cudaFree(sl.d_x);
        cudaFree(sl.d_out);
        cudaEventDestroy(sl.ev_in);
        cudaEventDestroy(sl.ev_comp);
        cudaEventDestroy(sl.ev_out);
      }
      cudaEventDestroy(ev_entry);
      cudaStreamDestroy(s_in);
      cudaStreamDestroy(s_comp);
      cudaStreamDestroy(s_out);
    }
    for (Group& g : groups) {
      cudaFree(g.d_tab);
      cudaFree(g.d_tab_tile);
    }
    for (int k = 0; k < 2; ++k) {
      cudaFree(sb_x[k]);
      cudaFree(sb_out[k]);
    }
    cudaFree(d_tc_image);
    cudaFree(d_tc_scales);
    if (ev_lb) cudaEventDestroy(ev_lb);
    cudaFree(d_ctrl);
    cudaFree(d_flags);
    cudaFree(d_agg);
    cudaFree(d_incl);
    cudaFree(d_taps);
    cudaFree(d_conv_tmp);
    cudaFree(d_x);
    cudaFree(d_out);
  }
};

namespace {

size_t elem_size(int precision) { return precision == SFTGPU_SINGLE ? sizeof(float) : sizeof(double); }

// ---------------------------------------------------------------- kernel dispatch
template <typename T>
void launch_scan(const sftgpu_plan* pl, const Group& g, const sftk::ScanParams<T>& p, cudaStream_t s) {
  if (g.nord < 1 || g.nord > sftk::kMaxOrd) fail(SFTGPU_EINTERNAL, "order group size out of range");
  const long long grid = pl->seq ? pl->batch * pl->n_chunks : pl->total_tiles;
  const sftk::LaunchKey key{g.nord, g.gm, pl->mode, pl->seq};
  switch (pl->mode) {
    case sftk::kModeReal:
      pl->seq ? sftk::launch_scan<T, sftk::kModeReal, true>(key, p, grid, s)
              : sftk::launch_scan<T, sftk::kModeReal, false>(key, p, grid, s);
      break;
    case sftk::kModeComplex:
      pl->seq ? sftk::launch_scan<T, sftk::kModeComplex, true>(key, p, grid, s)
              : sftk::launch_scan<T, sftk::kModeComplex, false>(key, p, grid, s);
      break;
    default: sftk::launch_scan<T, sftk::kModeComps, false>(key, p, grid, s); break;
  }
}

// ---------------------------------------------------------------- plan building
// Orders whose trailing-sample injection constants z^{2K} coincide share one g per
// position. Returns the group mode and reorders `ords` so the real-shared group comes
// first (na orders), followed by the complex-shared group.
int detect_groups(std::vector<Order>& ords, double alpha, int K, cd* cA, cd* cB, int* na) {
  auto cinj = [&](const Order& o) { return zpow(alpha, o.omega, 2.0 * K); };
  auto same = [](cd a, cd b) { return std::abs(a - b) <= 1e-13 * std::max(1.0, std::abs(a)); };
  auto is_real = [](cd a) { return std::abs(a.imag()) <= 1e-13 * std::max(1.0, std::abs(a)); };
  std::vector<cd> reps;
  for (const Order& o : ords) {
    const cd c = cinj(o);
    bool found = false;
    for (const cd& r : reps) found = found || same(r, c);
    if (!found) reps.push_back(c);
  }
  if (reps.size() == 1 && is_real(reps[0])) {
    *cA = cd(reps[0].real(), 0.0);
    *na = static_cast<int>(ords.size());
    return sftk::kGroupShared;
  }
  if (reps.size() <= 2) {
    int ireal = -1;
    for (size_t i = 0; i < reps.size(); ++i)
      if (is_real(reps[i])) ireal = static_cast<int>(i);
    if (reps.size() == 1 || ireal >= 0) {
      const cd a = ireal >= 0 ? cd(reps[ireal].real(), 0.0) : cd(0.0, 0.0);
      const cd b = reps.size() == 1 ? reps[0] : reps[1 - ireal];
      std::stable_partition(ords.begin(), ords.end(), [&](const Order& o) { return ireal >= 0 && same(cinj(o), a); });
      *na = 0;
      for (const Order& o : ords) *na += (ireal >= 0 && same(cinj(o), a)) ? 1 : 0;
      *cA = a;
      *cB = b;
      return sftk::kGroupSplit;
    }
  }
  *na = 0;
  return sftk::kGroupPerOrder;
}

template <typename T>
void fill_consts(sftk::ScanParams<T>& P, const std::vector<Order>& ords, double alpha, double pref,
                 int K, int L, bool comps, double* Dr, double* Di) {
  cd D(0.0, 0.0);
  for (size_t i = 0; i < ords.size(); ++i) {
    const double w = ords[i].omega;
    const cd z = zpow(alpha, w, 1.0), c = zpow(alpha, w, 2.0 * K);
    const cd a = zpow(alpha, w, -static_cast<double>(K)), b = zpow(alpha, w, static_cast<double>(K));
    double k[4];
    if (comps) {
      k[0] = a.real();
      k[1] = a.imag();
      k[2] = b.real();
      k[3] = b.imag();
    } else {
      const cd A = pref * (ords[i].wc + cd(0, 1) * ords[i].ws) * 0.5;
      const cd B = pref * (ords[i].wc - cd(0, 1) * ords[i].ws) * 0.5;
      const cd E = A * a, F = B * std::conj(a);
      k[0] = E.real() + F.real();
      k[1] = F.imag() - E.imag();
      k[2] = E.imag() + F.imag();
      k[3] = E.real() - F.real();
      D += A * b + B * std::conj(b);
    }
    for (double v : k)
      if (!std::isfinite(static_cast<double>(static_cast<T>(v))))
        fail(SFTGPU_EINVAL, "attenuation alpha*K too large for the requested precision");
    sftk::OrdConst<T>& o = P.oc[i];
    const T zr = static_cast<T>(z.real()), zi = static_cast<T>(z.imag());
    o.zz[0] = zr;
    o.zz[1] = zr;
    o.zx[0] = -zi;
    o.zx[1] = zi;
    o.ka[0] = static_cast<T>(k[0]);
    o.ka[1] = static_cast<T>(k[2]);
    o.kb[0] = static_cast<T>(k[1]);
    o.kb[1] = static_cast<T>(k[3]);
    o.cc[0] = static_cast<T>(c.real());
    o.cc[1] = static_cast<T>(c.imag());
    auto put4 = [](T* d, cd v) {  // {re, re, -im, im}
      d[0] = static_cast<T>(v.real());
      d[1] = static_cast<T>(v.real());
      d[2] = static_cast<T>(-v.imag());
      d[3] = static_cast<T>(v.imag());
    };
    for (int k2 = 0; k2 < 5; ++k2) put4(o.scan[k2], zpow(alpha, w, static_cast<double>(L) * (1 << k2)));
    for (int wi = 0; wi < 4; ++wi) put4(o.wrot[wi], zpow(alpha, w, 32.0 * L * wi));
    put4(o.m32, zpow(alpha, w, 32.0 * L));
    for (int j = 0; j < L; ++j) {
      const cd wj = zpow(alpha, w, static_cast<double>(L - 1 - j));
      const T wr = static_cast<T>(wj.real()), wi = static_cast<T>(wj.imag());
      o.w[j][0] = wr;
      o.w[j][1] = wi;
      o.w[j][2] = -wi;
      o.w[j][3] = wr;
    }
  }
  *Dr = D.real();
  *Di = D.imag();
}

template <typename T>
void build_tables(Group& g, const std::vector<Order>& ords, double alpha, int L, int NT, int K) {
  const int NW = NT / 32;
  const long long TT = static_cast<long long>(L) * NT;
  std::vector<T> tab(static_cast<size_t>(ords.size()) * sftk::kTabStride * 4, T(0));
  std::vector<double2> tt(static_cast<size_t>(ords.size()) * sftk::kTabTileStride);
  const long long cnt = (2LL * K) / TT + 1;  // LB window-carry predecessors (lb_D + 1)
  const int G = ords.size() <= 8 ? 4 : 2;
  const long long seg = (cnt + G - 1) / G;
  auto put = [](T* d, cd v) {  // {re, re, -im, im}
    d[0] = static_cast<T>(v.real());
    d[1] = static_cast<T>(v.real());
    d[2] = static_cast<T>(-v.imag());
    d[3] = static_cast<T>(v.imag());
  };
  for (size_t p = 0; p < ords.size(); ++p) {
    const double w = ords[p].omega;
    T* t = &tab[p * sftk::kTabStride * 4];
    for (int lane = 0; lane < 32; ++lane) put(t + lane * 4, zpow(alpha, w, static_cast<double>(L) * lane));
    for (int k = 0; k < 5; ++k) put(t + (32 + k) * 4, zpow(alpha, w, static_cast<double>(L) * (1 << k)));
    for (int wi = 0; wi < NW; ++wi) put(t + (40 + wi) * 4, zpow(alpha, w, 32.0 * L * wi));
    for (int k = 0; k < 4; ++k) put(t + (56 + k) * 4, zpow(alpha, w, 32.0 * L * (1 << k)));
    for (int l = 0; l < 2; ++l) {
      const cd v = zpow(alpha, w, static_cast<double>(TT) * (l == 0 ? 1 : 32));
      tt[p * sftk::kTabTileStride + l] = make_double2(v.real(), v.imag());
    }
    for (int gi = 0; gi < 4; ++gi) {
      const long long e = cnt - std::min(cnt, (gi + 1) * seg);
      const cd v = zpow(alpha, w, static_cast<double>(TT) * static_cast<double>(e));
      tt[p * sftk::kTabTileStride + 2 + gi] = make_double2(v.real(), v.imag());
    }
  }
  cuda_check(cudaMalloc(&g.d_tab, tab.size() * sizeof(T)), "cudaMalloc tables");
  cuda_check(cudaMemcpy(g.d_tab, tab.data(), tab.size() * sizeof(T), cudaMemcpyHostToDevice), "copy tables");
  cuda_check(cudaMalloc(&g.d_tab_tile, tt.size() * sizeof(double2)), "cudaMalloc tile tables");
  cuda_check(cudaMemcpy(g.d_tab_tile, tt.data(), tt.size() * sizeof(double2), cudaMemcpyHostToDevice),
             "copy tile tables");
}

template <typename T>
sftk::ScanParams<T>& params_of(Group& g);
template <>
sftk::ScanParams<float>& params_of<float>(Group& g) {
  return g.pf;
}
template <>
sftk::ScanParams<double>& params_of<double>(Group& g) {
  return g.pd;
}

template <typename T>
void build_groups(sftgpu_plan* pl, std::vector<Order> ords, double alpha, double pref, bool comps) {
  for (size_t g0 = 0; g0 < ords.size(); g0 += sftk::kMaxOrd) {
    const size_t g1 = std::min(ords.size(), g0 + sftk::kMaxOrd);
    std::vector<Order> sub(ords.begin() + g0, ords.begin() + g1);
    pl->groups.emplace_back();
    Group& g = pl->groups.back();
    g.nord = static_cast<int>(sub.size());
    sftk::ScanParams<T>& P = params_of<T>(g);
    std::memset(&P, 0, sizeof(P));
    cd cA(0, 0), cB(0, 0);
    int na = 0;
    // components keep their order (outputs are per order); transforms may regroup
    g.gm = comps ? sftk::kGroupPerOrder : detect_groups(sub, alpha, pl->K, &cA, &cB, &na);
    if (g.gm == sftk::kGroupSplit && na == 0 && pl->mode == sftk::kModeComplex && sftk::has_shared_complex(g.nord))
      g.gm = sftk::kGroupSharedC;  // one complex constant for every order
    else if (g.gm == sftk::kGroupSplit && (pl->mode != sftk::kModeComplex || sftk::split_na(g.nord) != na))
      g.gm = sftk::kGroupPerOrder;  // only the multiplication-method layout has a split kernel
    if (comps) {
      std::vector<Order> probe = sub;
      cd a2, b2;
      int n2;
      if (detect_groups(probe, alpha, pl->K, &a2, &b2, &n2) == sftk::kGroupShared) {
        g.gm = sftk::kGroupShared;
        cA = a2;
        na = n2;
      }
    }
    P.cAr = static_cast<T>(cA.real());
    P.cAi = static_cast<T>(cA.imag());
    P.cBr = static_cast<T>(cB.real());
    P.cBi = static_cast<T>(cB.imag());
    P.na = na;
    double Dr = 0, Di = 0;
    fill_consts<T>(P, sub, alpha, pref, pl->K, pl->L, comps, &Dr, &Di);
    // each launch adds its own orders' share of the x[n-K] term
    P.Dr = static_cast<T>(Dr);
    P.Di = static_cast<T>(Di);
    build_tables<T>(g, sub, alpha, pl->L, pl->NT, pl->K);
    P.tab = static_cast<const T*>(g.d_tab);
    P.tab_tile = g.d_tab_tile;
  }
  pl->max_nord = 1;
  for (const Group& g : pl->groups) pl->max_nord = std::max(pl->max_nord, g.nord);
}

// Geometry. SEQ: one CTA per (signal, chunk); a chunk starts from its own warm-up
// 2K positions early (phase-1 work only), so chunks are kept >= 8 tiles and >= 16K
// positions long (warm-up <= ~1/8 of the chunk's positions). LB: one tile per CTA
// with look-back. Auto picks SEQ when the (signal, chunk) grid gives >= 2 CTAs per SM.
void choose_geometry(sftgpu_plan* pl) {
  const bool dbl = pl->precision == SFTGPU_DOUBLE;
  const long long kSms = sftk::sm_count(), kTarget = 4 * kSms;
  pl->NT = sftk::kThreads;
  const long long tt_seq = static_cast<long long>(dbl ? sftk::kLSeqF64 : sftk::kLSeqF32) * pl->NT;
  const long long cmin = ((std::max(8 * tt_seq, 16LL * pl->K) + tt_seq - 1) / tt_seq) * tt_seq;
  const long long max_chunks = std::max(1LL, (pl->count + cmin - 1) / cmin);
  const long long want = std::max(1LL, (kTarget + pl->batch - 1) / pl->batch);
  long long chunks = std::min(max_chunks, want);
  bool seq;
  if (pl->is_components)
    seq = false;
  else if (pl->mode_hint == 1)
    seq = true;
  else if (pl->mode_hint == 2)
    seq = false;
  else
    seq = pl->batch * chunks >= 2 * kSms;
  pl->seq = seq ? 1 : 0;
  pl->L = seq ? (dbl ? sftk::kLSeqF64 : sftk::kLSeqF32) : (dbl ? sftk::kLLbF64 : sftk::kLLbF32);
  pl->TT = static_cast<long long>(pl->L) * pl->NT;
  pl->warm_tiles = (2LL * pl->K + pl->TT - 1) / pl->TT;
  if (seq) {
    const long long per = (pl->count + chunks - 1) / chunks;
    pl->chunk_len = ((per + pl->TT - 1) / pl->TT) * pl->TT;
    pl->n_chunks = (pl->count + pl->chunk_len - 1) / pl->chunk_len;
    pl->tiles_per_signal = pl->warm_tiles + pl->chunk_len / pl->TT;
    pl->total_tiles = pl->batch * pl->n_chunks;
  } else {
    pl->n_chunks = 1;
    pl->chunk_len = pl->count;
    pl->tiles_per_signal = pl->warm_tiles + (pl->count + pl->TT - 1) / pl->TT;
    pl->total_tiles = pl->tiles_per_signal * pl->batch;
  }
}

void alloc_workspace(sftgpu_plan* pl) {
  if (pl->seq) return;  // SEQ mode needs no inter-CTA state
  if (pl->total_tiles >= (1LL << 31)) fail(SFTGPU_EINVAL, "problem too large for one plan (tiles >= 2^31)");
  // ctrl[0..1]: the 64-bit started-CTA count (launch k has epoch k + 1 >= 1)
  cuda_check(cudaMalloc(&pl->d_ctrl, 4 * sizeof(unsigned int)), "cudaMalloc ctrl");
  cuda_check(cudaMemset(pl->d_ctrl, 0, 4 * sizeof(unsigned int)), "init ctrl");
  cuda_check(cudaMalloc(&pl->d_flags, pl->total_tiles * sizeof(unsigned long long)), "cudaMalloc flags");
  cuda_check(cudaMemset(pl->d_flags, 0, pl->total_tiles * sizeof(unsigned long long)), "memset flags");
  // Payloads are zeroed too: fp32 plans accept a payload word by its launch tag (low 4
  // bits, 1..15) and a zero word carries tag 0, which never matches. Without this a new
  // plan could accept the tagged payloads a freed plan left at the same address.
  const size_t pay = static_cast<size_t>(pl->total_tiles) * pl->max_nord * sizeof(double2);
  cuda_check(cudaMalloc(&pl->d_agg, pay), "cudaMalloc aggregates");
  cuda_check(cudaMalloc(&pl->d_incl, pay), "cudaMalloc prefixes");
  cuda_check(cudaMemset(pl->d_agg, 0, pay), "memset aggregates");
  cuda_check(cudaMemset(pl->d_incl, 0, pay), "memset prefixes");
  cuda_check(cudaEventCreateWithFlags(&pl->ev_lb, cudaEventDisableTiming), "event create");
  cuda_check(cudaStreamSynchronize(nullptr), "workspace init");  // memsets done before any launch
}

// Orders an LB launch after the plan's previous one (see sftgpu_plan::ev_lb). During
// stream capture the graph's own edges order the launches (one capture chain per plan).
bool lb_capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cuda_check(cudaStreamIsCapturing(st, &cs), "cudaStreamIsCapturing");
  return cs != cudaStreamCaptureStatusNone;
}
void lb_order_begin(sftgpu_plan* pl, cudaStream_t st, bool capturing) {
  if (capturing || !pl->lb_recorded || pl->lb_stream == st) return;
  cuda_check(cudaStreamWaitEvent(st, pl->ev_lb, 0), "stream wait (look-back ordering)");
}
void lb_order_end(sftgpu_plan* pl, cudaStream_t st, bool capturing) {
  if (capturing) return;
  cuda_check(cudaEventRecord(pl->ev_lb, st), "event record (look-back ordering)");
  pl->lb_stream = st;
  pl->lb_recorded = true;
}


// ---------------------------------------------------------------- K4 (tensor cores)
// Builds the SW128 operand image of sft_tc.cuh from the lowered orders (fp64), and the
// plan geometry. Eligible: fp32 transform, <= 8 orders sharing one injection constant
// z^{2K} (group modes 0 and 3), enough tiles to fill the GPU (or mode_hint 3).
uint32_t sw128(uint32_t row, uint32_t k) { return row * 128u + ((((k >> 2) ^ (row & 7u)) << 4) | ((k & 3u) << 2)); }
float tf32_head(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u &= 0xFFFFE000u;
  std::memcpy(&f, &u, 4);
  return f;
}

// K4 eligibility of one lowered spec: fp32, <= 8 orders sharing one injection constant
// z^{2K} (group modes 0 and 3). Returns the injection constant through cinj.
bool tc_eligible(const sftgpu_plan* pl, const Lowered& lw, bool force, cd* cinj_out) {
  auto no = [&](const char* why) {
    if (force) fail(SFTGPU_EINVAL, std::string("tensor-core mode unavailable: ") + why);
    return false;
  };
  if (pl->precision != SFTGPU_SINGLE) return no("needs single precision");
  if (lw.orders.empty() || lw.orders.size() > static_cast<size_t>(tck::kMaxOrd)) return no("needs 1..8 orders");
  std::vector<Order> ords = lw.orders;
  cd cA(0, 0), cB(0, 0);
  int na = 0;
  const int gm = detect_groups(ords, lw.alpha, lw.K, &cA, &cB, &na);
  if (gm == sftk::kGroupShared)
    *cinj_out = cA;
  else if (gm == sftk::kGroupSplit && na == 0)
    *cinj_out = cB;
  else
    return no("orders do not share one injection constant");
  return true;
}

// The SW128 operand image and scan tables of one spec (sft_tc.cuh), and its stream
// geometry for a plan whose first output position is lo.
void tc_build_scale(const Lowered& lw, cd cinj, long long lo, std::vector<unsigned char>& img, tck::TcScale& sc) {
  const std::vector<Order>& ords = lw.orders;
  const bool cplx = lw.complex_out;
  const int nord = static_cast<int>(ords.size());
  const double alpha = lw.alpha, pref = lw.prefactor;
  const int K = lw.K;
  // combine weights K_p(w) = (k0 Re w + k1 Im w, k2 Re w + k3 Im w) and the x[n-K] weight D
  std::vector<std::array<double, 4>> kw(nord);
  cd D(0, 0);
  for (int p = 0; p < nord; ++p) {
    const double w = ords[p].omega;
    const cd a = zpow(alpha, w, -static_cast<double>(K)), b = zpow(alpha, w, static_cast<double>(K));
    const cd A = pref * (ords[p].wc + cd(0, 1) * ords[p].ws) * 0.5;
    const cd B = pref * (ords[p].wc - cd(0, 1) * ords[p].ws) * 0.5;
    const cd E = A * a, F = B * std::conj(a);
    kw[p] = {E.real() + F.real(), F.imag() - E.imag(), E.imag() + F.imag(), E.real() - F.real()};
    D += A * b + B * std::conj(b);
  }
  auto Kp = [&](int p, cd v) { return cd(kw[p][0] * v.real() + kw[p][1] * v.imag(), kw[p][2] * v.real() + kw[p][3] * v.imag()); };
  img.assign(tck::kImage, 0);
  auto put = [&](uint32_t region, int row, int k, float v) { std::memcpy(&img[region + sw128(row, k)], &v, 4); };
  auto put_split = [&](uint32_t rh, uint32_t rl, int row, int k, double v) {
    const float h = tf32_head(static_cast<float>(v));
    put(rh, row, k, h);
    if (rl != 0xFFFFFFFFu) put(rl, row, k, static_cast<float>(v - static_cast<double>(h)));
    return static_cast<float>(v - static_cast<double>(h));
  };
  // effective kernel taps on the lead / trail streams, lag d = 0..31
  std::vector<cd> hl(tck::kQ), ht(tck::kQ);
  for (int d = 0; d < tck::kQ; ++d) {
    cd sl(0, 0), st(0, 0);
    for (int p = 0; p < nord; ++p) {
      const cd zd = zpow(alpha, ords[p].omega, d);
      sl += Kp(p, zd);
      st += Kp(p, -cinj * zd);
    }
    if (d == 0) st += D;
    hl[d] = sl;
    ht[d] = st;
  }
  const int comps = cplx ? 2 : 1;
  const int NO = comps * tck::kQ;  // output rows of the merged B operands; aggregates follow
  for (int i = 0; i < tck::kQ; ++i)
    for (int r = 0; r < comps; ++r) {
      const int j = comps * i + r;
      for (int m = 0; m <= i; ++m) {
        const cd vl = hl[i - m], vt = ht[i - m];
        put_split(tck::kBLh, tck::kBLl, j, m, r == 0 ? vl.real() : vl.imag());
        put_split(tck::kBTh, tck::kBTl, j, m, r == 0 ? vt.real() : vt.imag());
      }
      // chunk start state S_p -> output i: K_p(z^{i+1} S_p); columns [head | remainder]
      for (int p = 0; p < nord; ++p) {
        const cd a = zpow(alpha, ords[p].omega, i + 1.0);
        const double k0 = r == 0 ? kw[p][0] : kw[p][2], k1 = r == 0 ? kw[p][1] : kw[p][3];
        const double cr = k0 * a.real() + k1 * a.imag(), ci = -k0 * a.imag() + k1 * a.real();
        for (int q = 0; q < 2; ++q) {
          const double v = q == 0 ? cr : ci;
          const float h = tf32_head(static_cast<float>(v));
          put(tck::kBC, j, 2 * p + q, h);
          put(tck::kBC, j, 16 + 2 * p + q, static_cast<float>(v - static_cast<double>(h)));
        }
      }
    }
  // chunk aggregates A_p = sum_m z^{31-m} (xl[m] - c xt[m]) in rows NO + 2p (+1)
  for (int p = 0; p < nord; ++p)
    for (int m = 0; m < tck::kQ; ++m) {
      const cd zl = zpow(alpha, ords[p].omega, tck::kQ - 1.0 - m), zt = -cinj * zl;
      put_split(tck::kBLh, tck::kBLl, NO + 2 * p, m, zl.real());
      put_split(tck::kBLh, tck::kBLl, NO + 2 * p + 1, m, zl.imag());
      put_split(tck::kBTh, tck::kBTl, NO + 2 * p, m, zt.real());
      put_split(tck::kBTh, tck::kBTl, NO + 2 * p + 1, m, zt.imag());
    }
  for (int p = 0; p < nord; ++p) {
    const double w = ords[p].omega;
    for (int t = 0; t < 32; ++t) {
      const cd v = zpow(alpha, w, 128.0 * t);
      const float f2[2] = {static_cast<float>(v.real()), static_cast<float>(v.imag())};
      std::memcpy(&img[tck::kZ128 + (p * 32 + t) * 8], f2, 8);
    }
    for (int k = 0; k < 6; ++k) {
      const cd v = zpow(alpha, w, k == 0 ? 32.0 : 128.0 * (1 << (k - 1)));
      const float f2[2] = {static_cast<float>(v.real()), static_cast<float>(v.imag())};
      std::memcpy(&img[tck::kZs + (p * 8 + k) * 8], f2, 8);
    }
    const cd zt = zpow(alpha, w, static_cast<double>(tck::kTile));
    const double d2[2] = {zt.real(), zt.imag()};
    std::memcpy(&img[tck::kZd + p * 16], d2, 16);
  }
  std::memset(&sc, 0, sizeof(sc));
  sc.lo = lo;
  sc.K = K;
  sc.rl = static_cast<int>(((lo + K) % 4 + 4) % 4);
  sc.rt = static_cast<int>(((lo - K) % 4 + 4) % 4);
  sc.warm_tiles = static_cast<int>((2LL * K + tck::kTile - 1) / tck::kTile);
  {
    // leading warm-up tiles of a unit's first segment whose lead samples j = lo + o + K
    // are all < 0: the zeros before the warm start (Z positions) then the boundary value
    // v; state after them = v * sum_{e < E} z^e with E = 4096 skip - Z
    const long long W = sc.warm_tiles, jfirst = lo + K - W * tck::kTile;
    const long long skip = jfirst < 0 ? std::min(W, (-jfirst) / tck::kTile) : 0;
    const long long Z = W * tck::kTile - 2LL * K, E = skip * tck::kTile - Z;
    sc.skip0 = static_cast<int>(skip);
    for (int p = 0; p < nord; ++p) {
      cd g(0.0, 0.0);
      if (E > 0) {
        const cd z = zpow(alpha, ords[p].omega, 1.0), zE = zpow(alpha, ords[p].omega, static_cast<double>(E));
        g = std::abs(1.0 - z) < 1e-12 ? cd(static_cast<double>(E), 0.0) : (1.0 - zE) / (1.0 - z);
      }
      if (!std::isfinite(g.real()) || !std::isfinite(g.imag()))
        fail(SFTGPU_EINVAL, "attenuation alpha*K too large for the requested precision");
      sc.g0[p] = make_double2(g.real(), g.imag());
    }
  }
  // every table must be finite in its own precision (fp32 operands and scan constants,
  // fp64 carry tables)
  auto finite = [&](size_t a, size_t e, bool dbl) {
    for (size_t i = a; i < e; i += dbl ? 8 : 4) {
      double v;
      if (dbl) {
        std::memcpy(&v, &img[i], 8);
      } else {
        float f;
        std::memcpy(&f, &img[i], 4);
        v = f;
      }
      if (!std::isfinite(v)) return false;
    }
    return true;
  };
  if (!finite(0, tck::kZd, false) || !finite(tck::kZd, tck::kImage, true))
    fail(SFTGPU_EINVAL, "attenuation alpha*K too large for the requested precision");
}

// Fixed chunking of every scale's units and the global chunk / cost prefixes (TcGeom):
// chunks of at most max(256, 16 W) output tiles (warm-up <= 1/16 of a long chunk); a unit
// that short stays whole. Depends on the specs and the output count only.
void tc_geometry(tck::TcParams& P, const std::vector<tck::TcScale>& scales) {
  long long cbase = 0, wbase = 0;
  for (size_t i = 0; i < scales.size(); ++i) {
    const tck::TcScale& sc = scales[i];
    if (sc.lo < INT32_MIN / 2 || sc.lo > INT32_MAX / 2 || sc.warm_tiles > 255)
      fail(SFTGPU_EINVAL, "tensor-core plan geometry out of range");
    const long long T = P.tiles_unit, cmax = std::max<long long>(256, 16LL * sc.warm_tiles);
    const long long nc = (T + cmax - 1) / cmax, L = (T + nc - 1) / nc;
    tck::TcGeom& G = P.geo[i];
    G.lo = static_cast<int>(sc.lo);
    G.K = sc.K;
    G.rl = static_cast<unsigned char>(sc.rl);
    G.rt = static_cast<unsigned char>(sc.rt);
    G.warm = static_cast<unsigned char>(sc.warm_tiles);
    G.skip0 = static_cast<unsigned char>(sc.skip0);
    G.nc = static_cast<int>(nc);
    G.L = static_cast<int>(L);
    G.cbase = static_cast<int>(cbase);
    G.wbase = static_cast<int>(wbase);
    cbase += nc * P.nsig;
    wbase += (T + nc * sc.warm_tiles - sc.skip0) * P.nsig;
    if (cbase >= (1LL << 31) || wbase >= (1LL << 31)) fail(SFTGPU_EINVAL, "tensor-core plan too large");
  }
  P.total_chunks = static_cast<int>(cbase);
  P.total_cost = static_cast<int>(wbase);
}

// Uploads the images and scale descriptors of a K4 plan and fixes its launch geometry:
// units = signals x scales (scale-major), one persistent CTA per SM over contiguous,
// balanced ranges of output tiles.
void tc_finish(sftgpu_plan* pl, const std::vector<std::vector<unsigned char>>& imgs,
               std::vector<tck::TcScale>& scales, long long nsig, int nord, bool cplx) {
  const size_t ns = scales.size();
  cuda_check(cudaMalloc(&pl->d_tc_image, ns * tck::kImage), "cudaMalloc tc images");
  for (size_t i = 0; i < ns; ++i) {
    cuda_check(cudaMemcpy(static_cast<unsigned char*>(pl->d_tc_image) + i * tck::kImage, imgs[i].data(), tck::kImage,
                          cudaMemcpyHostToDevice),
               "copy tc image");
    scales[i].image = reinterpret_cast<const uint4*>(static_cast<unsigned char*>(pl->d_tc_image) + i * tck::kImage);
  }
  cuda_check(cudaMalloc(&pl->d_tc_scales, ns * sizeof(tck::TcScale)), "cudaMalloc tc scales");
  cuda_check(cudaMemcpy(pl->d_tc_scales, scales.data(), ns * sizeof(tck::TcScale), cudaMemcpyHostToDevice),
             "copy tc scales");
  tck::TcParams& P = pl->tcp;
  std::memset(&P, 0, sizeof(P));
  P.n = pl->n;
  P.count = pl->count;
  P.tiles_unit = static_cast<int>((pl->count + tck::kTile - 1) / tck::kTile);
  P.nsig = static_cast<int>(nsig);
  P.n_scales = static_cast<int>(ns);
  P.scales = pl->d_tc_scales;
  if (ns > static_cast<size_t>(tck::kMaxScales)) fail(SFTGPU_EINVAL, "too many scales for one tensor-core launch");
  tc_geometry(P, scales);
  P.boundary = pl->boundary;
  P.nord = nord;
  P.cplx = cplx ? 1 : 0;
  pl->tc_warm = scales[0].warm_tiles;
  pl->tc_grid = static_cast<int>(std::min<long long>(sftk::sm_count(), P.total_chunks));
  pl->tc = 1;
}

bool build_tc(sftgpu_plan* pl, const Lowered& lw, bool force) {
  cd cinj;
  if (!tc_eligible(pl, lw, force, &cinj)) return false;
  if (!force) {
    // auto: K4 once the transform spans >= 4 tiles per SM (SFTGPU_NO_TC=1 keeps K1)
    const char* env = std::getenv("SFTGPU_NO_TC");
    if (env && env[0] == '1') return false;
    const long long tiles = pl->batch * ((pl->count + tck::kTile - 1) / tck::kTile);
    if (tiles < 4LL * sftk::sm_count()) return false;
  }
  std::vector<std::vector<unsigned char>> imgs(1);
  std::vector<tck::TcScale> scales(1);
  tc_build_scale(lw, cinj, pl->lo, imgs[0], scales[0]);
  tc_finish(pl, imgs, scales, pl->batch, static_cast<int>(lw.orders.size()), lw.complex_out);
  return true;
}

Lowered lower_spec(const sftb::Spec& s) {
  Lowered lw;
  lw.alpha = s.alpha;
  switch (s.kind) {
    case sftb::TKind::Gauss:
    case sftb::TKind::GaussD:
    case sftb::TKind::GaussDD: {
      // proj/src/transforms.cpp:279-335
      const sftb::Bundle& b = s.bundle;
      lw.K = b.params.K;
      lw.prefactor = s.n0 == 0 ? 1.0 : std::exp(-s.alpha * s.alpha / (4.0 * b.params.gamma()));
      for (int p = 0; p <= b.P; ++p) {
        double wc = 0.0, ws = 0.0;
        const double ap = b.a[p], bp = p >= 1 ? b.b[p - 1] : 0.0, dp = b.d[p];
        if (s.kind == sftb::TKind::Gauss) {
          wc = ap;
        } else if (s.kind == sftb::TKind::GaussD) {
          ws = bp;
          if (s.n0 != 0) wc = -s.alpha * ap;
        } else {
          wc = dp;
          if (s.n0 != 0) {
            wc += s.alpha * s.alpha * ap;
            ws = -2.0 * s.alpha * bp;
          }
        }
        lw.orders.push_back({s.beta * p, wc, ws});
      }
      lw.complex_out = false;
      break;
    }
    case sftb::TKind::MorletDirect: {
      // proj/src/transforms.cpp:337-371 (sin weight only where the sin order exists)
      const sftb::Coeffs& c = s.morlet;
      lw.K = s.mparams.K;
      lw.prefactor = s.n0 == 0 ? 1.0 : std::exp(-s.alpha * s.alpha / (4.0 * s.mparams.gamma()));
      size_t si = 0;
      for (size_t ci = 0; ci < c.grid.cos_p.size(); ++ci) {
        const int p = c.grid.cos_p[ci];
        cd ws(0.0, 0.0);
        if (si < c.grid.sin_p.size() && c.grid.sin_p[si] == p) ws = c.sc[si++];
        lw.orders.push_back({s.beta * p, c.cc[ci], ws});
      }
      lw.complex_out = true;
      break;
    }
    case sftb::TKind::MorletMultiply: {
      // proj/src/transforms.cpp:373-428
      const sftb::Coeffs& e = s.envelope;
      const sftb::MorletP& mp = s.mparams;
      lw.K = mp.K;
      lw.prefactor = s.n0 == 0 ? 1.0 : std::exp(-s.alpha * s.alpha / (4.0 * mp.gamma()));
      const int P = s.max_order;
      const cd carrier = s.n0 == 0 ? cd(1.0, 0.0)
                                   : cd(std::cos(mp.xi * s.n0 / mp.sigma), std::sin(mp.xi * s.n0 / mp.sigma));
      for (int p = -P; p <= P; ++p) {
        const double ap = e.cc[std::abs(p)].real();
        const double apr = p == 0 ? ap : 0.5 * ap;
        lw.orders.push_back({mp.xi / mp.sigma + s.beta * p, carrier * apr, carrier * apr * cd(0, 1)});
      }
      for (int p = 0; p <= P; ++p)
        lw.orders.push_back({s.beta * p, cd(-mp.kappa() * e.cc[p].real(), 0.0), cd(0.0, 0.0)});
      lw.complex_out = true;
      break;
    }
    default: fail(SFTGPU_EINVAL, "lower_spec: not an SFT transform kind");
  }
  // Orders whose combine weights are below fp64 resolution of the largest weight add
  // nothing representable to the output, in either precision: the reference still
  // sums them (its result is unchanged by them), the kernel skips them. This is the
  // multiplication method's kappa correction once e^{-xi^2/2} < 2^-63 (xi >= 9.4).
  double wmax = 0.0;
  for (const Order& o : lw.orders) wmax = std::max({wmax, std::abs(o.wc), std::abs(o.ws)});
  const double floor_w = std::ldexp(wmax, -63);
  std::vector<Order> kept;
  for (const Order& o : lw.orders)
    if (std::max(std::abs(o.wc), std::abs(o.ws)) > floor_w) kept.push_back(o);
  if (!kept.empty()) lw.orders.swap(kept);
  return lw;
}

// ---------------------------------------------------------------- C struct <-> internal
sftb::Options to_options(const sftgpu_options* o) {
  sftb::Options r;
  if (!o) return r;
  r.has_K = o->has_half_width != 0;
  r.K = o->half_width;
  r.has_beta = o->has_beta != 0;
  r.beta = o->beta;
  r.tune = o->tune_beta != 0;
  r.has_ps = o->has_ps != 0;
  r.ps = o->ps;
  r.strategy = o->strategy;
  r.precision = o->precision;
  return r;
}

void coeffs_to_c(const sftb::Coeffs& c, sftgpu_coeffs* o) {
  std::memset(o, 0, sizeof(*o));
  if (c.grid.cos_p.size() > SFTGPU_MAX_COEFFS || c.grid.sin_p.size() > SFTGPU_MAX_COEFFS)
    fail(SFTGPU_EINVAL, "too many coefficients for sftgpu_coeffs");
  o->kind = c.kind;
  o->half_width = c.grid.K;
  o->beta = c.grid.beta;
  o->n_cos = static_cast<int>(c.grid.cos_p.size());
  o->n_sin = static_cast<int>(c.grid.sin_p.size());
  for (int i = 0; i < o->n_cos; ++i) {
    o->cos_orders[i] = c.grid.cos_p[i];
    o->cos_coeffs[2 * i] = c.cc[i].real();
    o->cos_coeffs[2 * i + 1] = c.cc[i].imag();
  }
  for (int i = 0; i < o->n_sin; ++i) {
    o->sin_orders[i] = c.grid.sin_p[i];
    o->sin_coeffs[2 * i] = c.sc[i].real();
    o->sin_coeffs[2 * i + 1] = c.sc[i].imag();
  }
  o->fit_rmse_percent = c.fit_rmse;
  o->sigma = c.sigma;
  o->xi = c.xi;
  o->n0 = c.n0;
}

sftb::Coeffs coeffs_from_c(const sftgpu_coeffs* o) {
  sftb::Coeffs c;
  c.kind = o->kind;
  std::vector<int> co(o->cos_orders, o->cos_orders + o->n_cos), so(o->sin_orders, o->sin_orders + o->n_sin);
  c.grid = sftb::Grid(o->half_width, o->beta, co, so);
  for (int i = 0; i < o->n_cos; ++i) c.cc.emplace_back(o->cos_coeffs[2 * i], o->cos_coeffs[2 * i + 1]);
  for (int i = 0; i < o->n_sin; ++i) c.sc.emplace_back(o->sin_coeffs[2 * i], o->sin_coeffs[2 * i + 1]);
  c.fit_rmse = o->fit_rmse_percent;
  c.sigma = o->sigma;
  c.xi = o->xi;
  c.n0 = o->n0;
  return c;
}

void bundle_to_c(const sftb::Bundle& b, sftgpu_gauss_bundle* o) {
  std::memset(o, 0, sizeof(*o));
  if (b.P + 1 > SFTGPU_MAX_COEFFS) fail(SFTGPU_EINVAL, "too many coefficients for sftgpu_gauss_bundle");
  o->sigma = b.params.sigma;
  o->half_width = b.params.K;
  o->beta = b.beta;
  o->max_order = b.P;
  for (size_t i = 0; i < b.a.size(); ++i) o->a[i] = b.a[i];
  for (size_t i = 0; i < b.b.size(); ++i) o->b[i] = b.b[i];
  for (size_t i = 0; i < b.d.size(); ++i) o->d[i] = b.d[i];
  o->fit_rmse_g = b.rmse_g;
  o->fit_rmse_gd = b.rmse_gd;
  o->fit_rmse_gdd = b.rmse_gdd;
}

sftb::Bundle bundle_from_c(const sftgpu_gauss_bundle* o) {
  sftb::Bundle b;
  b.params = sftb::GaussP(o->sigma, o->half_width);
  b.beta = o->beta;
  b.P = o->max_order;
  b.a.assign(o->a, o->a + o->max_order + 1);
  b.b.assign(o->b, o->b + o->max_order);
  b.d.assign(o->d, o->d + o->max_order + 1);
  b.rmse_g = o->fit_rmse_g;
  b.rmse_gd = o->fit_rmse_gd;
  b.rmse_gdd = o->fit_rmse_gdd;
  return b;
}

void spec_to_c(const sftb::Spec& s, sftgpu_spec* o) {
  std::memset(o, 0, sizeof(*o));
  o->kind = static_cast<int>(s.kind);
  if (s.has_gauss) {
    o->sigma = s.gparams.sigma;
    o->half_width = s.gparams.K;
  }
  if (s.has_morlet) {
    o->sigma = s.mparams.sigma;
    o->xi = s.mparams.xi;
    o->half_width = s.mparams.K;
  }
  o->max_order = s.max_order;
  o->ps = s.ps;
  o->pd = s.pd;
  o->beta = s.beta;
  o->n0 = s.n0;
  o->alpha = s.alpha;
  o->strategy = s.strategy;
  o->precision = s.precision;
  std::strncpy(o->abbreviation, s.abbrev.c_str(), sizeof(o->abbreviation) - 1);
  o->kernel_rmse_percent = s.kernel_rmse;
  if (s.has_bundle) bundle_to_c(s.bundle, &o->gauss);
  if (s.has_mcoef) coeffs_to_c(s.morlet, &o->morlet);
  if (s.has_env) coeffs_to_c(s.envelope, &o->envelope);
}

sftb::Spec spec_from_c(const sftgpu_spec* o) {
  if (!o) fail(SFTGPU_EINVAL, "null spec");
  sftb::Spec s;
  s.kind = static_cast<sftb::TKind>(o->kind);
  switch (s.kind) {
    case sftb::TKind::Gauss:
    case sftb::TKind::GaussD:
    case sftb::TKind::GaussDD:
      s.has_gauss = true;
      s.gparams = sftb::GaussP(o->sigma, o->half_width);
      s.bundle = bundle_from_c(&o->gauss);
      s.has_bundle = true;
      break;
    case sftb::TKind::MorletDirect:
      s.has_morlet = true;
      s.mparams = sftb::MorletP(o->sigma, o->xi, o->half_width);
      s.morlet = coeffs_from_c(&o->morlet);
      s.has_mcoef = true;
      break;
    case sftb::TKind::MorletMultiply:
      s.has_morlet = true;
      s.mparams = sftb::MorletP(o->sigma, o->xi, o->half_width);
      s.envelope = coeffs_from_c(&o->envelope);
      s.has_env = true;
      break;
    case sftb::TKind::TruncGauss:
      s.has_gauss = true;
      s.gparams = sftb::GaussP(o->sigma, o->half_width);
      break;
    case sftb::TKind::TruncMorlet:
      s.has_morlet = true;
      s.mparams = sftb::MorletP(o->sigma, o->xi, o->half_width);
      break;
    default: fail(SFTGPU_EINVAL, "unknown transform kind");
  }
  s.max_order = o->max_order;
  s.ps = o->ps;
  s.pd = o->pd;
  s.beta = o->beta;
  s.n0 = o->n0;
  s.alpha = o->alpha;
  s.strategy = o->strategy;
  s.precision = o->precision;
  s.abbrev = o->abbreviation;
  s.kernel_rmse = o->kernel_rmse_percent;
  return s;
}

// TMA view of the transform output for K4's epilogue: complex [batch][rows][2 halves][32
// floats], real [batch][rows][32 floats], rows = 32-position chunks. Requires whole
// chunks per signal (count % 32 == 0) and 16-byte aligned rows; otherwise K4 stores with
// regular 16-byte stores.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

bool make_out_map(sftgpu_plan* pl, void* out, long long ld_out, long long nsig, CUtensorMap* map) {
  const tck::TcParams& P = pl->tcp;
  const int cw = P.cplx ? 2 : 1;
  if (pl->count % tck::kQ != 0 || reinterpret_cast<uintptr_t>(out) % 16 != 0) return false;
  if ((static_cast<unsigned long long>(ld_out) * cw * sizeof(float)) % 16 != 0) return false;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  const cuuint64_t rows = static_cast<cuuint64_t>(pl->count / tck::kQ);
  const cuuint64_t sig_stride = static_cast<cuuint64_t>(ld_out) * cw * sizeof(float);
  CUresult r;
  if (cw == 2) {
    const cuuint64_t dims[4] = {32, 2, rows, static_cast<cuuint64_t>(nsig)};
    const cuuint64_t strides[3] = {128, 256, sig_stride};
    const cuuint32_t box[4] = {32, 1, 128, 1}, es[4] = {1, 1, 1, 1};
    r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[3] = {32, rows, static_cast<cuuint64_t>(nsig)};
    const cuuint64_t strides[2] = {128, sig_stride};
    const cuuint32_t box[3] = {32, 128, 1}, es[3] = {1, 1, 1};
    r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  return r == CUDA_SUCCESS;
}

// TMA view of the input for K4's loader: [signal][row][64 samples] with rows 32 samples
// (128 B) apart, i.e. overlapping rows, so a box of 32 samples x 129 rows may start at
// any 16-byte aligned sample. Needs a 16-byte aligned base and signal stride; rows are
// limited so that every element of the view lies inside the signal.
bool make_in_map(sftgpu_plan* pl, const void* x, long long ld_x, long long nsig, CUtensorMap* map,
                 long long* rows_out) {
  *rows_out = 0;
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0 || (static_cast<unsigned long long>(ld_x) * sizeof(float)) % 16 != 0)
    return false;
  if (pl->n < 64 + 32) return false;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  const long long rows = (pl->n - 64) / 32 + 1;
  const cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(nsig)};
  const cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(ld_x) * sizeof(float)};
  const cuuint32_t box[3] = {32, tck::kBoxRows, 1}, es[3] = {1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(x), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  *rows_out = rows;
  return true;
}

long long* g_tc_trace = nullptr;    // diagnostics: sftgpu_debug_set_tc_trace
long long* g_scan_trace = nullptr;  // diagnostics: sftgpu_debug_set_scan_trace

// K4 over the plan's signals, or over the first `nsig` signals at x / out (sub-batches of
// the pipelined host path: same geometry, fewer items)
void run_tc(sftgpu_plan* pl, const void* x, long long ld_x, void* out, long long ld_out, cudaStream_t st,
            long long nsig = -1) {
  tck::TcParams& C = pl->tcp;
  tck::TcParams P;
  // output rows: units (signals x scales); input rows: signals
  const long long rows = static_cast<long long>(C.nsig) * C.n_scales;
  if (nsig < 0 || nsig == C.nsig) {
    if (pl->tc_map_out != out || pl->tc_map_ld != ld_out) {
      C.use_tma = make_out_map(pl, out, ld_out, rows, &C.out_map) ? 1 : 0;
      pl->tc_map_out = out;
      pl->tc_map_ld = ld_out;
    }
    if (pl->tc_map_in != x || pl->tc_map_in_ld != ld_x) {
      C.use_tma_in = make_in_map(pl, x, ld_x, C.nsig, &C.in_map, &C.in_rows) ? 1 : 0;
      pl->tc_map_in = x;
      pl->tc_map_in_ld = ld_x;
    }
    P = C;
  } else {  // sub-batch of a single-scale plan
    P = C;
    P.nsig = static_cast<int>(nsig);
    std::vector<tck::TcScale> one(1);
    one[0].lo = P.geo[0].lo;
    one[0].K = P.geo[0].K;
    one[0].rl = P.geo[0].rl;
    one[0].rt = P.geo[0].rt;
    one[0].warm_tiles = P.geo[0].warm;
    one[0].skip0 = P.geo[0].skip0;
    tc_geometry(P, one);
    P.use_tma = make_out_map(pl, out, ld_out, nsig, &P.out_map) ? 1 : 0;
    P.use_tma_in = make_in_map(pl, x, ld_x, nsig, &P.in_map, &P.in_rows) ? 1 : 0;
  }
  P.x = static_cast<const float*>(x);
  P.out = static_cast<float*>(out);
  P.ld_x = ld_x;
  P.ld_out = ld_out;
  const size_t rowb = static_cast<size_t>(ld_out) * sizeof(float) * (P.cplx ? 2 : 1);
  P.vec_ok = (reinterpret_cast<uintptr_t>(out) % 16 == 0 && rowb % 16 == 0) ? 1 : 0;
  if (const char* e = std::getenv("SFTGPU_TC_NO_TMA")) P.use_tma = e[0] == '1' ? 0 : P.use_tma;
  if (const char* e = std::getenv("SFTGPU_TC_NO_TMA_IN")) P.use_tma_in = e[0] == '1' ? 0 : P.use_tma_in;
  P.trace = g_tc_trace;
  if (const char* e = std::getenv("SFTGPU_TC_DBG")) P.dbg = std::atoi(e);
  const int grid = static_cast<int>(std::min<long long>(pl->tc_grid, P.total_chunks));
  cuda_check(tck::launch_tc(P, grid, st), "sft_tc_kernel launch");
}

template <typename T>
void run_groups(sftgpu_plan* pl, const void* x, long long ld_x, void* out, void* out_s, long long ld_out,
                int accumulate_first, cudaStream_t st) {
  if (pl->tc) {
    if constexpr (std::is_same<T, float>::value) run_tc(pl, x, ld_x, out, ld_out, st);
    return;
  }
  const bool lb = !pl->seq && pl->d_ctrl != nullptr;
  const bool capturing = lb && lb_capturing(st);
  if (lb) lb_order_begin(pl, st, capturing);
  for (size_t gi = 0; gi < pl->groups.size(); ++gi) {
    Group& g = pl->groups[gi];
    sftk::ScanParams<T> P = params_of<T>(g);
    P.x = static_cast<const T*>(x);
    P.n = pl->n;
    P.ld_x = ld_x;
    P.out = static_cast<T*>(out);
    P.out_s = static_cast<T*>(out_s);
    P.ld_out = ld_out;
    P.ord_stride = pl->batch * ld_out;
    P.lo = pl->lo;
    P.count = pl->count;
    P.K = pl->K;
    P.boundary = pl->boundary;
    P.accumulate = (gi > 0 && !pl->is_components) ? 1 : accumulate_first;
    {
      const size_t rowb = static_cast<size_t>(ld_out) * sizeof(T) * (pl->mode == sftk::kModeComplex ? 2 : 1);
      P.vec_ok = (reinterpret_cast<uintptr_t>(out) % 16 == 0 && rowb % 16 == 0) ? 1 : 0;
    }
    P.tiles_per_signal = pl->tiles_per_signal;
    P.warm_tiles = pl->warm_tiles;
    P.total_tiles = pl->total_tiles;
    P.chunk_len = pl->chunk_len;
    P.n_chunks = pl->n_chunks;
    P.lb_D = static_cast<int>((2LL * pl->K) / pl->TT);
    {
      const long long r = 2LL * pl->K - static_cast<long long>(P.lb_D) * pl->TT;
      P.lb_sfx = static_cast<int>(pl->TT - r);
    }
    P.ctrl = pl->d_ctrl;
    P.trace = g_scan_trace;
    P.flags = pl->d_flags;
    P.agg = pl->d_agg;
    P.incl = pl->d_incl;
    if (pl->is_components && gi > 0) {
      // later component groups write further down the [order] axis
      long long skip = 0;
      for (size_t k = 0; k < gi; ++k) skip += pl->groups[k].nord;
      P.out = static_cast<T*>(out) + skip * P.ord_stride;
      P.out_s = static_cast<T*>(out_s) + skip * P.ord_stride;
    }
    launch_scan<T>(pl, g, P, st);
    cuda_check(cudaGetLastError(), "sft_scan_kernel launch");
  }
  if (lb) lb_order_end(pl, st, capturing);
}

// GCT3/MCT3 (proj/src/transforms.cpp:430-442): fp64 accumulation into a complex
// scratch row, then copied into the output layout (real for GCT3, complex for MCT3).
// Like the reference, the direct path always computes in double precision.
void run_conv(sftgpu_plan* pl, const void* x, long long ld_x, void* out, long long ld_out, cudaStream_t st) {
  constexpr int BO = 256, BT = 1024;
  const long long blocks = (pl->n + BO - 1) / BO;
  for (long long b = 0; b < pl->batch; ++b) {
    const double* xb = static_cast<const double*>(x) + b * ld_x;
    sftk::truncated_conv_kernel<double, BO, BT><<<blocks, BO, 0, st>>>(xb, pl->n, pl->boundary, pl->d_taps,
                                                                       pl->n_taps, pl->tap_lo, pl->d_conv_tmp);
    cuda_check(cudaGetLastError(), "truncated_conv_kernel launch");
    if (pl->mode == sftk::kModeComplex) {
      double* ob = static_cast<double*>(out) + 2 * b * ld_out;
      cuda_check(cudaMemcpyAsync(ob, pl->d_conv_tmp, pl->n * sizeof(double2), cudaMemcpyDeviceToDevice, st),
                 "conv copy");
    } else {
      double* ob = static_cast<double*>(out) + b * ld_out;
      cuda_check(cudaMemcpy2DAsync(ob, sizeof(double), pl->d_conv_tmp, sizeof(double2), sizeof(double), pl->n,
                                   cudaMemcpyDeviceToDevice, st),
                 "conv real copy");
    }
  }
}

}  // namespace

void sftgpu_set_error(const std::string& m) { g_err = m; }

extern "C" {

const char* sftgpu_last_error(void) { return g_err.c_str(); }
const char* sftgpu_version(void) { return "sftgpu 0.1.0 (sm_100a)"; }

int sftgpu_parse_abbreviation(const char* abbrev, int* kind, int* n0, int* order) {
  return guarded([&] {
    if (!abbrev) fail(SFTGPU_EINVAL, "null abbreviation");
    const sftb::Abbrev a = sftb::parse_abbreviation(abbrev);
    *kind = static_cast<int>(a.kind);
    *n0 = a.n0;
    *order = a.order;
  });
}

int sftgpu_encode_abbreviation(int kind, int n0, int order, char* out, int out_len) {
  return guarded([&] {
    const std::string s = sftb::encode_abbreviation(static_cast<sftb::TKind>(kind), n0, order);
    if (static_cast<int>(s.size()) + 1 > out_len) fail(SFTGPU_EINVAL, "buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
}

int sftgpu_make_transform_spec(const char* abbrev, double sigma, double xi, const sftgpu_options* opt,
                               sftgpu_spec* out) {
  return guarded([&] {
    if (!abbrev) fail(SFTGPU_EINVAL, "null abbreviation");
    spec_to_c(sftb::make_transform_spec(abbrev, sigma, xi, to_options(opt)), out);
  });
}

int sftgpu_make_gauss_spec(double sigma, int gauss_kind, int max_order, int n0, const sftgpu_options* opt,
                           sftgpu_spec* out) {
  return guarded([&] {
    spec_to_c(sftb::make_gauss_spec(sigma, static_cast<sftb::GKind>(gauss_kind), max_order, n0, to_options(opt)),
              out);
  });
}

int sftgpu_make_morlet_direct_spec(double sigma, double xi, int pd, int n0, const sftgpu_options* opt,
                                   sftgpu_spec* out) {
  return guarded([&] { spec_to_c(sftb::make_morlet_direct_spec(sigma, xi, pd, n0, to_options(opt)), out); });
}

int sftgpu_make_morlet_multiply_spec(double sigma, double xi, int pm, int n0, const sftgpu_options* opt,
                                     sftgpu_spec* out) {
  return guarded([&] { spec_to_c(sftb::make_morlet_multiply_spec(sigma, xi, pm, n0, to_options(opt)), out); });
}

int sftgpu_effective_kernel(const sftgpu_spec* spec, double* taps, int64_t cap, int64_t* n_taps, int64_t* tap_lo) {
  return guarded([&] {
    const sftb::Taps t = sftb::effective_kernel(spec_from_c(spec));
    *n_taps = static_cast<int64_t>(t.taps.size());
    *tap_lo = t.lo;
    if (taps) {
      if (cap < static_cast<int64_t>(t.taps.size())) fail(SFTGPU_EINVAL, "taps buffer too small");
      for (size_t i = 0; i < t.taps.size(); ++i) {
        taps[2 * i] = t.taps[i].real();
        taps[2 * i + 1] = t.taps[i].imag();
      }
    }
  });
}

int sftgpu_fit_mmse(const double* target, int K, double beta, int n_cos, const int* cos_orders, int n_sin,
                    const int* sin_orders, int kind, sftgpu_coeffs* out) {
  return guarded([&] {
    const sftb::Grid g(K, beta, std::vector<int>(cos_orders, cos_orders + n_cos),
                       std::vector<int>(sin_orders, sin_orders + n_sin));
    std::vector<cd> t(2 * static_cast<size_t>(K) + 1);
    for (size_t i = 0; i < t.size(); ++i) t[i] = cd(target[2 * i], target[2 * i + 1]);
    coeffs_to_c(sftb::fit_mmse(t, g, kind), out);
  });
}

int sftgpu_fit_gaussian_bundle(double sigma, int K, int P, double beta, sftgpu_gauss_bundle* out) {
  return guarded([&] { bundle_to_c(sftb::fit_gaussian_bundle(sftb::GaussP(sigma, K), P, beta), out); });
}

int sftgpu_fit_morlet_direct(double sigma, double xi, int K, int ps, int pd, double beta, int n0,
                             sftgpu_coeffs* out) {
  return guarded([&] { coeffs_to_c(sftb::fit_morlet_direct(sftb::MorletP(sigma, xi, K), ps, pd, beta, n0), out); });
}

int sftgpu_fit_morlet_envelope(double sigma, double xi, int K, int P, double beta, sftgpu_coeffs* out) {
  return guarded([&] { coeffs_to_c(sftb::fit_morlet_envelope(sftb::MorletP(sigma, xi, K), P, beta), out); });
}

int sftgpu_select_optimal_ps(double sigma, double xi, int K, int pd, int n0, int* ps) {
  return guarded([&] { *ps = sftb::select_optimal_ps(sftb::MorletP(sigma, xi, K), pd, n0); });
}

int sftgpu_morlet_direct_kernel_rmse(double sigma, double xi, int K, int ps, int pd, int n0, double* rmse) {
  return guarded([&] { *rmse = sftb::morlet_direct_kernel_rmse(sftb::MorletP(sigma, xi, K), ps, pd, n0); });
}

int sftgpu_morlet_multiply_kernel_rmse(double sigma, double xi, int K, int pm, int n0, double* rmse) {
  return guarded([&] { *rmse = sftb::morlet_multiply_kernel_rmse(sftb::MorletP(sigma, xi, K), pm, n0); });
}

int sftgpu_gauss_kernel_rmse(const sftgpu_gauss_bundle* b, int kind, int n0, double* rmse) {
  return guarded([&] { *rmse = sftb::gauss_kernel_rmse(bundle_from_c(b), static_cast<sftb::GKind>(kind), n0); });
}

int sftgpu_tune_beta_gauss(double sigma, int K, int P, int n0, double* beta, double* rmse) {
  return guarded([&] {
    const sftb::BetaTune r = sftb::tune_beta_gauss(sftb::GaussP(sigma, K), P, n0);
    *beta = r.beta;
    *rmse = r.rmse;
  });
}

int sftgpu_tune_beta(double (*rmse_of_beta)(double beta, void* user), void* user, int half_width, double* beta,
                     double* rmse) {
  return guarded([&] {
    if (!rmse_of_beta || !beta || !rmse) fail(SFTGPU_EINVAL, "null argument");
    if (half_width < 1) fail(SFTGPU_EINVAL, "tune_beta: K must be >= 1");
    const sftb::BetaTune r = sftb::tune_beta_callback(rmse_of_beta, user, half_width);
    *beta = r.beta;
    *rmse = r.rmse;
  });
}

int sftgpu_reconstruct(const sftgpu_coeffs* coeffs, const double* points, int64_t n, double* out_re_im) {
  return guarded([&] {
    if (!coeffs || (!points && n > 0) || (!out_re_im && n > 0)) fail(SFTGPU_EINVAL, "null argument");
    const sftb::Coeffs c = coeffs_from_c(coeffs);
    const std::vector<double> q(points, points + n);
    const std::vector<cd> v = sftb::reconstruct(c, q);
    for (int64_t i = 0; i < n; ++i) {
      out_re_im[2 * i] = v[i].real();
      out_re_im[2 * i + 1] = v[i].imag();
    }
  });
}

int sftgpu_write_coefficient_sets(const char* path, const sftgpu_coeffs* sets, int n_sets) {
  return guarded([&] {
    if (!path || (!sets && n_sets > 0)) fail(SFTGPU_EINVAL, "null argument");
    std::vector<sftb::Coeffs> v;
    for (int i = 0; i < n_sets; ++i) v.push_back(coeffs_from_c(&sets[i]));
    const std::string text = sftb::write_coefficient_sets(v);
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(SFTGPU_EINVAL, std::string("cannot open coefficient file: ") + path);
    const size_t w = std::fwrite(text.data(), 1, text.size(), f);
    std::fclose(f);
    if (w != text.size()) fail(SFTGPU_EINTERNAL, "short write to coefficient file");
  });
}

int sftgpu_read_coefficient_sets(const char* path, sftgpu_coeffs* sets, int capacity, int* n_sets) {
  return guarded([&] {
    if (!path || !n_sets) fail(SFTGPU_EINVAL, "null argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) fail(SFTGPU_EINVAL, std::string("cannot open coefficient file: ") + path);
    std::string text;
    char buf[65536];
    size_t r;
    while ((r = std::fread(buf, 1, sizeof(buf), f)) > 0) text.append(buf, r);
    std::fclose(f);
    const std::vector<sftb::Coeffs> v = sftb::read_coefficient_sets(text);
    *n_sets = static_cast<int>(v.size());
    if (sets) {
      if (capacity < *n_sets) fail(SFTGPU_EINVAL, "coefficient set buffer too small");
      for (size_t i = 0; i < v.size(); ++i) coeffs_to_c(v[i], &sets[i]);
    }
  });
}

int sftgpu_make_morlet_direct_spec_from_coeffs(const sftgpu_coeffs* set, int precision, int strategy,
                                               int recompute_rmse, sftgpu_spec* out) {
  return guarded([&] {
    if (!set || !out) fail(SFTGPU_EINVAL, "null argument");
    spec_to_c(sftb::morlet_direct_spec_from_coeffs(coeffs_from_c(set), precision, strategy, recompute_rmse != 0),
              out);
  });
}

int sftgpu_transform_plan_create(const sftgpu_spec* spec, int64_t n, int64_t batch, int boundary,
                                 sftgpu_plan** plan) {
  return sftgpu_transform_plan_create_range(spec, n, batch, boundary, 0, n, plan);
}

int sftgpu_transform_plan_create_range(const sftgpu_spec* spec, int64_t n, int64_t batch, int boundary,
                                       int64_t out_begin, int64_t out_count, sftgpu_plan** plan) {
  return sftgpu_transform_plan_create_ex(spec, n, batch, boundary, out_begin, out_count, 0, plan);
}

int sftgpu_transform_plan_create_ex(const sftgpu_spec* spec, int64_t n, int64_t batch, int boundary,
                                    int64_t out_begin, int64_t out_count, int mode_hint, sftgpu_plan** plan) {
  return guarded([&] {
    if (mode_hint < 0 || mode_hint > 3)
      fail(SFTGPU_EINVAL, "mode_hint must be 0 (auto), 1 (sequential), 2 (look-back), 3 (tensor cores)");
    if (!plan) fail(SFTGPU_EINVAL, "null plan pointer");
    *plan = nullptr;
    if (n < 1) fail(SFTGPU_EINVAL, "Signal: need at least one sample");
    if (batch < 1) fail(SFTGPU_EINVAL, "batch must be >= 1");
    if (boundary != SFTGPU_BOUNDARY_ZERO && boundary != SFTGPU_BOUNDARY_CLAMP)
      fail(SFTGPU_EINVAL, "unknown boundary policy");
    if (out_begin < 0 || out_count < 1 || out_begin + out_count > n) fail(SFTGPU_EINVAL, "output range outside the signal");
    const sftb::Spec s = spec_from_c(spec);
    require_device();
    auto pl = std::make_unique<sftgpu_plan>();
    cuda_check(cudaGetDevice(&pl->device), "cudaGetDevice");
    pl->precision = s.precision == SFTGPU_SINGLE ? SFTGPU_SINGLE : SFTGPU_DOUBLE;
    pl->n = n;
    pl->batch = batch;
    pl->boundary = boundary;
    if (s.kind == sftb::TKind::TruncGauss || s.kind == sftb::TKind::TruncMorlet) {
      if (out_begin != 0 || out_count != n) fail(SFTGPU_EINVAL, "truncated-convolution plans cover the whole signal");
      const sftb::Taps t = sftb::effective_kernel(s);
      pl->conv = 1;
      pl->mode = s.kind == sftb::TKind::TruncMorlet ? sftk::kModeComplex : sftk::kModeReal;
      pl->precision = SFTGPU_DOUBLE;
      pl->count = n;
      pl->n_taps = static_cast<long long>(t.taps.size());
      pl->tap_lo = t.lo;
      std::vector<double2> h(t.taps.size());
      for (size_t i = 0; i < h.size(); ++i) h[i] = make_double2(t.taps[i].real(), t.taps[i].imag());
      cuda_check(cudaMalloc(&pl->d_taps, h.size() * sizeof(double2)), "cudaMalloc taps");
      cuda_check(cudaMemcpy(pl->d_taps, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice), "copy taps");
      cuda_check(cudaMalloc(&pl->d_conv_tmp, n * sizeof(double2)), "cudaMalloc conv scratch");
      *plan = pl.release();
      return;
    }
    const Lowered lw = lower_spec(s);
    pl->K = lw.K;
    pl->lo = out_begin - static_cast<long long>(s.n0);  // window read at n - n0 (transforms.cpp:287-288)
    pl->count = out_count;
    pl->mode = lw.complex_out ? sftk::kModeComplex : sftk::kModeReal;
    pl->mode_hint = mode_hint == 3 ? 0 : mode_hint;
    if ((mode_hint == 0 || mode_hint == 3) && build_tc(pl.get(), lw, mode_hint == 3)) {
      *plan = pl.release();
      return;
    }
    choose_geometry(pl.get());
    if (pl->precision == SFTGPU_SINGLE)
      build_groups<float>(pl.get(), lw.orders, lw.alpha, lw.prefactor, false);
    else
      build_groups<double>(pl.get(), lw.orders, lw.alpha, lw.prefactor, false);
    alloc_workspace(pl.get());
    *plan = pl.release();
  });
}

int sftgpu_components_plan_create(const sftgpu_config* cfgs, int n_orders, int64_t n, int64_t batch, int boundary,
                                  int64_t lo, int64_t hi, int mode, sftgpu_plan** plan) {
  return guarded([&] {
    if (!plan) fail(SFTGPU_EINVAL, "null plan pointer");
    *plan = nullptr;
    if (!cfgs || n_orders < 1) fail(SFTGPU_EINVAL, "need at least one order");
    if (n < 1) fail(SFTGPU_EINVAL, "Signal: need at least one sample");
    if (batch < 1) fail(SFTGPU_EINVAL, "batch must be >= 1");
    if (boundary != SFTGPU_BOUNDARY_ZERO && boundary != SFTGPU_BOUNDARY_CLAMP)
      fail(SFTGPU_EINVAL, "unknown boundary policy");
    const sftgpu_config& c0 = cfgs[0];
    std::vector<Order> ords;
    for (int i = 0; i < n_orders; ++i) {
      const sftgpu_config& c = cfgs[i];
      // SftConfig::validate (proj/include/sft/engine.hpp:51-59)
      if (c.half_width < 1) fail(SFTGPU_EINVAL, "SftConfig: K must be >= 1");
      if (!(c.beta > 0.0) && c.integer_order) fail(SFTGPU_EINVAL, "SftConfig: beta must be > 0");
      if (c.alpha < 0.0) fail(SFTGPU_EINVAL, "SftConfig: alpha must be >= 0");
      if (c.integer_order && c.p < 0) fail(SFTGPU_EINVAL, "OrderSpec: p must be >= 0");
      if (!c.integer_order && c.strategy != SFTGPU_KERNEL_INTEGRAL)
        fail(SFTGPU_EINVAL, "SftConfig: real-frequency components require the kernel-integral strategy");
      if (c.half_width != c0.half_width || c.alpha != c0.alpha || c.precision != c0.precision)
        fail(SFTGPU_EINVAL, "components plan: orders must share K, alpha and precision");
      ords.push_back({c.integer_order ? c.beta * c.p : c.omega, cd(0, 0), cd(0, 0)});
    }
    // proj/src/engine.cpp:247, :260-269
    if (mode == 1 && c0.alpha != 0.0) fail(SFTGPU_EINVAL, "sft_components: alpha must be 0 (use asft_components)");
    if (mode == 2 && !(c0.alpha > 0.0)) fail(SFTGPU_EINVAL, "asft_components: alpha must be > 0");
    if (lo > hi) fail(SFTGPU_EINVAL, "components_over: empty range");
    require_device();
    auto pl = std::make_unique<sftgpu_plan>();
    cuda_check(cudaGetDevice(&pl->device), "cudaGetDevice");
    pl->is_components = 1;
    pl->precision = c0.precision == SFTGPU_SINGLE ? SFTGPU_SINGLE : SFTGPU_DOUBLE;
    pl->mode = sftk::kModeComps;
    pl->n = n;
    pl->batch = batch;
    pl->boundary = boundary;
    pl->K = c0.half_width;
    pl->lo = lo;
    pl->count = hi - lo + 1;
    choose_geometry(pl.get());
    if (pl->precision == SFTGPU_SINGLE)
      build_groups<float>(pl.get(), ords, c0.alpha, 1.0, true);
    else
      build_groups<double>(pl.get(), ords, c0.alpha, 1.0, true);
    alloc_workspace(pl.get());
    *plan = pl.release();
  });
}

int sftgpu_multiscale_plan_create(const sftgpu_spec* specs, int n_specs, int64_t n, int boundary,
                                  int64_t out_begin, int64_t out_count, sftgpu_plan** plan) {
  return guarded([&] {
    if (!plan) fail(SFTGPU_EINVAL, "null plan pointer");
    *plan = nullptr;
    if (!specs || n_specs < 1 || n_specs > tck::kMaxScales) fail(SFTGPU_EINVAL, "need 1..128 specs");
    if (n < 1) fail(SFTGPU_EINVAL, "Signal: need at least one sample");
    if (boundary != SFTGPU_BOUNDARY_ZERO && boundary != SFTGPU_BOUNDARY_CLAMP)
      fail(SFTGPU_EINVAL, "unknown boundary policy");
    if (out_begin < 0 || out_count < 1 || out_begin + out_count > n) fail(SFTGPU_EINVAL, "output range outside the signal");
    require_device();
    auto pl = std::make_unique<sftgpu_plan>();
    cuda_check(cudaGetDevice(&pl->device), "cudaGetDevice");
    pl->precision = SFTGPU_SINGLE;
    pl->n = n;
    pl->batch = n_specs;
    pl->in_batch = 1;
    pl->boundary = boundary;
    pl->count = out_count;
    std::vector<std::vector<unsigned char>> imgs(n_specs);
    std::vector<tck::TcScale> scales(n_specs);
    int nord = -1;
    bool cplx = false;
    for (int i = 0; i < n_specs; ++i) {
      const sftb::Spec s = spec_from_c(&specs[i]);
      if (s.precision != SFTGPU_SINGLE) fail(SFTGPU_EINVAL, "multi-scale plans are single precision");
      if (s.kind == sftb::TKind::TruncGauss || s.kind == sftb::TKind::TruncMorlet)
        fail(SFTGPU_EINVAL, "multi-scale plans take sliding-transform specs");
      const Lowered lw = lower_spec(s);
      cd cinj;
      tc_eligible(pl.get(), lw, true, &cinj);
      if (i == 0) {
        nord = static_cast<int>(lw.orders.size());
        cplx = lw.complex_out;
        pl->K = lw.K;
        pl->lo = out_begin - static_cast<long long>(s.n0);
        pl->mode = cplx ? sftk::kModeComplex : sftk::kModeReal;
      } else if (static_cast<int>(lw.orders.size()) != nord || lw.complex_out != cplx) {
        fail(SFTGPU_EINVAL, "multi-scale plan: every spec needs the same number of orders and output kind");
      }
      tc_build_scale(lw, cinj, out_begin - static_cast<long long>(s.n0), imgs[i], scales[i]);
    }
    tc_finish(pl.get(), imgs, scales, 1, nord, cplx);
    *plan = pl.release();
  });
}

int sftgpu_transform_execute(sftgpu_plan* pl, const void* x, int64_t ld_x, void* out, int64_t ld_out,
                             void* stream) {
  return guarded([&] {
    if (!pl || pl->is_components) fail(SFTGPU_EINVAL, "not a transform plan");
    if (!x || !out) fail(SFTGPU_EINVAL, "null buffer");
    if (ld_x < pl->n || ld_out < pl->count) fail(SFTGPU_EINVAL, "leading dimension smaller than the row length");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (pl->conv) {
      run_conv(pl, x, ld_x, out, ld_out, st);
      return;
    }
    if (pl->precision == SFTGPU_SINGLE)
      run_groups<float>(pl, x, ld_x, out, nullptr, ld_out, 0, st);
    else
      run_groups<double>(pl, x, ld_x, out, nullptr, ld_out, 0, st);
  });
}

namespace {
size_t plan_in_bytes(const sftgpu_plan* pl) {
  return static_cast<size_t>(pl->n * (pl->in_batch >= 0 ? pl->in_batch : pl->batch)) * elem_size(pl->precision);
}
size_t plan_out_bytes(const sftgpu_plan* pl) {
  return static_cast<size_t>(pl->count * pl->batch) * elem_size(pl->precision) * (pl->mode == sftk::kModeComplex ? 2 : 1);
}
void ensure_buffer(void** p, size_t* cap, size_t bytes, const char* what) {
  if (*cap >= bytes) return;
  cudaFree(*p);
  *p = nullptr;
  cuda_check(cudaMalloc(p, bytes), what);
  *cap = bytes;
}
void run_transform(sftgpu_plan* pl, const void* d_x, void* d_out, cudaStream_t st) {
  if (pl->conv) {
    run_conv(pl, d_x, pl->n, d_out, pl->n, st);
  } else if (pl->precision == SFTGPU_SINGLE) {
    run_groups<float>(pl, d_x, pl->n, d_out, nullptr, pl->count, 0, st);
  } else {
    run_groups<double>(pl, d_x, pl->n, d_out, nullptr, pl->count, 0, st);
  }
}
}  // namespace

namespace {
void ensure_pipeline(sftgpu_plan* pl) {
  if (pl->s_in) return;
  const unsigned fl = cudaStreamNonBlocking;
  cuda_check(cudaStreamCreateWithFlags(&pl->s_in, fl), "stream create");
  cuda_check(cudaStreamCreateWithFlags(&pl->s_comp, fl), "stream create");
  cuda_check(cudaStreamCreateWithFlags(&pl->s_out, fl), "stream create");
  cuda_check(cudaEventCreateWithFlags(&pl->ev_entry, cudaEventDisableTiming), "event create");
  for (auto& sl : pl->slots) {
    cuda_check(cudaEventCreateWithFlags(&sl.ev_in, cudaEventDisableTiming), "event create");
    cuda_check(cudaEventCreateWithFlags(&sl.ev_comp, cudaEventDisableTiming), "event create");
    cuda_check(cudaEventCreateWithFlags(&sl.ev_out, cudaEventDisableTiming), "event create");
  }
}

// Large K4 plans from host memory: sub-batches of signals flow through two device staging
// slots on the copy-in / compute / copy-out streams, so H2D of sub-batch k+1, the kernel
// of k and D2H of k-1 overlap (the whole-batch copies are otherwise serial).
void execute_host_subbatched(sftgpu_plan* pl, const void* x_host, void* out_host, cudaStream_t user) {
  ensure_pipeline(pl);
  const long long parts = std::min<long long>(8, pl->batch);
  const long long sub = (pl->batch + parts - 1) / parts;
  const size_t es = sizeof(float), cw = pl->mode == sftk::kModeComplex ? 2 : 1;
  const size_t xsig = static_cast<size_t>(pl->n) * es, osig = static_cast<size_t>(pl->count) * cw * es;
  for (int k = 0; k < 2; ++k) {
    ensure_buffer(&pl->sb_x[k], &pl->sb_cap_x[k], sub * xsig, "cudaMalloc sub-batch x");
    ensure_buffer(&pl->sb_out[k], &pl->sb_cap_out[k], sub * osig, "cudaMalloc sub-batch out");
  }
  cuda_check(cudaEventRecord(pl->ev_entry, user), "event record");
  cuda_check(cudaStreamWaitEvent(pl->s_in, pl->ev_entry, 0), "stream wait");
  for (long long k = 0; k * sub < pl->batch; ++k) {
    const long long s0 = k * sub, ns = std::min(sub, pl->batch - s0);
    auto& sl = pl->slots[k & 1];
    if (k >= 2) cuda_check(cudaStreamWaitEvent(pl->s_in, sl.ev_comp, 0), "stream wait");
    cuda_check(cudaMemcpyAsync(pl->sb_x[k & 1], static_cast<const char*>(x_host) + s0 * xsig, ns * xsig,
                               cudaMemcpyHostToDevice, pl->s_in),
               "H2D");
    cuda_check(cudaEventRecord(sl.ev_in, pl->s_in), "event record");
    cuda_check(cudaStreamWaitEvent(pl->s_comp, sl.ev_in, 0), "stream wait");
    if (k >= 2) cuda_check(cudaStreamWaitEvent(pl->s_comp, sl.ev_out, 0), "stream wait");
    run_tc(pl, pl->sb_x[k & 1], pl->n, pl->sb_out[k & 1], pl->count, pl->s_comp, ns);
    cuda_check(cudaEventRecord(sl.ev_comp, pl->s_comp), "event record");
    cuda_check(cudaStreamWaitEvent(pl->s_out, sl.ev_comp, 0), "stream wait");
    cuda_check(cudaMemcpyAsync(static_cast<char*>(out_host) + s0 * osig, pl->sb_out[k & 1], ns * osig,
                               cudaMemcpyDeviceToHost, pl->s_out),
               "D2H");
    cuda_check(cudaEventRecord(sl.ev_out, pl->s_out), "event record");
  }
  cuda_check(cudaStreamSynchronize(pl->s_out), "stream sync");
}
}  // namespace

int sftgpu_transform_execute_host(sftgpu_plan* pl, const void* x_host, void* out_host, void* stream) {
  return guarded([&] {
    if (!pl || pl->is_components) fail(SFTGPU_EINVAL, "not a transform plan");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t xb = plan_in_bytes(pl), ob = plan_out_bytes(pl);
    if (pl->tc && pl->in_batch < 0 && pl->batch >= 4 && xb + ob >= (256u << 20)) {
      execute_host_subbatched(pl, x_host, out_host, st);
      return;
    }
    ensure_buffer(&pl->d_x, &pl->cap_x, xb, "cudaMalloc staging x");
    ensure_buffer(&pl->d_out, &pl->cap_out, ob, "cudaMalloc staging out");
    cuda_check(cudaMemcpyAsync(pl->d_x, x_host, xb, cudaMemcpyHostToDevice, st), "H2D");
    run_transform(pl, pl->d_x, pl->d_out, st);
    cuda_check(cudaMemcpyAsync(out_host, pl->d_out, ob, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "stream sync");
  });
}

int sftgpu_transform_execute_host_async(sftgpu_plan* pl, const void* x_host, void* out_host, void* stream) {
  return guarded([&] {
    if (!pl || pl->is_components) fail(SFTGPU_EINVAL, "not a transform plan");
    if (!x_host || !out_host) fail(SFTGPU_EINVAL, "null host buffer");
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    ensure_pipeline(pl);
    const size_t xb = plan_in_bytes(pl), ob = plan_out_bytes(pl);
    auto& sl = pl->slots[pl->next_slot];
    pl->next_slot = (pl->next_slot + 1) % sftgpu_plan::kSlots;
    size_t cap = sl.d_x ? xb : 0, capo = sl.d_out ? ob : 0;
    ensure_buffer(&sl.d_x, &cap, xb, "cudaMalloc async staging x");
    ensure_buffer(&sl.d_out, &capo, ob, "cudaMalloc async staging out");
    // no entry dependency on the caller's stream: that stream waits for every earlier
    // call's copy-out, and ordering copy-in behind it would serialise the pipeline
    // (x_host is host data, ready at call time)
    // copy-in may overwrite this slot's input once the slot's previous kernel has read it
    cuda_check(cudaStreamWaitEvent(pl->s_in, sl.ev_comp, 0), "stream wait");
    cuda_check(cudaMemcpyAsync(sl.d_x, x_host, xb, cudaMemcpyHostToDevice, pl->s_in), "H2D");
    cuda_check(cudaEventRecord(sl.ev_in, pl->s_in), "event record");
    // the kernel may overwrite this slot's output once its previous copy-out is done
    cuda_check(cudaStreamWaitEvent(pl->s_comp, sl.ev_in, 0), "stream wait");
    cuda_check(cudaStreamWaitEvent(pl->s_comp, sl.ev_out, 0), "stream wait");
    run_transform(pl, sl.d_x, sl.d_out, pl->s_comp);
    cuda_check(cudaEventRecord(sl.ev_comp, pl->s_comp), "event record");
    cuda_check(cudaStreamWaitEvent(pl->s_out, sl.ev_comp, 0), "stream wait");
    cuda_check(cudaMemcpyAsync(out_host, sl.d_out, ob, cudaMemcpyDeviceToHost, pl->s_out), "D2H");
    cuda_check(cudaEventRecord(sl.ev_out, pl->s_out), "event record");
    cuda_check(cudaStreamWaitEvent(user, sl.ev_out, 0), "stream wait");
  });
}

int sftgpu_plan_synchronize(sftgpu_plan* pl) {
  return guarded([&] {
    if (!pl) fail(SFTGPU_EINVAL, "null plan");
    if (pl->s_in) {
      cuda_check(cudaStreamSynchronize(pl->s_in), "stream sync");
      cuda_check(cudaStreamSynchronize(pl->s_comp), "stream sync");
      cuda_check(cudaStreamSynchronize(pl->s_out), "stream sync");
    }
  });
}

int sftgpu_plan_output_is_complex(const sftgpu_plan* pl) { return pl && pl->mode == sftk::kModeComplex ? 1 : 0; }

int sftgpu_plan_describe(const sftgpu_plan* pl, int64_t* info, int n_info) {
  return guarded([&] {
    if (!pl || !info) fail(SFTGPU_EINVAL, "null argument");
    int64_t orders = 0;
    for (const Group& g : pl->groups) orders += g.nord;
    if (pl->tc) {
      const long long units = static_cast<long long>(pl->tcp.nsig) * pl->tcp.n_scales;
      const int64_t v[11] = {0, 0, 0, tck::kTile, pl->tc_warm, pl->tcp.total_chunks / std::max(1LL, units),
                             pl->tc_grid, 1,
                             pl->tcp.nord, -1, 1};
      for (int i = 0; i < n_info && i < 11; ++i) info[i] = v[i];
      return;
    }
    const int64_t v[11] = {pl->seq, pl->conv, pl->L * 1LL, pl->TT, pl->warm_tiles, pl->n_chunks, pl->total_tiles,
                           static_cast<int64_t>(pl->groups.size()), orders,
                           pl->groups.empty() ? -1 : pl->groups[0].gm, 0};
    for (int i = 0; i < n_info && i < 11; ++i) info[i] = v[i];
  });
}

int sftgpu_plan_launches_per_execute(const sftgpu_plan* pl) {
  if (!pl) return 0;
  if (pl->conv) return static_cast<int>(pl->batch);
  if (pl->tc) return 1;
  return static_cast<int>(pl->groups.size());
}

int sftgpu_components_execute(sftgpu_plan* pl, const void* x, void* c, void* s, void* stream) {
  return guarded([&] {
    if (!pl || !pl->is_components) fail(SFTGPU_EINVAL, "not a components plan");
    if (!x || !c || !s) fail(SFTGPU_EINVAL, "null buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (pl->precision == SFTGPU_SINGLE)
      run_groups<float>(pl, x, pl->n, c, s, pl->count, 0, st);
    else
      run_groups<double>(pl, x, pl->n, c, s, pl->count, 0, st);
  });
}

int sftgpu_components_execute_host(sftgpu_plan* pl, const void* x_host, void* c_host, void* s_host, void* stream) {
  return guarded([&] {
    if (!pl || !pl->is_components) fail(SFTGPU_EINVAL, "not a components plan");
    if (!x_host || !c_host || !s_host) fail(SFTGPU_EINVAL, "null buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t es = elem_size(pl->precision);
    const size_t xb = static_cast<size_t>(pl->n * pl->batch) * es;
    size_t nord = 0;
    for (const Group& g : pl->groups) nord += g.nord;
    const size_t ob = nord * static_cast<size_t>(pl->batch * pl->count) * es;
    if (pl->cap_x < xb) {
      cudaFree(pl->d_x);
      pl->d_x = nullptr;
      cuda_check(cudaMalloc(&pl->d_x, xb), "cudaMalloc staging x");
      pl->cap_x = xb;
    }
    if (pl->cap_out < 2 * ob) {
      cudaFree(pl->d_out);
      pl->d_out = nullptr;
      cuda_check(cudaMalloc(&pl->d_out, 2 * ob), "cudaMalloc staging out");
      pl->cap_out = 2 * ob;
    }
    char* dc = static_cast<char*>(pl->d_out);
    cuda_check(cudaMemcpyAsync(pl->d_x, x_host, xb, cudaMemcpyHostToDevice, st), "H2D");
    if (pl->precision == SFTGPU_SINGLE)
      run_groups<float>(pl, pl->d_x, pl->n, dc, dc + ob, pl->count, 0, st);
    else
      run_groups<double>(pl, pl->d_x, pl->n, dc, dc + ob, pl->count, 0, st);
    cuda_check(cudaMemcpyAsync(c_host, dc, ob, cudaMemcpyDeviceToHost, st), "D2H c");
    cuda_check(cudaMemcpyAsync(s_host, dc + ob, ob, cudaMemcpyDeviceToHost, st), "D2H s");
    cuda_check(cudaStreamSynchronize(st), "stream sync");
  });
}

void sftgpu_plan_destroy(sftgpu_plan* pl) { delete pl; }

// ---------------------------------------------------------------- one-shot calls
// Library-owned plan cache for the reference-signature entry points (a reference user
// calls morlet_direct_transform(sig, spec) per signal; creating a plan per call would cost
// allocations and a table upload each time).
extern "C++" {
namespace {
struct OneShot {
  std::string key;
  sftgpu_plan* plan = nullptr;
  void* h_x = nullptr;  // pinned staging in the plan's precision
  void* h_out = nullptr;
  cudaStream_t st = nullptr;
  std::mutex mu;
  ~OneShot() {
    if (st) cudaStreamSynchronize(st);
    if (st) cudaStreamDestroy(st);
    cudaFreeHost(h_x);
    cudaFreeHost(h_out);
    delete plan;
  }
};
std::mutex g_oneshot_mu;
std::list<std::shared_ptr<OneShot>> g_oneshot;  // most recently used first
constexpr size_t kOneShotMax = 8;

std::shared_ptr<OneShot> oneshot_get(const sftgpu_spec* spec, int64_t n, int boundary) {
  sftgpu_spec canon;  // canonical bytes (zeroed padding) of the spec's contents
  spec_to_c(spec_from_c(spec), &canon);
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::string key(reinterpret_cast<const char*>(&canon), sizeof(canon));
  key.append(reinterpret_cast<const char*>(&n), sizeof(n));
  key.append(reinterpret_cast<const char*>(&boundary), sizeof(boundary));
  key.append(reinterpret_cast<const char*>(&dev), sizeof(dev));
  std::lock_guard<std::mutex> lk(g_oneshot_mu);
  for (auto it = g_oneshot.begin(); it != g_oneshot.end(); ++it)
    if ((*it)->key == key) {
      auto e = *it;
      g_oneshot.erase(it);
      g_oneshot.push_front(e);
      return e;
    }
  auto e = std::make_shared<OneShot>();
  e->key = key;
  const int rc = sftgpu_transform_plan_create(spec, n, 1, boundary, &e->plan);
  if (rc != SFTGPU_OK) throw ApiError{rc, sftgpu_last_error()};
  const size_t xb = plan_in_bytes(e->plan), ob = plan_out_bytes(e->plan);
  cuda_check(cudaHostAlloc(&e->h_x, xb, cudaHostAllocDefault), "cudaHostAlloc one-shot x");
  cuda_check(cudaHostAlloc(&e->h_out, ob, cudaHostAllocDefault), "cudaHostAlloc one-shot out");
  cuda_check(cudaStreamCreateWithFlags(&e->st, cudaStreamNonBlocking), "cudaStreamCreate one-shot");
  ensure_buffer(&e->plan->d_x, &e->plan->cap_x, xb, "cudaMalloc staging x");
  ensure_buffer(&e->plan->d_out, &e->plan->cap_out, ob, "cudaMalloc staging out");
  g_oneshot.push_front(e);
  if (g_oneshot.size() > kOneShotMax) g_oneshot.pop_back();
  return e;
}

// Host worker pool for the one-shot path's precision conversions (fp64 <-> the plan's
// precision, ~300k elements per headline call: ~100 us on one core). Workers sleep on a
// condition variable between jobs; the caller takes a share of every job. Created on first
// use, never destroyed (detached at process exit with the library).
class ConvPool {
 public:
  static ConvPool& get() {
    static ConvPool* pool = new ConvPool();
    return *pool;
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }
  // fn(part, parts) for part in [0, parts), parts = size(); returns when all are done
  void run(const std::function<void(int, int)>& fn) {
    const int parts = size();
    if (parts == 1) {
      fn(0, 1);
      return;
    }
    std::unique_lock<std::mutex> job_lock(job_mu_);  // one job at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      pending_ = parts - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0, parts);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  ConvPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    const int n = static_cast<int>(std::min(7u, hw > 1 ? hw / 2 : 0u));
    for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i + 1); });
    for (auto& t : workers_) t.detach();
  }
  void loop(int part) {
    unsigned long long seen = 0;
    for (;;) {
      const std::function<void(int, int)>* fn;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        fn = fn_;
      }
      (*fn)(part, size());
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, job_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int, int)>* fn_ = nullptr;
  int pending_ = 0;
  unsigned long long gen_ = 0;
};

// dst[i] = (To) src[i], split over the pool when the array is large
template <typename To, typename From>
void convert(To* dst, const From* src, long long count) {
  if (count < (1LL << 15)) {
    for (long long i = 0; i < count; ++i) dst[i] = static_cast<To>(src[i]);
    return;
  }
  ConvPool::get().run([&](int part, int parts) {
    const long long per = (count + parts - 1) / parts, b = part * per, e = std::min(count, b + per);
    for (long long i = b; i < e; ++i) dst[i] = static_cast<To>(src[i]);
  });
}

// fp64 host signal -> plan precision in pinned staging (host), one H2D, transform, one D2H,
// -> fp64 (host). Measured alternatives on the B200 box: converting on the device with
// pageable fp64 copies costs more (the driver stages pageable copies through the host
// anyway), and chunked copy/convert overlap loses to the per-chunk synchronisation.
template <typename T>
void oneshot_run(OneShot& e, const double* x, double* out) {
  sftgpu_plan* pl = e.plan;
  const long long n = pl->n, no = static_cast<long long>(plan_out_bytes(pl) / sizeof(T));
  T* hx = static_cast<T*>(e.h_x);
  T* ho = static_cast<T*>(e.h_out);
  convert(hx, x, n);
  cuda_check(cudaMemcpyAsync(pl->d_x, hx, n * sizeof(T), cudaMemcpyHostToDevice, e.st), "H2D");
  run_transform(pl, pl->d_x, pl->d_out, e.st);
  cuda_check(cudaMemcpyAsync(ho, pl->d_out, no * sizeof(T), cudaMemcpyDeviceToHost, e.st), "D2H");
  cuda_check(cudaStreamSynchronize(e.st), "stream sync");
  convert(out, ho, no);
}
}  // namespace
}  // extern "C++"

int sftgpu_transform_oneshot(const sftgpu_spec* spec, int64_t n, int boundary, const double* x_host,
                             double* out_host, int* complex_out) {
  return guarded([&] {
    if (!spec || !x_host || !out_host) fail(SFTGPU_EINVAL, "null argument");
    if (n < 1) fail(SFTGPU_EINVAL, "Signal: need at least one sample");
    require_device();
    std::shared_ptr<OneShot> e = oneshot_get(spec, n, boundary);
    std::lock_guard<std::mutex> lk(e->mu);
    if (complex_out) *complex_out = e->plan->mode == sftk::kModeComplex ? 1 : 0;
    if (e->plan->precision == SFTGPU_SINGLE)
      oneshot_run<float>(*e, x_host, out_host);
    else
      oneshot_run<double>(*e, x_host, out_host);
  });
}

void sftgpu_oneshot_cache_clear(void) {
  std::lock_guard<std::mutex> lk(g_oneshot_mu);
  g_oneshot.clear();
}

/* Diagnostics (not part of the reference interface): device buffer of 64 x 16 int64 that
 * K4 fills with per-tile event clocks of CTA 0 (tools/tc_trace.py); NULL disables. */
void sftgpu_debug_set_tc_trace(void* dev_buf) { g_tc_trace = static_cast<long long*>(dev_buf); }
/* Diagnostics: device buffer of tiles x 8 int64 that K1 LB fills with per-tile phase
 * timestamps when built with -DSFTK_TRACE=1 (tools/scan_trace.py); NULL disables. */
void sftgpu_debug_set_scan_trace(void* dev_buf) { g_scan_trace = static_cast<long long*>(dev_buf); }

int sftgpu_generate_signal(int kind, int64_t n, uint64_t seed, int64_t batch, int dtype, void* out, void* stream) {
  return guarded([&] {
    if (n < 1) fail(SFTGPU_EINVAL, "make_test_signal: N must be >= 1");
    if (kind < 0 || kind > 3) fail(SFTGPU_EINVAL, "make_test_signal: unknown kind");
    require_device();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long total = n * batch;
    const int threads = 256;
    const long long blocks = std::min<long long>((total + threads - 1) / threads, sftk::sm_count() * 16LL);
    if (dtype == SFTGPU_SINGLE)
      sftk::generate_signal_kernel<float><<<blocks, threads, 0, st>>>(kind, n, seed, batch, static_cast<float*>(out));
    else
      sftk::generate_signal_kernel<double><<<blocks, threads, 0, st>>>(kind, n, seed, batch, static_cast<double*>(out));
    cuda_check(cudaGetLastError(), "generate_signal_kernel launch");
  });
}

int sftgpu_truncated_convolution(const double* x, int64_t n, int boundary, const double* taps, int64_t n_taps,
                                 int64_t tap_lo, double* out, void* stream) {
  return guarded([&] {
    if (n_taps < 1) fail(SFTGPU_EINVAL, "truncated_convolution: empty kernel");
    if (n < 1) fail(SFTGPU_EINVAL, "Signal: need at least one sample");
    require_device();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    constexpr int BO = 256, BT = 1024;
    sftk::truncated_conv_kernel<double, BO, BT><<<(n + BO - 1) / BO, BO, 0, st>>>(
        x, n, boundary, reinterpret_cast<const double2*>(taps), n_taps, tap_lo, reinterpret_cast<double2*>(out));
    cuda_check(cudaGetLastError(), "truncated_conv_kernel launch");
  });
}

}  // extern "C"

namespace {
// RAII device buffer for the synchronous host-memory helpers.
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { cuda_check(cudaMalloc(&p, bytes), "cudaMalloc"); }
  ~DevBuf() { cudaFree(p); }
};
}  // namespace

extern "C" int sftgpu_generate_signal_host(int kind, int64_t n, uint64_t seed, double* out_host) {
  return guarded([&] {
    if (!out_host) fail(SFTGPU_EINVAL, "null buffer");
    if (n < 1) fail(SFTGPU_EINVAL, "make_test_signal: N must be >= 1");
    require_device();
    DevBuf d(static_cast<size_t>(n) * sizeof(double));
    const int rc = sftgpu_generate_signal(kind, n, seed, 1, SFTGPU_DOUBLE, d.p, nullptr);
    if (rc != SFTGPU_OK) fail(rc, g_err);
    cuda_check(cudaMemcpy(out_host, d.p, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  });
}

extern "C" int sftgpu_truncated_convolution_host(const double* x_host, int64_t n, int boundary, const double* taps_host,
                                                 int64_t n_taps, int64_t tap_lo, double* out_host) {
  return guarded([&] {
    if (!x_host || !taps_host || !out_host) fail(SFTGPU_EINVAL, "null buffer");
    if (n < 1) fail(SFTGPU_EINVAL, "Signal: need at least one sample");
    if (n_taps < 1) fail(SFTGPU_EINVAL, "truncated_convolution: empty kernel");
    require_device();
    DevBuf dx(static_cast<size_t>(n) * sizeof(double)), dt(static_cast<size_t>(n_taps) * 2 * sizeof(double)),
        dout(static_cast<size_t>(n) * 2 * sizeof(double));
    cuda_check(cudaMemcpy(dx.p, x_host, static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice), "H2D x");
    cuda_check(cudaMemcpy(dt.p, taps_host, static_cast<size_t>(n_taps) * 2 * sizeof(double), cudaMemcpyHostToDevice),
               "H2D taps");
    const int rc = sftgpu_truncated_convolution(static_cast<const double*>(dx.p), n, boundary,
                                                static_cast<const double*>(dt.p), n_taps, tap_lo,
                                                static_cast<double*>(dout.p), nullptr);
    if (rc != SFTGPU_OK) fail(rc, g_err);
    cuda_check(cudaMemcpy(out_host, dout.p, static_cast<size_t>(n) * 2 * sizeof(double), cudaMemcpyDeviceToHost),
               "D2H");
  });
}


