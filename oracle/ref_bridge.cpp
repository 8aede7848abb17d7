// TEST INFRASTRUCTURE ONLY — C ABI over the reference library compiled from its own
// sources (/root/reference/proj/src/*.cpp minus cli.cpp, with the mini-Eigen shim in
// oracle/ref_shim), so Python tests and bench.py's reference arm can call the literal
// reference through ctypes. Built by oracle/ref.mk into oracle/_ref/libsftref.so.
// Never linked by the product.
//
// Every entry point returns 0 on success, 1 on std::invalid_argument, 2 on any other
// exception (message: ref_last_error()).
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

#include "sft/engine.hpp"
#include "sft/kernels.hpp"
#include "sft/signal.hpp"
#include "sft/sliding_sum.hpp"
#include "sft/transforms.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

sft::Signal make_signal(const double* x, int64_t n, int boundary) {
  Eigen::ArrayXd s(n);
  for (int64_t i = 0; i < n; ++i) s[i] = x[i];
  return sft::Signal(s, boundary == 0 ? sft::BoundaryPolicy::Zero : sft::BoundaryPolicy::Clamp);
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// sft::make_transform_spec (proj/src/transforms.cpp:215-242) with TransformOptions
// (proj/include/sft/transforms.hpp:43-50); the spec is owned by the caller (ref_spec_free).
int ref_make_transform_spec(const char* abbrev, double sigma, double xi, int has_k, int k, int has_beta, double beta,
                            int tune_beta, int has_ps, int ps, int strategy, int precision, void** out) {
  return guarded([&] {
    sft::TransformOptions o;
    if (has_k) o.half_width = k;
    if (has_beta) o.beta = beta;
    o.tune_beta = tune_beta != 0;
    if (has_ps) o.ps = ps;
    o.strategy = static_cast<sft::Strategy>(strategy);
    o.precision = static_cast<sft::Precision>(precision);
    *out = new sft::TransformSpec(sft::make_transform_spec(abbrev, sigma, xi, o));
  });
}

void ref_spec_free(void* spec) { delete static_cast<sft::TransformSpec*>(spec); }

int ref_spec_set_engine(void* spec, int strategy, int precision) {
  return guarded([&] {
    auto* s = static_cast<sft::TransformSpec*>(spec);
    s->strategy = static_cast<sft::Strategy>(strategy);
    s->precision = static_cast<sft::Precision>(precision);
  });
}

// info: kind, K, beta, n0, alpha, ps, pd, max_order, kernel_rmse_percent, sigma, xi
int ref_spec_info(const void* spec, double* info) {
  return guarded([&] {
    const auto* s = static_cast<const sft::TransformSpec*>(spec);
    int k = 0;
    double sigma = 0, xi = 0;
    if (s->gaussian) {
      k = s->gaussian->half_width;
      sigma = s->gaussian->sigma;
    }
    if (s->morlet) {
      k = s->morlet->half_width;
      sigma = s->morlet->sigma;
      xi = s->morlet->xi;
    }
    const double v[11] = {static_cast<double>(s->kind), static_cast<double>(k), s->beta, static_cast<double>(s->n0),
                          s->alpha, static_cast<double>(s->ps), static_cast<double>(s->pd),
                          static_cast<double>(s->max_order), s->kernel_rmse_percent, sigma, xi};
    std::memcpy(info, v, sizeof(v));
  });
}

// sft::apply_transform (proj/src/transforms.cpp:444-459): out = interleaved complex[n]
int ref_apply_transform(const void* spec, const double* x, int64_t n, int boundary, int workers, double* out) {
  return guarded([&] {
    const sft::Signal sig = make_signal(x, n, boundary);
    const sft::TransformResult r = sft::apply_transform(sig, *static_cast<const sft::TransformSpec*>(spec), workers);
    for (int64_t i = 0; i < r.values.size(); ++i) {
      out[2 * i] = r.values[i].real();
      out[2 * i + 1] = r.values[i].imag();
    }
  });
}

// sft::effective_kernel (proj/src/transforms.cpp:461-477); taps NULL: size query
int ref_effective_kernel(const void* spec, double* taps, int64_t cap, int64_t* n_taps, int64_t* lo) {
  return guarded([&] {
    const sft::KernelTaps t = sft::effective_kernel(*static_cast<const sft::TransformSpec*>(spec));
    *n_taps = t.taps.size();
    *lo = t.lo;
    if (taps) {
      if (cap < t.taps.size()) throw std::invalid_argument("taps buffer too small");
      for (int64_t i = 0; i < t.taps.size(); ++i) {
        taps[2 * i] = t.taps[i].real();
        taps[2 * i + 1] = t.taps[i].imag();
      }
    }
  });
}

// Coefficients of a Gauss (a, b, d) or Morlet (cos/sin orders + complex coefficients)
// spec, so the restated oracle can be run on exactly the reference's coefficients.
// gauss: a[P+1], b[P], d[P+1]; morlet: orders[n], coeffs[2n] per cos / sin list.
int ref_spec_gauss_coeffs(const void* spec, int cap, int* P, double* a, double* b, double* d) {
  return guarded([&] {
    const auto* s = static_cast<const sft::TransformSpec*>(spec);
    if (!s->gauss_coeffs) throw std::invalid_argument("not a Gaussian spec");
    const auto& g = *s->gauss_coeffs;
    *P = g.max_order;
    if (g.max_order + 1 > cap) throw std::invalid_argument("buffer too small");
    for (int p = 0; p <= g.max_order; ++p) {
      a[p] = g.a[p];
      d[p] = g.d[p];
      if (p < g.max_order) b[p] = g.b[p];
    }
  });
}

int ref_spec_morlet_coeffs(const void* spec, int which, int cap, int* n_cos, int* cos_orders, double* cos_coeffs,
                           int* n_sin, int* sin_orders, double* sin_coeffs) {
  return guarded([&] {
    const auto* s = static_cast<const sft::TransformSpec*>(spec);
    const auto& opt = which == 0 ? s->morlet_coeffs : s->envelope_coeffs;
    if (!opt) throw std::invalid_argument("spec has no such coefficient set");
    const sft::CoefficientSet& c = *opt;
    *n_cos = static_cast<int>(c.grid.cos_orders.size());
    *n_sin = static_cast<int>(c.grid.sin_orders.size());
    if (*n_cos > cap || *n_sin > cap) throw std::invalid_argument("buffer too small");
    for (int i = 0; i < *n_cos; ++i) {
      cos_orders[i] = c.grid.cos_orders[i];
      cos_coeffs[2 * i] = c.cos_coeffs[i].real();
      cos_coeffs[2 * i + 1] = c.cos_coeffs[i].imag();
    }
    for (int i = 0; i < *n_sin; ++i) {
      sin_orders[i] = c.grid.sin_orders[i];
      sin_coeffs[2 * i] = c.sin_coeffs[i].real();
      sin_coeffs[2 * i + 1] = c.sin_coeffs[i].imag();
    }
  });
}

// sft::components_over / sft_via_sliding_sum (proj/src/engine.cpp:255-337)
int ref_components(const double* x, int64_t n, int boundary, int K, double beta, int integer_order, int p,
                   double omega, double alpha, int strategy, int precision, int window_2k1, int64_t lo, int64_t hi,
                   int route, double* c, double* s) {
  return guarded([&] {
    const sft::Signal sig = make_signal(x, n, boundary);
    sft::SftConfig cfg;
    cfg.half_width = K;
    cfg.beta = beta;
    cfg.order = integer_order ? sft::OrderSpec::order(p) : sft::OrderSpec::frequency(omega);
    cfg.alpha = alpha;
    cfg.strategy = static_cast<sft::Strategy>(strategy);
    cfg.precision = static_cast<sft::Precision>(precision);
    cfg.window_2k1 = window_2k1 != 0;
    const sft::ComponentSeq r = route == 1 ? sft::sft_via_sliding_sum(sig, cfg) : sft::components_over(sig, cfg, lo, hi);
    for (int64_t i = 0; i < r.c.size(); ++i) {
      c[i] = r.c[i];
      s[i] = r.s[i];
    }
  });
}

// sft::make_test_signal (proj/src/signal.cpp:24-51)
int ref_make_test_signal(int kind, int64_t n, uint64_t seed, double* out) {
  return guarded([&] {
    const sft::Signal s = sft::make_test_signal(static_cast<sft::TestSignalKind>(kind), n, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = s.samples[i];
  });
}

// sft::sliding_sum_flat<int64_t> (proj/include/sft/sliding_sum.hpp:89-121)
int ref_sliding_sum_flat_i64(const int64_t* f, int64_t n, int64_t window, int64_t* out) {
  return guarded([&] {
    Eigen::ArrayX<std::int64_t> a(n);
    for (int64_t i = 0; i < n; ++i) a[i] = f[i];
    const Eigen::ArrayX<std::int64_t> h = sft::sliding_sum_flat<std::int64_t>(a, window);
    for (int64_t i = 0; i < h.size(); ++i) out[i] = h[i];
  });
}

}  // extern "C"
