// sft_b200/sft.hpp — drop-in C++ API of the reference library's transform path
// (namespace sft, /root/reference/proj/include/sft/{signal,engine,kernels,
// fourier_fit,transforms}.hpp), executed on the B200 through the C ABI of
// sftgpu.h (libsftgpu.so). Header-only; link with -lsftgpu.
//
// Same names, argument order, enums and error behaviour as the reference:
// validation failures throw std::invalid_argument, Gram-condition failures throw
// sft::FitDegenerateError, CUDA failures (including "no device": there is no CPU
// fallback) throw std::runtime_error. Containers are std::vector instead of
// Eigen arrays (ArrayXd -> std::vector<double>, ArrayXcd -> std::vector<complex>);
// see INTEGRATION.md for the Eigen adapters.
#pragma once

#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../sftgpu.h"

namespace sft {

using ArrayXd = std::vector<double>;
using ArrayXcd = std::vector<std::complex<double>>;

enum class BoundaryPolicy { Zero = SFTGPU_BOUNDARY_ZERO, Clamp = SFTGPU_BOUNDARY_CLAMP };
enum class Precision { Single = SFTGPU_SINGLE, Double = SFTGPU_DOUBLE };
enum class Strategy { KernelIntegral = SFTGPU_KERNEL_INTEGRAL, Recursive1 = SFTGPU_RECURSIVE1, Recursive2 = SFTGPU_RECURSIVE2 };
enum class TransformKind {
  Gauss = SFTGPU_GAUSS,
  GaussD = SFTGPU_GAUSS_D,
  GaussDD = SFTGPU_GAUSS_DD,
  MorletDirect = SFTGPU_MORLET_DIRECT,
  MorletMultiply = SFTGPU_MORLET_MULTIPLY,
  TruncConvGauss = SFTGPU_TRUNC_CONV_GAUSS,
  TruncConvMorlet = SFTGPU_TRUNC_CONV_MORLET
};
enum class GaussKind { Value = SFTGPU_GK_VALUE, Deriv1 = SFTGPU_GK_DERIV1, Deriv2 = SFTGPU_GK_DERIV2 };
enum class TestSignalKind { Impulse = SFTGPU_SIG_IMPULSE, Constant = SFTGPU_SIG_CONSTANT, Chirp = SFTGPU_SIG_CHIRP,
                            SeededNoise = SFTGPU_SIG_NOISE };

class FitDegenerateError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc) {
  if (rc == SFTGPU_OK) return;
  const std::string m = sftgpu_last_error();
  if (rc == SFTGPU_EINVAL) throw std::invalid_argument(m);
  if (rc == SFTGPU_EDEGENERATE) throw FitDegenerateError(m);
  throw std::runtime_error(m);
}

// RAII plan handle
struct Plan {
  sftgpu_plan* p = nullptr;
  Plan() = default;
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;
  ~Plan() { sftgpu_plan_destroy(p); }
};
}  // namespace detail

// ------------------------------------------------------------------ signal (signal.hpp)
struct Signal {
  ArrayXd samples;
  BoundaryPolicy boundary = BoundaryPolicy::Clamp;

  Signal() = default;
  Signal(ArrayXd s, BoundaryPolicy b = BoundaryPolicy::Clamp) : samples(std::move(s)), boundary(b) {
    if (samples.empty()) throw std::invalid_argument("Signal: need at least one sample");
    for (double v : samples)
      if (!std::isfinite(v)) throw std::invalid_argument("Signal: samples must be finite");
  }
  std::int64_t size() const { return static_cast<std::int64_t>(samples.size()); }
};

inline double extended_sample(const Signal& sig, std::int64_t n) {
  const std::int64_t size = sig.size();
  if (n >= 0 && n < size) return sig.samples[static_cast<size_t>(n)];
  if (sig.boundary == BoundaryPolicy::Zero) return 0.0;
  return n < 0 ? sig.samples.front() : sig.samples.back();
}

// Generated on the device (splitmix64 noise is bit-identical to the reference).
inline Signal make_test_signal(TestSignalKind kind, std::int64_t n, std::uint64_t seed,
                               BoundaryPolicy boundary = BoundaryPolicy::Clamp) {
  if (n < 1) throw std::invalid_argument("make_test_signal: N must be >= 1");
  ArrayXd x(static_cast<size_t>(n));
  detail::check(sftgpu_generate_signal_host(static_cast<int>(kind), n, seed, x.data()));
  return Signal(std::move(x), boundary);
}

// ------------------------------------------------------------------ engine (engine.hpp)
struct OrderSpec {
  bool integer_order = true;
  int p = 0;
  double omega = 0.0;
  static OrderSpec order(int p) {
    if (p < 0) throw std::invalid_argument("OrderSpec: p must be >= 0");
    OrderSpec s;
    s.p = p;
    return s;
  }
  static OrderSpec frequency(double omega) {
    OrderSpec s;
    s.integer_order = false;
    s.omega = omega;
    return s;
  }
  double angular(double beta) const { return integer_order ? beta * p : omega; }
};

struct SftConfig {
  int half_width;
  double beta;
  OrderSpec order;
  double alpha = 0.0;
  int n0 = 0;
  Strategy strategy = Strategy::Recursive2;
  Precision precision = Precision::Double;
  bool window_2k1 = false;

  sftgpu_config raw() const {
    sftgpu_config c{};
    c.half_width = half_width;
    c.beta = beta;
    c.integer_order = order.integer_order ? 1 : 0;
    c.p = order.p;
    c.omega = order.omega;
    c.alpha = alpha;
    c.n0 = n0;
    c.strategy = static_cast<int>(strategy);
    c.precision = static_cast<int>(precision);
    c.window_2k1 = window_2k1 ? 1 : 0;
    return c;
  }
};

struct ComponentSeq {
  ArrayXd c;
  ArrayXd s;
};

namespace detail {
template <typename T>
ComponentSeq run_components(const Signal& sig, const SftConfig& cfg, std::int64_t lo, std::int64_t hi, int mode) {
  const sftgpu_config rc = cfg.raw();
  Plan plan;
  check(sftgpu_components_plan_create(&rc, 1, sig.size(), 1, static_cast<int>(sig.boundary), lo, hi, mode, &plan.p));
  std::vector<T> x(sig.samples.begin(), sig.samples.end());
  const size_t cnt = static_cast<size_t>(hi - lo + 1);
  std::vector<T> c(cnt), s(cnt);
  check(sftgpu_components_execute_host(plan.p, x.data(), c.data(), s.data(), nullptr));
  return ComponentSeq{ArrayXd(c.begin(), c.end()), ArrayXd(s.begin(), s.end())};
}
inline ComponentSeq components(const Signal& sig, const SftConfig& cfg, std::int64_t lo, std::int64_t hi, int mode) {
  if (cfg.precision == Precision::Single) return run_components<float>(sig, cfg, lo, hi, mode);
  return run_components<double>(sig, cfg, lo, hi, mode);
}
}  // namespace detail

inline ComponentSeq components_over(const Signal& sig, const SftConfig& cfg, std::int64_t lo, std::int64_t hi) {
  return detail::components(sig, cfg, lo, hi, 0);
}
inline ComponentSeq sft_components(const Signal& sig, const SftConfig& cfg) {
  return detail::components(sig, cfg, 0, sig.size() - 1, 1);
}
inline ComponentSeq asft_components(const Signal& sig, const SftConfig& cfg) {
  return detail::components(sig, cfg, 0, sig.size() - 1, 2);
}
// engine.cpp:323-337: every GPU output is a fresh bounded-state window sum already;
// the reference's overflow guard for its rebased sequence is kept for API parity.
inline ComponentSeq sft_via_sliding_sum(const Signal& sig, const SftConfig& cfg, int /*workers*/ = 1) {
  if (cfg.alpha * (0.5 * static_cast<double>(sig.size()) + cfg.half_width) > 600.0)
    throw std::invalid_argument("sft_via_sliding_sum: alpha * N / 2 too large for the attenuated phased sequence");
  SftConfig k = cfg;
  k.strategy = Strategy::KernelIntegral;
  return detail::components(sig, k, 0, sig.size() - 1, 0);
}

// ------------------------------------------------------------------ kernels (kernels.hpp)
struct GaussianParams {
  double sigma;
  int half_width;
  explicit GaussianParams(double s, int k = 0) : sigma(s), half_width(k > 0 ? k : default_half_width(s)) {
    if (!(sigma > 0.0)) throw std::invalid_argument("GaussianParams: sigma must be > 0");
    if (half_width < 1) throw std::invalid_argument("GaussianParams: K must be >= 1");
  }
  double gamma() const { return 1.0 / (2.0 * sigma * sigma); }
  static int default_half_width(double s) { return static_cast<int>(std::ceil(3.0 * s)); }
};

struct MorletParams {
  double sigma, xi;
  int half_width;
  MorletParams(double s, double x, int k = 0)
      : sigma(s), xi(x), half_width(k > 0 ? k : GaussianParams::default_half_width(s)) {
    if (!(sigma > 0.0)) throw std::invalid_argument("MorletParams: sigma must be > 0");
    if (!(xi > 0.0)) throw std::invalid_argument("MorletParams: xi must be > 0");
    if (half_width < 1) throw std::invalid_argument("MorletParams: K must be >= 1");
  }
  double kappa_xi() const { return std::exp(-0.5 * xi * xi); }
  double c_xi() const { return 1.0 / std::sqrt(1.0 + std::exp(-xi * xi) - 2.0 * std::exp(-0.75 * xi * xi)); }
  double gamma() const { return 1.0 / (2.0 * sigma * sigma); }
};

inline double gauss(const GaussianParams& p, double n) {
  const double g = p.gamma();
  return std::sqrt(g / M_PI) * std::exp(-g * n * n);
}
inline double gauss_d(const GaussianParams& p, double n) { return -2.0 * p.gamma() * n * gauss(p, n); }
inline double gauss_dd(const GaussianParams& p, double n) {
  const double g = p.gamma();
  return (4.0 * g * g * n * n - 2.0 * g) * gauss(p, n);
}
inline std::complex<double> morlet(const MorletParams& p, double n) {
  const double env =
      p.c_xi() / (std::pow(M_PI, 0.25) * std::sqrt(p.sigma)) * std::exp(-n * n / (2.0 * p.sigma * p.sigma));
  const double ph = p.xi * n / p.sigma;
  return env * (std::complex<double>(std::cos(ph), std::sin(ph)) - p.kappa_xi());
}

struct KernelTaps {
  ArrayXcd taps;
  std::int64_t lo = 0;
  std::int64_t hi() const { return lo + static_cast<std::int64_t>(taps.size()) - 1; }
};

// kernels.cpp:35-51 on the GPU (fp64): out[n] = sum_k taps[k] x[n - (lo + k)].
inline ArrayXcd truncated_convolution(const Signal& sig, const KernelTaps& kernel, int /*workers*/ = 1) {
  if (kernel.taps.empty()) throw std::invalid_argument("truncated_convolution: empty kernel");
  ArrayXcd out(static_cast<size_t>(sig.size()));
  detail::check(sftgpu_truncated_convolution_host(sig.samples.data(), sig.size(), static_cast<int>(sig.boundary),
                                                  reinterpret_cast<const double*>(kernel.taps.data()),
                                                  static_cast<std::int64_t>(kernel.taps.size()), kernel.lo,
                                                  reinterpret_cast<double*>(out.data())));
  return out;
}

// ------------------------------------------------------------------ transforms (transforms.hpp)
struct TransformOptions {
  std::optional<int> half_width;
  std::optional<double> beta;
  bool tune_beta = false;
  std::optional<int> ps;
  Strategy strategy = Strategy::Recursive2;
  Precision precision = Precision::Double;

  sftgpu_options raw() const {
    sftgpu_options o{};
    o.has_half_width = half_width.has_value();
    o.half_width = half_width.value_or(0);
    o.has_beta = beta.has_value();
    o.beta = beta.value_or(0.0);
    o.tune_beta = tune_beta;
    o.has_ps = ps.has_value();
    o.ps = ps.value_or(0);
    o.strategy = static_cast<int>(strategy);
    o.precision = static_cast<int>(precision);
    return o;
  }
};

struct AbbrevInfo {
  TransformKind kind;
  int n0 = 0;
  int order = 0;
};

inline AbbrevInfo parse_abbreviation(const std::string& a) {
  int k = 0, n0 = 0, o = 0;
  detail::check(sftgpu_parse_abbreviation(a.c_str(), &k, &n0, &o));
  return AbbrevInfo{static_cast<TransformKind>(k), n0, o};
}

inline std::string encode_abbreviation(TransformKind kind, int n0, int order) {
  char buf[32];
  detail::check(sftgpu_encode_abbreviation(static_cast<int>(kind), n0, order, buf, sizeof(buf)));
  return buf;
}

// A fully resolved transform. The engine knobs (n0, alpha, strategy, precision) are
// public like the reference's fields; everything else lives in the fitted C spec.
struct TransformSpec {
  TransformKind kind = TransformKind::Gauss;
  int max_order = 0, ps = 0, pd = 0;
  double beta = 0.0;
  int n0 = 0;
  double alpha = 0.0;
  Strategy strategy = Strategy::Recursive2;
  Precision precision = Precision::Double;
  std::string abbreviation;
  double kernel_rmse_percent = 0.0;
  sftgpu_spec raw{};

  static TransformSpec from_raw(const sftgpu_spec& r) {
    TransformSpec s;
    s.raw = r;
    s.kind = static_cast<TransformKind>(r.kind);
    s.max_order = r.max_order;
    s.ps = r.ps;
    s.pd = r.pd;
    s.beta = r.beta;
    s.n0 = r.n0;
    s.alpha = r.alpha;
    s.strategy = static_cast<Strategy>(r.strategy);
    s.precision = static_cast<Precision>(r.precision);
    s.abbreviation = r.abbreviation;
    s.kernel_rmse_percent = r.kernel_rmse_percent;
    return s;
  }
  sftgpu_spec synced() const {
    sftgpu_spec r = raw;
    r.n0 = n0;
    r.alpha = alpha;
    r.strategy = static_cast<int>(strategy);
    r.precision = static_cast<int>(precision);
    return r;
  }
  int half_width() const { return raw.half_width; }
  double sigma() const { return raw.sigma; }
};

struct TransformResult {
  ArrayXcd values;
  bool complex_valued = false;
  std::string abbreviation;
  Strategy strategy = Strategy::Recursive2;
  Precision precision = Precision::Double;
  double kernel_rmse_percent = 0.0;
};

inline TransformSpec make_transform_spec(const std::string& a, double sigma, double xi,
                                         const TransformOptions& options = {}) {
  sftgpu_spec r;
  const sftgpu_options o = options.raw();
  detail::check(sftgpu_make_transform_spec(a.c_str(), sigma, xi, &o, &r));
  return TransformSpec::from_raw(r);
}
inline TransformSpec make_gauss_spec(double sigma, GaussKind kind, int max_order, int n0,
                                     const TransformOptions& options = {}) {
  sftgpu_spec r;
  const sftgpu_options o = options.raw();
  detail::check(sftgpu_make_gauss_spec(sigma, static_cast<int>(kind), max_order, n0, &o, &r));
  return TransformSpec::from_raw(r);
}
inline TransformSpec make_morlet_direct_spec(double sigma, double xi, int pd, int n0,
                                             const TransformOptions& options = {}) {
  sftgpu_spec r;
  const sftgpu_options o = options.raw();
  detail::check(sftgpu_make_morlet_direct_spec(sigma, xi, pd, n0, &o, &r));
  return TransformSpec::from_raw(r);
}
inline TransformSpec make_morlet_multiply_spec(double sigma, double xi, int pm, int n0,
                                               const TransformOptions& options = {}) {
  sftgpu_spec r;
  const sftgpu_options o = options.raw();
  detail::check(sftgpu_make_morlet_multiply_spec(sigma, xi, pm, n0, &o, &r));
  return TransformSpec::from_raw(r);
}

inline KernelTaps effective_kernel(const TransformSpec& spec) {
  const sftgpu_spec r = spec.synced();
  std::int64_t n = 0, lo = 0;
  detail::check(sftgpu_effective_kernel(&r, nullptr, 0, &n, &lo));
  KernelTaps t;
  t.taps.resize(static_cast<size_t>(n));
  t.lo = lo;
  detail::check(sftgpu_effective_kernel(&r, reinterpret_cast<double*>(t.taps.data()), n, &n, &lo));
  return t;
}

namespace detail {
// One call = one library one-shot transform (sftgpu_transform_oneshot): the plan, its
// device buffers and pinned staging are cached inside the library, so a reference user
// calling morlet_direct_transform(sig, spec) per signal pays no plan creation per call.
inline TransformResult transform(const Signal& sig, const TransformSpec& spec) {
  const sftgpu_spec r = spec.synced();
  TransformResult res;
  res.values.resize(static_cast<size_t>(sig.size()));
  int cplx = 0;
  static_assert(sizeof(std::complex<double>) == 2 * sizeof(double), "complex<double> layout");
  std::vector<double> real;  // real outputs land here, then widen to complex
  double* out = reinterpret_cast<double*>(res.values.data());
  const bool maybe_real = spec.kind == TransformKind::Gauss || spec.kind == TransformKind::GaussD ||
                          spec.kind == TransformKind::GaussDD || spec.kind == TransformKind::TruncConvGauss;
  if (maybe_real) {
    real.resize(static_cast<size_t>(sig.size()));
    out = real.data();
  }
  check(sftgpu_transform_oneshot(&r, sig.size(), static_cast<int>(sig.boundary), sig.samples.data(), out, &cplx));
  if (maybe_real)
    for (size_t i = 0; i < real.size(); ++i) res.values[i] = std::complex<double>(real[i], 0.0);
  res.complex_valued = cplx != 0;
  res.abbreviation = spec.abbreviation;
  res.strategy = spec.strategy;
  res.precision = spec.precision;
  res.kernel_rmse_percent = spec.kernel_rmse_percent;
  return res;
}
}  // namespace detail

inline TransformResult gauss_smooth(const Signal& sig, const TransformSpec& spec, int /*workers*/ = 1) {
  if (spec.kind != TransformKind::Gauss && spec.kind != TransformKind::GaussD && spec.kind != TransformKind::GaussDD)
    throw std::invalid_argument("gauss_smooth: spec kind mismatch");
  return detail::transform(sig, spec);
}
inline TransformResult morlet_direct_transform(const Signal& sig, const TransformSpec& spec, int /*workers*/ = 1) {
  if (spec.kind != TransformKind::MorletDirect) throw std::invalid_argument("morlet_direct_transform: spec mismatch");
  return detail::transform(sig, spec);
}
inline TransformResult morlet_multiply_transform(const Signal& sig, const TransformSpec& spec, int /*workers*/ = 1) {
  if (spec.kind != TransformKind::MorletMultiply)
    throw std::invalid_argument("morlet_multiply_transform: spec mismatch");
  return detail::transform(sig, spec);
}
inline TransformResult truncated_reference(const Signal& sig, const TransformSpec& spec, int /*workers*/ = 1) {
  if (spec.kind != TransformKind::TruncConvGauss && spec.kind != TransformKind::TruncConvMorlet)
    throw std::invalid_argument("truncated_reference: spec mismatch");
  return detail::transform(sig, spec);
}
inline TransformResult apply_transform(const Signal& sig, const TransformSpec& spec, int /*workers*/ = 1) {
  return detail::transform(sig, spec);
}

// ------------------------------------------------------------------ fits (fourier_fit.hpp)
inline int select_optimal_ps(const MorletParams& p, int pd, int n0 = 0) {
  int ps = 0;
  detail::check(sftgpu_select_optimal_ps(p.sigma, p.xi, p.half_width, pd, n0, &ps));
  return ps;
}
inline double morlet_direct_kernel_rmse(const MorletParams& p, int ps, int pd, int n0) {
  double r = 0.0;
  detail::check(sftgpu_morlet_direct_kernel_rmse(p.sigma, p.xi, p.half_width, ps, pd, n0, &r));
  return r;
}
inline double morlet_multiply_kernel_rmse(const MorletParams& p, int pm, int n0) {
  double r = 0.0;
  detail::check(sftgpu_morlet_multiply_kernel_rmse(p.sigma, p.xi, p.half_width, pm, n0, &r));
  return r;
}

}  // namespace sft
