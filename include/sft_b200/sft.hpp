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

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <functional>
#include <optional>
#include <type_traits>
#include <utility>
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
// Recursive1/2 (engine.cpp:53-120) replayed on the GPU with the reference's rounding (K7)
inline ComponentSeq replay(const Signal& sig, const SftConfig& cfg, std::int64_t lo, std::int64_t hi, int mode,
                           double* max_state = nullptr) {
  if (mode == 1 && cfg.alpha != 0.0) throw std::invalid_argument("sft_components: alpha must be 0 (use asft_components)");
  if (mode == 2 && !(cfg.alpha > 0.0)) throw std::invalid_argument("asft_components: alpha must be > 0");
  const sftgpu_config rc = cfg.raw();
  const size_t cnt = hi >= lo ? static_cast<size_t>(hi - lo + 1) : 1;
  ComponentSeq out{ArrayXd(cnt), ArrayXd(cnt)};
  check(sftgpu_components_replay(&rc, 1, sig.samples.data(), sig.size(), static_cast<int>(sig.boundary), lo, hi,
                                 out.c.data(), out.s.data(), max_state));
  return out;
}
inline ComponentSeq components(const Signal& sig, const SftConfig& cfg, std::int64_t lo, std::int64_t hi, int mode) {
  if (cfg.strategy != Strategy::KernelIntegral && cfg.order.integer_order) return replay(sig, cfg, lo, hi, mode);
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
// engine.cpp:183-219, 323-337: the sliding-sum route on the GPU (phased sequence, K5
// flat window sums, rescale / phase removal).
inline ComponentSeq sft_via_sliding_sum(const Signal& sig, const SftConfig& cfg, int /*workers*/ = 1) {
  const sftgpu_config rc = cfg.raw();
  ComponentSeq out{ArrayXd(static_cast<size_t>(sig.size())), ArrayXd(static_cast<size_t>(sig.size()))};
  detail::check(sftgpu_sft_via_sliding_sum(&rc, sig.samples.data(), sig.size(), static_cast<int>(sig.boundary),
                                           out.c.data(), out.s.data()));
  return out;
}


// engine.hpp:82-102 --------------------------------------------------------------------
/// Kernel-integral window state u_{(2K+1)}[n+K] = sum_{j=n-K}^{n+K} x[j] e^{i omega j}
/// two ways (engine.cpp:270-300), both on the GPU: via_prefix by the sliding-sum route
/// (K5 window sums of the phased sequence), via_recurrence by the window-recurrence scan
/// (K1); each GPU result carries the output phase removed, re-applied here. Plain SFT only.
struct WindowState {
  ArrayXcd via_prefix;
  ArrayXcd via_recurrence;
};
inline WindowState sliding_window_state(const Signal& sig, const SftConfig& cfg) {
  if (cfg.alpha != 0.0) throw std::invalid_argument("sliding_window_state: plain SFT only");
  SftConfig k = cfg;
  k.strategy = Strategy::KernelIntegral;
  k.precision = Precision::Double;
  const ComponentSeq a = sft_via_sliding_sum(sig, k);
  const ComponentSeq b = sft_components(sig, k);
  const double omega = cfg.order.integer_order ? cfg.beta * cfg.order.p : cfg.order.omega;
  WindowState st;
  st.via_prefix.resize(a.c.size());
  st.via_recurrence.resize(b.c.size());
  for (size_t n = 0; n < a.c.size(); ++n) {
    const std::complex<double> ph(std::cos(omega * static_cast<double>(n)), std::sin(omega * static_cast<double>(n)));
    st.via_prefix[n] = ph * std::complex<double>(a.c[n], -a.s[n]);
    st.via_recurrence[n] = ph * std::complex<double>(b.c[n], -b.s[n]);
  }
  return st;
}

/// engine.cpp:302-320: cfg at single precision against a double-precision run of the same
/// configuration (both on the GPU). abs_error[n] = max(|dc|, |ds|); max_component_error is
/// its max over the reference's peak component. max_state_magnitude is the peak |window
/// state| the fp32 scan carries (the GPU keeps the 2K-window state, not the reference's
/// running recursion).
struct StabilityReport {
  double max_state_magnitude = 0.0;
  double max_component_error = 0.0;
  double reference_scale = 0.0;
  ArrayXd abs_error;
};
inline StabilityReport stability_probe(const Signal& sig, const SftConfig& cfg) {
  SftConfig sc = cfg, dc = cfg;
  sc.precision = Precision::Single;
  dc.precision = Precision::Double;
  // recursive strategies: the reference's own fp32 recurrence and its peak filter state
  const bool rec = cfg.strategy != Strategy::KernelIntegral && cfg.order.integer_order;
  double peak = 0.0;
  const ComponentSeq lo = rec ? detail::replay(sig, sc, 0, sig.size() - 1, 0, &peak)
                              : components_over(sig, sc, 0, sig.size() - 1);
  const ComponentSeq ref = components_over(sig, dc, 0, sig.size() - 1);
  StabilityReport r;
  r.abs_error.resize(ref.c.size());
  double emax = 0.0;
  for (size_t n = 0; n < ref.c.size(); ++n) {
    r.abs_error[n] = std::max(std::abs(lo.c[n] - ref.c[n]), std::abs(lo.s[n] - ref.s[n]));
    emax = std::max(emax, r.abs_error[n]);
    r.reference_scale = std::max({r.reference_scale, std::abs(ref.c[n]), std::abs(ref.s[n])});
    if (!rec) r.max_state_magnitude = std::max(r.max_state_magnitude, std::hypot(lo.c[n], lo.s[n]));
  }
  if (rec) r.max_state_magnitude = peak;
  r.max_component_error = r.reference_scale > 0.0 ? emax / r.reference_scale : emax;
  return r;
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

// fourier_fit.hpp:14-160 ---------------------------------------------------------------
struct HarmonicGrid {
  int half_width;
  double beta;
  std::vector<int> cos_orders;
  std::vector<int> sin_orders;
  HarmonicGrid(int k, double beta_, std::vector<int> cos_p, std::vector<int> sin_p)
      : half_width(k), beta(beta_), cos_orders(std::move(cos_p)), sin_orders(std::move(sin_p)) {}
  std::size_t basis_size() const { return cos_orders.size() + sin_orders.size(); }
};
enum class CoeffKind { GaussCos = 0, GaussDerivSin, GaussDeriv2Cos, MorletDirect, MorletMultiply };
struct CoefficientSet {
  CoeffKind kind = CoeffKind::GaussCos;
  HarmonicGrid grid{1, 1.0, {}, {}};
  ArrayXcd cos_coeffs;
  ArrayXcd sin_coeffs;
  double fit_rmse_percent = 0.0;
  double sigma = 0.0;
  double xi = 0.0;
  int n0 = 0;

  static CoefficientSet from_raw(const sftgpu_coeffs& r) {
    CoefficientSet c;
    c.kind = static_cast<CoeffKind>(r.kind);
    c.grid = HarmonicGrid(r.half_width, r.beta, std::vector<int>(r.cos_orders, r.cos_orders + r.n_cos),
                          std::vector<int>(r.sin_orders, r.sin_orders + r.n_sin));
    for (int i = 0; i < r.n_cos; ++i) c.cos_coeffs.emplace_back(r.cos_coeffs[2 * i], r.cos_coeffs[2 * i + 1]);
    for (int i = 0; i < r.n_sin; ++i) c.sin_coeffs.emplace_back(r.sin_coeffs[2 * i], r.sin_coeffs[2 * i + 1]);
    c.fit_rmse_percent = r.fit_rmse_percent;
    c.sigma = r.sigma;
    c.xi = r.xi;
    c.n0 = r.n0;
    return c;
  }
  sftgpu_coeffs raw() const {
    sftgpu_coeffs r;
    std::memset(&r, 0, sizeof(r));
    if (grid.cos_orders.size() > SFTGPU_MAX_COEFFS || grid.sin_orders.size() > SFTGPU_MAX_COEFFS)
      throw std::invalid_argument("CoefficientSet: too many orders");
    r.kind = static_cast<int>(kind);
    r.half_width = grid.half_width;
    r.beta = grid.beta;
    r.n_cos = static_cast<int>(grid.cos_orders.size());
    r.n_sin = static_cast<int>(grid.sin_orders.size());
    for (int i = 0; i < r.n_cos; ++i) {
      r.cos_orders[i] = grid.cos_orders[i];
      r.cos_coeffs[2 * i] = i < static_cast<int>(cos_coeffs.size()) ? cos_coeffs[i].real() : 0.0;
      r.cos_coeffs[2 * i + 1] = i < static_cast<int>(cos_coeffs.size()) ? cos_coeffs[i].imag() : 0.0;
    }
    for (int i = 0; i < r.n_sin; ++i) {
      r.sin_orders[i] = grid.sin_orders[i];
      r.sin_coeffs[2 * i] = i < static_cast<int>(sin_coeffs.size()) ? sin_coeffs[i].real() : 0.0;
      r.sin_coeffs[2 * i + 1] = i < static_cast<int>(sin_coeffs.size()) ? sin_coeffs[i].imag() : 0.0;
    }
    r.fit_rmse_percent = fit_rmse_percent;
    r.sigma = sigma;
    r.xi = xi;
    r.n0 = n0;
    return r;
  }
};

/// fit_mmse (fourier_fit.cpp:67-105): least squares on the nodes [-K, K]; a real target
/// is the complex one with zero imaginary part.
inline CoefficientSet fit_mmse(const ArrayXcd& target, const HarmonicGrid& grid, CoeffKind kind) {
  std::vector<double> t(2 * target.size());
  for (size_t i = 0; i < target.size(); ++i) {
    t[2 * i] = target[i].real();
    t[2 * i + 1] = target[i].imag();
  }
  if (target.size() != static_cast<size_t>(2 * grid.half_width + 1))
    throw std::invalid_argument("fit_mmse: target size must be 2K+1");
  sftgpu_coeffs r;
  detail::check(sftgpu_fit_mmse(t.data(), grid.half_width, grid.beta, static_cast<int>(grid.cos_orders.size()),
                                grid.cos_orders.data(), static_cast<int>(grid.sin_orders.size()),
                                grid.sin_orders.data(), static_cast<int>(kind), &r));
  return CoefficientSet::from_raw(r);
}
inline CoefficientSet fit_mmse(const ArrayXd& target, const HarmonicGrid& grid, CoeffKind kind) {
  return fit_mmse(ArrayXcd(target.begin(), target.end()), grid, kind);
}

/// reconstruct (fourier_fit.cpp:107-129): the fitted series at arbitrary points.
inline ArrayXcd reconstruct(const CoefficientSet& coeffs, const ArrayXd& points) {
  const sftgpu_coeffs r = coeffs.raw();
  ArrayXcd out(points.size());
  detail::check(sftgpu_reconstruct(&r, points.data(), static_cast<std::int64_t>(points.size()),
                                   reinterpret_cast<double*>(out.data())));
  return out;
}

struct GaussianFitBundle {
  GaussianParams params{1.0, 1};
  double beta = 0.0;
  int max_order = 0;
  ArrayXd a, b, d;
  double fit_rmse_g = 0.0, fit_rmse_gd = 0.0, fit_rmse_gdd = 0.0;
};
inline GaussianFitBundle fit_gaussian_bundle(const GaussianParams& params, int max_order, double beta) {
  sftgpu_gauss_bundle r;
  detail::check(sftgpu_fit_gaussian_bundle(params.sigma, params.half_width, max_order, beta, &r));
  GaussianFitBundle g;
  g.params = params;
  g.beta = r.beta;
  g.max_order = r.max_order;
  g.a.assign(r.a, r.a + r.max_order + 1);
  g.b.assign(r.b, r.b + r.max_order);
  g.d.assign(r.d, r.d + r.max_order + 1);
  g.fit_rmse_g = r.fit_rmse_g;
  g.fit_rmse_gd = r.fit_rmse_gd;
  g.fit_rmse_gdd = r.fit_rmse_gdd;
  return g;
}
inline double gauss_kernel_rmse(const GaussianFitBundle& bundle, GaussKind kind, int n0) {
  sftgpu_gauss_bundle r;
  std::memset(&r, 0, sizeof(r));
  r.sigma = bundle.params.sigma;
  r.half_width = bundle.params.half_width;
  r.beta = bundle.beta;
  r.max_order = bundle.max_order;
  std::copy(bundle.a.begin(), bundle.a.end(), r.a);
  std::copy(bundle.b.begin(), bundle.b.end(), r.b);
  std::copy(bundle.d.begin(), bundle.d.end(), r.d);
  double v = 0.0;
  detail::check(sftgpu_gauss_kernel_rmse(&r, static_cast<int>(kind), n0, &v));
  return v;
}
inline CoefficientSet fit_morlet_direct(const MorletParams& params, int ps, int pd, double beta, int n0 = 0) {
  sftgpu_coeffs r;
  detail::check(sftgpu_fit_morlet_direct(params.sigma, params.xi, params.half_width, ps, pd, beta, n0, &r));
  return CoefficientSet::from_raw(r);
}
inline CoefficientSet fit_morlet_envelope(const MorletParams& params, int max_order, double beta) {
  sftgpu_coeffs r;
  detail::check(sftgpu_fit_morlet_envelope(params.sigma, params.xi, params.half_width, max_order, beta, &r));
  return CoefficientSet::from_raw(r);
}

struct BetaTuneResult {
  double beta = 0.0;
  double rmse_percent = 0.0;
};
/// tune_beta (fourier_fit.cpp:395-438) over any RMSE profile.
inline BetaTuneResult tune_beta(const std::function<double(double)>& rmse_of_beta, int half_width) {
  auto tramp = [](double beta, void* u) { return (*static_cast<const std::function<double(double)>*>(u))(beta); };
  BetaTuneResult r;
  detail::check(sftgpu_tune_beta(tramp, const_cast<std::function<double(double)>*>(&rmse_of_beta), half_width,
                                 &r.beta, &r.rmse_percent));
  return r;
}
inline BetaTuneResult tune_beta_gauss(const GaussianParams& params, int max_order, int n0 = 0) {
  BetaTuneResult r;
  detail::check(sftgpu_tune_beta_gauss(params.sigma, params.half_width, max_order, n0, &r.beta, &r.rmse_percent));
  return r;
}

// sliding_sum.hpp ----------------------------------------------------------------------
enum class SsVariant { FlatDoubling, Blocked8 };
/// Round / stage schedule of the data-parallel sliding sum (sliding_sum.hpp:23-64).
struct SlidingSumPlan {
  std::int64_t input_size = 0, window = 0;
  int rounds = 0;
  SsVariant variant = SsVariant::FlatDoubling;
  std::int64_t core_budget = 1;
  std::int64_t padded_size = 0;
  int block_rows = 16, block_cols = 8;
  static SlidingSumPlan make(std::int64_t n, std::int64_t window, SsVariant variant = SsVariant::FlatDoubling,
                             std::int64_t core_budget = 1) {
    if (core_budget < 1) throw std::invalid_argument("SlidingSumPlan: M must be >= 1");
    std::int64_t info[5];
    detail::check(sftgpu_sliding_sum_plan(n, window, variant == SsVariant::Blocked8, info));
    SlidingSumPlan p;
    p.input_size = n;
    p.window = window;
    p.variant = variant;
    p.core_budget = core_budget;
    p.rounds = static_cast<int>(info[0]);
    p.padded_size = info[1];
    return p;
  }
  int blocked_stages() const { return blocked_stages_for(window); }
  static int blocked_stages_for(std::int64_t window) {
    int st = 0;
    for (std::int64_t rest = window; rest > 0; rest /= 8) ++st;
    return st;
  }
};
struct RoundRecord {
  int round = 0, stage = 0, r = 0, bit = 0;
  std::int64_t active = 0, adds = 0;
};
struct RoundTrace {
  std::vector<RoundRecord> rounds;
  std::int64_t total_adds() const {
    std::int64_t t = 0;
    for (const auto& rec : rounds) t += rec.adds;
    return t;
  }
};
namespace detail {
// the rounds the GPU kernels execute (K5: flat doubling; K6: three rounds per base-8 digit)
inline void fill_trace(const SlidingSumPlan& p, RoundTrace* tr) {
  if (!tr) return;
  tr->rounds.clear();
  if (p.variant == SsVariant::FlatDoubling) {
    for (int r = 0; r < p.rounds; ++r) {
      const int b = static_cast<int>((p.window >> r) & 1);
      tr->rounds.push_back({r, 0, r, b, p.input_size, p.input_size * (1 + b)});
    }
    return;
  }
  std::int64_t rows = p.padded_size, cols = 1, rest = p.window;
  int g = 0, stage = 0;
  while (rest > 0) {
    const std::int64_t blocks = ((rows + 63) / 64) * cols;
    for (int r = 0; r < 3; ++r) {
      const int b = static_cast<int>((rest >> r) & 1);
      const std::int64_t active = static_cast<std::int64_t>(16 - (1 << r)) * 8 * blocks;
      tr->rounds.push_back({g++, stage, r, b, active, active * (1 + b)});
    }
    rows /= 8;
    cols *= 8;
    rest /= 8;
    ++stage;
  }
}
template <typename T>
constexpr int ss_dtype() {
  if constexpr (std::is_same<T, std::int64_t>::value) return SFTGPU_SS_I64;
  else if constexpr (std::is_same<T, double>::value) return SFTGPU_SS_F64;
  else {
    static_assert(std::is_same<T, std::complex<double>>::value, "sliding sums: int64, double or complex<double>");
    return SFTGPU_SS_C128;
  }
}
template <typename T>
std::vector<T> sliding_sum(const std::vector<T>& f, std::int64_t window, bool blocked, RoundTrace* trace) {
  const SlidingSumPlan p = SlidingSumPlan::make(static_cast<std::int64_t>(f.size()), window,
                                                blocked ? SsVariant::Blocked8 : SsVariant::FlatDoubling);
  std::vector<T> out(f.size() - static_cast<size_t>(window) + 1);
  check(sftgpu_sliding_sum_host(ss_dtype<T>(), blocked ? 1 : 0, f.data(), static_cast<std::int64_t>(f.size()), window,
                                out.data()));
  fill_trace(p, trace);
  return out;
}
}  // namespace detail
/// Paper Algorithm 1 (sliding_sum.hpp:89-121) on the GPU (K5), bit-identical addition trees.
template <typename T>
std::vector<T> sliding_sum_flat(const std::vector<T>& f, std::int64_t window, int /*workers*/ = 1,
                                RoundTrace* trace = nullptr) {
  return detail::sliding_sum(f, window, false, trace);
}
/// Paper Algorithms 2-3 (sliding_sum.hpp:144-234) on the GPU (K6), bit-identical addition trees.
template <typename T>
std::vector<T> sliding_sum_blocked8(const std::vector<T>& f, std::int64_t window, int /*workers*/ = 1,
                                    RoundTrace* trace = nullptr) {
  return detail::sliding_sum(f, window, true, trace);
}
inline std::pair<std::int64_t, std::int64_t> blocked8_layout(std::int64_t index, int stages) {
  std::int64_t div = 1;
  for (int t = 0; t < stages; ++t) div *= 8;
  std::int64_t rem = index % div, col = 0;
  for (int t = 0; t < stages; ++t) {
    col = col * 8 + rem % 8;
    rem /= 8;
  }
  return {index / div, col};
}

struct CostReport {
  std::int64_t parallel_steps = 0;
  int outer_iterations = 0;
  std::int64_t total_adds = 0;
  std::int64_t total_mults = 0;
  std::string predicted_regime;
};
/// cost_model (src/sliding_sum.cpp:7-40): exact operation counts of a plan's rounds.
inline CostReport cost_model(const SlidingSumPlan& plan) {
  std::int64_t info[5];
  detail::check(sftgpu_sliding_sum_plan(plan.input_size, plan.window, plan.variant == SsVariant::Blocked8, info));
  CostReport r;
  r.parallel_steps = info[3];
  r.outer_iterations = plan.variant == SsVariant::Blocked8 ? plan.blocked_stages() : 1;
  r.total_adds = info[4];
  r.total_mults = 0;
  r.predicted_regime = plan.core_budget >= plan.input_size ? "O(log2 L) parallel time (M >= N)"
                                                           : "O(N log2 L / M) parallel time (M < N)";
  return r;
}
struct MethodOpCounts {
  std::int64_t mults = 0, adds = 0;
  std::string regime;
};
/// src/sliding_sum.cpp:42-66: method-level operation counts of the benchmark comparisons.
inline MethodOpCounts sft_method_counts(std::int64_t n, int orders, std::int64_t half_width, std::int64_t core_budget) {
  MethodOpCounts c;
  c.mults = 7 * n * orders;
  c.adds = n * orders * (2 * half_width + 1);
  c.regime = core_budget >= n ? "O(P log2 K) time (M >= N)" : "O(N P log2 K / M) time (M < N)";
  return c;
}
inline MethodOpCounts conv_method_counts(std::int64_t n, double sigma, std::int64_t core_budget) {
  MethodOpCounts c;
  const std::int64_t window = static_cast<std::int64_t>(std::llround(6.0 * sigma)) + 1;
  c.mults = n * window;
  c.adds = n * window;
  c.regime = core_budget >= c.adds ? "O(log2 sigma) time (M >= N(6 sigma + 1))" : "O(N sigma log2 sigma / M) time";
  return c;
}

}  // namespace sft
