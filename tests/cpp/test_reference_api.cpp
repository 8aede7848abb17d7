// The reference's own engine and transform suites (proj/tests/test_engine.cpp,
// proj/tests/test_transforms.cpp), written against the drop-in C++ API
// (include/sft_b200/sft.hpp) so every case runs the B200 kernels through the C ABI.
// Checkers are the reference's: brute-force defining sums, closed forms, and
// truncated convolution with the effective kernel (here the GPU fp64 kernel K3).
#include <algorithm>
#include <cmath>
#include <complex>

#include "doctest_lite.hpp"
#include "sft_b200/sft.hpp"

using namespace sft;
using doctest::Approx;

namespace {

ComponentSeq brute_components(const Signal& sig, int k, double omega, double alpha) {
  ComponentSeq out;
  out.c.assign(static_cast<size_t>(sig.size()), 0.0);
  out.s.assign(static_cast<size_t>(sig.size()), 0.0);
  for (std::int64_t n = 0; n < sig.size(); ++n) {
    double c = 0.0, s = 0.0;
    for (int lag = -k; lag <= k; ++lag) {
      const double w = std::exp(-alpha * lag) * extended_sample(sig, n - lag);
      c += w * std::cos(omega * lag);
      s += w * std::sin(omega * lag);
    }
    out.c[n] = c;
    out.s[n] = s;
  }
  return out;
}

SftConfig config(int k, double beta, int p, double alpha, Strategy strategy,
                 Precision precision = Precision::Double) {
  SftConfig cfg{k, beta, OrderSpec::order(p)};
  cfg.alpha = alpha;
  cfg.strategy = strategy;
  cfg.precision = precision;
  return cfg;
}

double max_abs_diff(const ComponentSeq& a, const ComponentSeq& b) {
  double m = 0.0;
  for (size_t i = 0; i < a.c.size(); ++i) m = std::max({m, std::fabs(a.c[i] - b.c[i]), std::fabs(a.s[i] - b.s[i])});
  return m;
}

double maxabs(const ArrayXd& v) {
  double m = 0.0;
  for (double x : v) m = std::max(m, std::fabs(x));
  return m;
}

double exactness_error(const Signal& sig, const TransformSpec& spec) {
  const TransformResult result = apply_transform(sig, spec);
  const ArrayXcd reference = truncated_convolution(sig, effective_kernel(spec));
  double scale = 1e-30, err = 0.0;
  for (size_t i = 0; i < reference.size(); ++i) {
    scale = std::max(scale, std::abs(reference[i]));
    err = std::max(err, std::abs(result.values[i] - reference[i]));
  }
  return err / scale;
}

}  // namespace

TEST_CASE("constant signal: order zero sums the window") {
  const int k = 8;
  const Signal ones = make_test_signal(TestSignalKind::Constant, 40, 0);
  for (Strategy strategy : {Strategy::KernelIntegral, Strategy::Recursive1, Strategy::Recursive2}) {
    const ComponentSeq comp = sft_components(ones, config(k, M_PI / k, 0, 0.0, strategy));
    for (std::int64_t n = 0; n < 40; ++n) {
      CHECK(comp.c[n] == Approx(2.0 * k + 1.0).epsilon(1e-12));
      CHECK(std::abs(comp.s[n]) < 1e-10);
    }
  }
}

TEST_CASE("all strategies agree with brute-force window sums") {
  const int k = 8;
  const Signal noise = make_test_signal(TestSignalKind::SeededNoise, 64, 7);
  for (double beta : {M_PI / k, 1.07 * M_PI / k}) {
    const ComponentSeq reference = brute_components(noise, k, beta * 3, 0.0);
    for (Strategy strategy : {Strategy::KernelIntegral, Strategy::Recursive1, Strategy::Recursive2}) {
      const ComponentSeq comp = sft_components(noise, config(k, beta, 3, 0.0, strategy));
      CHECK(max_abs_diff(comp, reference) < 1e-10);
    }
  }
}

TEST_CASE("single precision stays within the coarse tolerance") {
  const int k = 12;
  const Signal noise = make_test_signal(TestSignalKind::SeededNoise, 200, 11);
  const ComponentSeq reference = brute_components(noise, k, M_PI / k * 3, 0.0);
  const double bound = 1e-4 * (2 * k + 1) * maxabs(noise.samples);
  for (Strategy strategy : {Strategy::KernelIntegral, Strategy::Recursive1, Strategy::Recursive2}) {
    const ComponentSeq comp = sft_components(noise, config(k, M_PI / k, 3, 0.0, strategy, Precision::Single));
    CHECK(max_abs_diff(comp, reference) < bound);
  }
}

TEST_CASE("attenuated components match brute-force attenuated sums") {
  const int k = 8;
  const double alpha = 0.05;
  const Signal noise = make_test_signal(TestSignalKind::SeededNoise, 64, 19);
  const ComponentSeq reference = brute_components(noise, k, M_PI / k * 2, alpha);
  for (Strategy strategy : {Strategy::KernelIntegral, Strategy::Recursive1, Strategy::Recursive2}) {
    const ComponentSeq comp = asft_components(noise, config(k, M_PI / k, 2, alpha, strategy));
    CHECK(max_abs_diff(comp, reference) < 1e-9);
  }
}

TEST_CASE("real-frequency mode reproduces integer order exactly") {
  const int k = 9;
  const double beta = M_PI / k;
  const Signal noise = make_test_signal(TestSignalKind::SeededNoise, 70, 13);
  SftConfig integer_cfg = config(k, beta, 3, 0.0, Strategy::KernelIntegral);
  SftConfig real_cfg = integer_cfg;
  real_cfg.order = OrderSpec::frequency(beta * 3);
  const ComponentSeq a = sft_components(noise, integer_cfg);
  const ComponentSeq b = sft_components(noise, real_cfg);
  for (std::int64_t n = 0; n < 70; ++n) {
    CHECK(a.c[n] == b.c[n]);
    CHECK(a.s[n] == b.s[n]);
  }
}

TEST_CASE("engine validation") {
  const Signal noise = make_test_signal(TestSignalKind::SeededNoise, 16, 1);
  CHECK_THROWS_AS(asft_components(noise, config(4, M_PI / 4, 1, 0.0, Strategy::Recursive1)), std::invalid_argument);
  CHECK_THROWS_AS(sft_components(noise, config(4, M_PI / 4, 1, 0.5, Strategy::Recursive1)), std::invalid_argument);
  CHECK_THROWS_AS(sft_components(noise, config(0, 1.0, 0, 0.0, Strategy::Recursive1)), std::invalid_argument);
  SftConfig rf = config(8, M_PI / 8, 1, 0.0, Strategy::Recursive1);
  rf.order = OrderSpec::frequency(0.3);
  CHECK_THROWS_AS(sft_components(noise, rf), std::invalid_argument);
}

TEST_CASE("every transform equals convolution with its fitted kernel") {
  const Signal noise = make_test_signal(TestSignalKind::SeededNoise, 96, 101);
  TransformOptions options;
  for (Strategy strategy : {Strategy::KernelIntegral, Strategy::Recursive1, Strategy::Recursive2}) {
    options.strategy = strategy;
    for (int n0 : {0, 1}) {
      for (GaussKind kind : {GaussKind::Value, GaussKind::Deriv1, GaussKind::Deriv2})
        CHECK(exactness_error(noise, make_gauss_spec(6.0, kind, 4, n0, options)) < 1e-9);
      CHECK(exactness_error(noise, make_morlet_direct_spec(8.0, 6.0, 5, n0, options)) < 1e-9);
      CHECK(exactness_error(noise, make_morlet_multiply_spec(8.0, 6.0, 3, n0, options)) < 1e-9);
    }
  }
}

TEST_CASE("zero shift reduces to the plain transform") {
  const Signal noise = make_test_signal(TestSignalKind::SeededNoise, 80, 3);
  const TransformSpec sft = make_gauss_spec(8.0, GaussKind::Value, 4, 0, {});
  TransformSpec asft_zero = sft;
  asft_zero.n0 = 0;
  asft_zero.alpha = 0.0;
  const TransformResult a = gauss_smooth(noise, sft);
  const TransformResult b = gauss_smooth(noise, asft_zero);
  double m = 0.0;
  for (size_t i = 0; i < a.values.size(); ++i) m = std::max(m, std::abs(a.values[i] - b.values[i]));
  CHECK(m == 0.0);
}

TEST_CASE("reference paths use the 3-sigma truncated true kernels") {
  const Signal impulse = make_test_signal(TestSignalKind::Impulse, 97, 0, BoundaryPolicy::Zero);
  const TransformSpec gct3 = make_transform_spec("GCT3", 8.0, 0.0, {});
  const TransformResult rg = apply_transform(impulse, gct3);
  CHECK(rg.values[48].real() == Approx(gauss(GaussianParams(8.0), 0)).epsilon(1e-14));
  CHECK(rg.values[48 + 24].real() == Approx(gauss(GaussianParams(8.0), 24)).epsilon(1e-12));
  CHECK(rg.values[48 + 25].real() == 0.0);
  const TransformSpec mct3 = make_transform_spec("MCT3", 8.0, 6.0, {});
  const TransformResult rm = apply_transform(impulse, mct3);
  const MorletParams params(8.0, 6.0);
  CHECK(rm.values[48].real() == Approx(morlet(params, 0).real()).epsilon(1e-13));
  CHECK(rm.values[40].imag() == Approx(morlet(params, -8).imag()).epsilon(1e-12).scale(1.0));
}

TEST_CASE("single-precision transforms track the double-precision results") {
  const Signal noise = make_test_signal(TestSignalKind::SeededNoise, 256, 33);
  for (int n0 : {0, 2}) {
    TransformSpec spec = make_gauss_spec(12.0, GaussKind::Value, 4, n0, {});
    const TransformResult ref = gauss_smooth(noise, spec);
    spec.precision = Precision::Single;
    const TransformResult lo = gauss_smooth(noise, spec);
    double scale = 0.0, err = 0.0;
    for (size_t i = 0; i < ref.values.size(); ++i) {
      scale = std::max(scale, std::abs(ref.values[i]));
      err = std::max(err, std::abs(lo.values[i] - ref.values[i]));
    }
    CHECK(err < 1e-3 * scale);
  }
}

TEST_CASE("abbreviation factory covers the published filter names") {
  for (const char* name : {"GDP6", "MDP5", "MDP6", "MDP7", "MDS5P5", "MDS5P7", "MMP2", "MMP3", "MMS5P3", "GCT3", "MCT3"}) {
    const double sigma = name[0] == 'G' ? 16.0 : 60.0;
    const TransformSpec spec = make_transform_spec(name, sigma, 10.0, {});
    const Signal noise = make_test_signal(TestSignalKind::SeededNoise, 64, 5);
    const TransformResult result = apply_transform(noise, spec);
    CHECK(result.values.size() == 64);
    bool finite = true;
    for (auto v : result.values) finite = finite && std::isfinite(v.real()) && std::isfinite(v.imag());
    CHECK(finite);
  }
  const AbbrevInfo direct = parse_abbreviation("MDS5P7");
  CHECK(direct.kind == TransformKind::MorletDirect);
  CHECK(direct.n0 == 5);
  CHECK(direct.order == 7);
  CHECK_THROWS_AS(parse_abbreviation("XP3"), std::invalid_argument);
  CHECK_THROWS_AS(parse_abbreviation("MDP0"), std::invalid_argument);
}

TEST_CASE("shift validation") {
  CHECK_THROWS_AS(make_gauss_spec(8.0, GaussKind::Value, 4, 3, {}), std::invalid_argument);
  CHECK_THROWS_AS(make_morlet_direct_spec(8.0, 6.0, 5, 3, {}), std::invalid_argument);
  CHECK_NOTHROW(make_gauss_spec(8.0, GaussKind::Value, 4, 2, {}));
}

// ---- the rest of the reference's public surface (engine.hpp:82-109, sliding_sum.hpp,
// fourier_fit.hpp), proj/tests/test_engine.cpp / test_sliding_sum.cpp / test_fourier_fit.cpp
TEST_CASE("window state: prefix route equals the in-window recurrence") {
  const Signal sig = make_test_signal(TestSignalKind::SeededNoise, 300, 4);
  const WindowState st = sliding_window_state(sig, config(12, M_PI / 12, 3, 0.0, Strategy::KernelIntegral));
  double m = 0.0, scale = 0.0;
  for (size_t i = 0; i < st.via_prefix.size(); ++i) {
    m = std::max(m, std::abs(st.via_prefix[i] - st.via_recurrence[i]));
    scale = std::max(scale, std::abs(st.via_recurrence[i]));
  }
  CHECK(m < 1e-10 * scale);
  CHECK_THROWS_AS(sliding_window_state(sig, config(12, M_PI / 12, 3, 0.1, Strategy::KernelIntegral)),
                  std::invalid_argument);
}

TEST_CASE("sliding-sum route equals the kernel integral") {
  const Signal sig = make_test_signal(TestSignalKind::SeededNoise, 500, 9);
  for (int p : {0, 2, 5}) {
    const SftConfig cfg = config(20, M_PI / 20, p, 0.003, Strategy::KernelIntegral);
    CHECK(max_abs_diff(sft_via_sliding_sum(sig, cfg), asft_components(sig, cfg)) < 1e-9);
  }
  CHECK_THROWS_AS(sft_via_sliding_sum(make_test_signal(TestSignalKind::SeededNoise, 20000, 1),
                                      config(16, M_PI / 16, 1, 0.1, Strategy::KernelIntegral)),
                  std::invalid_argument);
}

TEST_CASE("stability probe: single precision against double") {
  const Signal sig = make_test_signal(TestSignalKind::SeededNoise, 4000, 11);
  const StabilityReport r = stability_probe(sig, config(64, M_PI / 64, 2, 0.0, Strategy::KernelIntegral));
  CHECK(r.abs_error.size() == 4000);
  CHECK(r.reference_scale > 0.0);
  CHECK(r.max_component_error < 1e-5);
  CHECK(r.max_state_magnitude > 0.0);
}

TEST_CASE("sliding sums: known answers and the blocked8 trace") {
  const std::vector<std::int64_t> f = {1, 2, 3, 4, 5};
  const std::vector<std::int64_t> want = {6, 9, 12};
  CHECK(sliding_sum_flat(f, 3) == want);
  CHECK(sliding_sum_blocked8(f, 3) == want);
  std::vector<double> g(500);
  for (size_t i = 0; i < g.size(); ++i) g[i] = std::sin(0.37 * static_cast<double>(i)) + 1e-3 * static_cast<double>(i);
  RoundTrace tr;
  const std::vector<double> a = sliding_sum_blocked8(g, 37, 1, &tr);
  const std::vector<double> b = sliding_sum_flat(g, 37);
  CHECK(a.size() == 464);
  double m = 0.0;
  for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::fabs(a[i] - b[i]));
  CHECK(m < 1e-12);
  CHECK(tr.rounds.size() == 6);  // test_output.txt:41
  CHECK(tr.total_adds() == 7744);
  const CostReport cr = cost_model(SlidingSumPlan::make(500, 37, SsVariant::Blocked8));
  CHECK(cr.total_adds == 7744);
  CHECK(cr.outer_iterations == 2);
  CHECK(cost_model(SlidingSumPlan::make(500, 37)).parallel_steps == 6);
  const MethodOpCounts sc = sft_method_counts(1000, 7, 24, 1);
  CHECK(sc.mults == 49000);
  CHECK(conv_method_counts(1000, 8.0, 1).adds == 49000);
}

TEST_CASE("fits: reconstruct, Gaussian bundle, Morlet fits, beta tuning") {
  const GaussianParams gp(6.0);
  const GaussianFitBundle b = fit_gaussian_bundle(gp, 6, M_PI / gp.half_width);
  CHECK(b.a.size() == 7);
  CHECK(b.b.size() == 6);
  CHECK(b.fit_rmse_g < 1.0);
  CHECK(gauss_kernel_rmse(b, GaussKind::Value, 0) < 1.0);
  // fit_mmse of the Gaussian on [-K, K] reproduces the bundle's cos coefficients
  ArrayXd target(2 * gp.half_width + 1);
  for (int k = -gp.half_width; k <= gp.half_width; ++k) target[k + gp.half_width] = gauss(gp, k);
  std::vector<int> cos_p = {0, 1, 2, 3, 4, 5, 6};
  const CoefficientSet cs = fit_mmse(target, HarmonicGrid(gp.half_width, M_PI / gp.half_width, cos_p, {}),
                                     CoeffKind::GaussCos);
  for (int p = 0; p <= 6; ++p) CHECK(std::fabs(cs.cos_coeffs[p].real() - b.a[p]) < 1e-12);
  ArrayXd pts = {-3.0, 0.0, 2.5};
  const ArrayXcd rec = reconstruct(cs, pts);
  for (size_t i = 0; i < pts.size(); ++i) CHECK(std::fabs(rec[i].real() - gauss(gp, pts[i])) < 2e-3 * gauss(gp, 0));
  const MorletParams mp(60.0, 8.0);
  const CoefficientSet md = fit_morlet_direct(mp, 5, 6, M_PI / mp.half_width, 0);
  CHECK(md.cos_coeffs.size() == 6);
  const CoefficientSet env = fit_morlet_envelope(mp, 3, M_PI / mp.half_width);
  CHECK(env.cos_coeffs.size() == 4);
  // generic tuner on a known profile: minimum of (beta - 0.9 pi/K)^2 + 1
  const int K = 40;
  const BetaTuneResult t = tune_beta([&](double beta) { return (beta - 0.9 * M_PI / K) * (beta - 0.9 * M_PI / K) + 1.0; }, K);
  CHECK(std::fabs(t.beta - 0.9 * M_PI / K) < 1e-3 * M_PI / K);
  CHECK(std::fabs(t.rmse_percent - 1.0) < 1e-9);
  const BetaTuneResult tg = tune_beta_gauss(gp, 4, 0);
  CHECK(tg.beta > 0.5 * M_PI / gp.half_width);
  CHECK(tg.beta < 1.5 * M_PI / gp.half_width);
}

DOCTEST_LITE_MAIN
