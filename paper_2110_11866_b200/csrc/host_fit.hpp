// Host precompute for the SFT/ASFT path: MMSE trigonometric fits, effective
// kernels and spec factories. These run once per (sigma, xi, P, n0) before any
// signal is processed (the reference builds specs before its timed loop,
// proj/src/eval.cpp:186-190), so they stay on the CPU in fp64.
//
// Restates proj/src/fourier_fit.cpp, proj/include/sft/kernels.hpp:14-73 and the
// spec factories of proj/src/transforms.cpp:16-242 without Eigen.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace sftb {

using cd = std::complex<double>;

class FitDegenerate : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

enum class TKind { Gauss = 0, GaussD, GaussDD, MorletDirect, MorletMultiply, TruncGauss, TruncMorlet };
enum class GKind { Value = 0, Deriv1, Deriv2 };
enum CoeffKind { kGaussCos = 0, kGaussDerivSin, kGaussDeriv2Cos, kMorletDirect, kMorletMultiply };

// proj/include/sft/kernels.hpp:15-52
struct GaussP {
  double sigma;
  int K;
  GaussP(double s, int k = 0);
  double gamma() const { return 1.0 / (2.0 * sigma * sigma); }
  static int default_K(double sigma);
};

struct MorletP {
  double sigma, xi;
  int K;
  MorletP(double s, double x, int k = 0);
  double kappa() const;
  double cxi() const;
  double gamma() const { return 1.0 / (2.0 * sigma * sigma); }
};

double gauss(const GaussP& p, double t);
double gauss_d(const GaussP& p, double t);
double gauss_dd(const GaussP& p, double t);
cd morlet(const MorletP& p, double t);

// proj/include/sft/fourier_fit.hpp:18-46
struct Grid {
  int K = 1;
  double beta = 1.0;
  std::vector<int> cos_p, sin_p;
  Grid() = default;
  Grid(int k, double b, std::vector<int> c, std::vector<int> s);
  size_t size() const { return cos_p.size() + sin_p.size(); }
};

struct Coeffs {
  int kind = 0;
  Grid grid;
  std::vector<cd> cc, sc;
  double fit_rmse = 0.0;
  double sigma = 0.0, xi = 0.0;
  int n0 = 0;
};

struct Bundle {
  GaussP params{1.0, 1};
  double beta = 0.0;
  int P = 0;
  std::vector<double> a, b, d;
  double rmse_g = 0, rmse_gd = 0, rmse_gdd = 0;
};

struct Taps {
  std::vector<cd> taps;
  int64_t lo = 0;
};

Coeffs fit_mmse(const std::vector<cd>& target, const Grid& grid, int kind);
std::vector<cd> reconstruct(const Coeffs& c, const std::vector<double>& q);
Bundle fit_gaussian_bundle(const GaussP& params, int P, double beta);
Taps gauss_effective_taps(const Bundle& b, GKind kind, int n0);
Taps morlet_direct_effective_taps(const Coeffs& c, const MorletP& p, int n0);
Taps morlet_multiply_effective_taps(const Coeffs& env, const MorletP& p, int n0);
double gauss_kernel_rmse(const Bundle& b, GKind kind, int n0);
Coeffs fit_morlet_direct(const MorletP& p, int ps, int pd, double beta, int n0);
Coeffs fit_morlet_envelope(const MorletP& p, int P, double beta);
double morlet_direct_kernel_rmse(const MorletP& p, int ps, int pd, int n0, Coeffs* out = nullptr);
double morlet_multiply_kernel_rmse(const MorletP& p, int pm, int n0, Coeffs* out = nullptr);
int select_optimal_ps(const MorletP& p, int pd, int n0);
struct BetaTune {
  double beta = 0, rmse = 0;
};
BetaTune tune_beta_gauss(const GaussP& p, int P, int n0);
// tune_beta (proj/src/fourier_fit.cpp:395-438) over a caller-supplied RMSE profile
BetaTune tune_beta_callback(double (*f)(double, void*), void* user, int K);

// TransformSpec (proj/include/sft/transforms.hpp:23-41)
struct Options {
  bool has_K = false;
  int K = 0;
  bool has_beta = false;
  double beta = 0.0;
  bool tune = false;
  bool has_ps = false;
  int ps = 0;
  int strategy = 2;
  int precision = 1;
};

struct Spec {
  TKind kind = TKind::Gauss;
  bool has_gauss = false, has_morlet = false;
  GaussP gparams{1.0, 1};
  MorletP mparams{1.0, 1.0, 1};
  int max_order = 0, ps = 0, pd = 0;
  double beta = 0.0;
  int n0 = 0;
  double alpha = 0.0;
  int strategy = 2, precision = 1;
  std::string abbrev;
  double kernel_rmse = 0.0;
  Bundle bundle;
  Coeffs morlet, envelope;
  bool has_bundle = false, has_mcoef = false, has_env = false;
};

struct Abbrev {
  TKind kind;
  int n0 = 0, order = 0;
};
Abbrev parse_abbreviation(const std::string& a);
std::string encode_abbreviation(TKind k, int n0, int order);
Spec make_gauss_spec(double sigma, GKind kind, int P, int n0, const Options& o);
Spec make_morlet_direct_spec(double sigma, double xi, int pd, int n0, const Options& o);
Spec make_morlet_multiply_spec(double sigma, double xi, int pm, int n0, const Options& o);
Spec make_transform_spec(const std::string& a, double sigma, double xi, const Options& o);
Taps effective_kernel(const Spec& s);
Taps sample_gauss(const GaussP& p);
Taps sample_morlet(const MorletP& p);
double relative_rmse(const std::vector<cd>& approx, const std::vector<cd>& truth);
std::string write_coefficient_sets(const std::vector<Coeffs>& sets);
std::vector<Coeffs> read_coefficient_sets(const std::string& text);
Spec morlet_direct_spec_from_coeffs(const Coeffs& c, int precision, int strategy, bool recompute_rmse);

}  // namespace sftb
