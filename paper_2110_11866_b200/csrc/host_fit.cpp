// Host precompute: MMSE fits, effective kernels, spec factories.
// See host_fit.hpp; each function cites the reference routine it restates.
#include "host_fit.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <functional>
#include <cstdio>
#include <map>
#include <numeric>
#include <sstream>

namespace sftb {

// ------------------------------------------------------------------ kernels
// proj/include/sft/kernels.hpp:15-73
int GaussP::default_K(double s) { return static_cast<int>(std::ceil(3.0 * s)); }

GaussP::GaussP(double s, int k) : sigma(s), K(k > 0 ? k : default_K(s)) {
  if (!(sigma > 0.0)) throw std::invalid_argument("GaussianParams: sigma must be > 0");
  if (K < 1) throw std::invalid_argument("GaussianParams: K must be >= 1");
}

MorletP::MorletP(double s, double x, int k) : sigma(s), xi(x), K(k > 0 ? k : GaussP::default_K(s)) {
  if (!(sigma > 0.0)) throw std::invalid_argument("MorletParams: sigma must be > 0");
  if (!(xi > 0.0)) throw std::invalid_argument("MorletParams: xi must be > 0");
  if (K < 1) throw std::invalid_argument("MorletParams: K must be >= 1");
}
double MorletP::kappa() const { return std::exp(-0.5 * xi * xi); }
double MorletP::cxi() const {
  return 1.0 / std::sqrt(1.0 + std::exp(-xi * xi) - 2.0 * std::exp(-0.75 * xi * xi));
}

double gauss(const GaussP& p, double t) {
  const double g = p.gamma();
  return std::sqrt(g / M_PI) * std::exp(-g * t * t);
}
double gauss_d(const GaussP& p, double t) { return -2.0 * p.gamma() * t * gauss(p, t); }
double gauss_dd(const GaussP& p, double t) {
  const double g = p.gamma();
  return (4.0 * g * g * t * t - 2.0 * g) * gauss(p, t);
}
cd morlet(const MorletP& p, double t) {
  const double env =
      p.cxi() / (std::pow(M_PI, 0.25) * std::sqrt(p.sigma)) * std::exp(-t * t / (2.0 * p.sigma * p.sigma));
  const double ph = p.xi * t / p.sigma;
  return env * (cd(std::cos(ph), std::sin(ph)) - p.kappa());
}

Taps sample_gauss(const GaussP& p) {
  Taps t;
  t.lo = -p.K;
  for (int i = -p.K; i <= p.K; ++i) t.taps.push_back(gauss(p, i));
  return t;
}
Taps sample_morlet(const MorletP& p) {
  Taps t;
  t.lo = -p.K;
  for (int i = -p.K; i <= p.K; ++i) t.taps.push_back(morlet(p, i));
  return t;
}

// proj/include/sft/metrics.hpp:14-23
double relative_rmse(const std::vector<cd>& a, const std::vector<cd>& t) {
  if (a.size() != t.size()) throw std::invalid_argument("relative_rmse: grids differ");
  double den = 0.0, num = 0.0;
  for (size_t i = 0; i < t.size(); ++i) {
    den += std::norm(t[i]);
    num += std::norm(a[i] - t[i]);
  }
  if (!(den > 0.0)) throw std::invalid_argument("relative_rmse: truth has zero norm");
  return std::sqrt(num / den) * 100.0;
}

// ------------------------------------------------------------------ grid / fit
// proj/include/sft/fourier_fit.hpp:24-46
Grid::Grid(int k, double b, std::vector<int> c, std::vector<int> s)
    : K(k), beta(b), cos_p(std::move(c)), sin_p(std::move(s)) {
  if (K < 1) throw std::invalid_argument("HarmonicGrid: K must be >= 1");
  if (!(beta > 0.0)) throw std::invalid_argument("HarmonicGrid: beta must be > 0");
  for (int p : sin_p)
    if (p == 0) throw std::invalid_argument("HarmonicGrid: sin order 0 is identically zero");
  auto distinct = [](const std::vector<int>& v) {
    for (size_t i = 0; i < v.size(); ++i)
      for (size_t j = i + 1; j < v.size(); ++j)
        if (v[i] == v[j]) throw std::invalid_argument("HarmonicGrid: duplicate order");
  };
  distinct(cos_p);
  distinct(sin_p);
  if (size() == 0) throw std::invalid_argument("HarmonicGrid: empty basis");
  if (size() > static_cast<size_t>(2 * K + 1))
    throw std::invalid_argument("HarmonicGrid: more basis functions than nodes");
}

namespace {

std::vector<double> nodes_of(int K) {
  std::vector<double> q(2 * static_cast<size_t>(K) + 1);
  for (int i = 0; i <= 2 * K; ++i) q[i] = static_cast<double>(i - K);
  return q;
}

// Column-major design matrix (proj/src/fourier_fit.cpp:12-23): cos columns, then sin.
std::vector<double> design(const Grid& g, const std::vector<double>& q) {
  const size_t R = q.size(), Cn = g.size();
  std::vector<double> D(R * Cn);
  size_t col = 0;
  for (int p : g.cos_p) {
    const double bp = g.beta * p;
    for (size_t r = 0; r < R; ++r) D[col * R + r] = std::cos(bp * q[r]);
    ++col;
  }
  for (int p : g.sin_p) {
    const double bp = g.beta * p;
    for (size_t r = 0; r < R; ++r) D[col * R + r] = std::sin(bp * q[r]);
    ++col;
  }
  return D;
}

// Symmetric eigenvalues by cyclic Jacobi (condition estimate only).
std::vector<double> sym_eigenvalues(std::vector<double> A, int n) {
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < n; ++i) {
      diag += A[i * n + i] * A[i * n + i];
      for (int j = i + 1; j < n; ++j) off += A[i * n + j] * A[i * n + j];
    }
    if (off <= 1e-30 * diag) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (apq == 0.0) continue;
        const double app = A[p * n + p], aqq = A[q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
      }
  }
  std::vector<double> ev(n);
  for (int i = 0; i < n; ++i) ev[i] = A[i * n + i];
  return ev;
}

// LDL^T with symmetric diagonal pivoting (the factorisation Eigen::LDLT performs).
struct Ldlt {
  int n;
  std::vector<double> L;     // unit lower, row-major n*n
  std::vector<double> Dg;
  std::vector<int> perm;     // row i of factored matrix = original row perm[i]
  explicit Ldlt(std::vector<double> A, int n_) : n(n_), L(n_ * n_, 0.0), Dg(n_), perm(n_) {
    std::iota(perm.begin(), perm.end(), 0);
    for (int k = 0; k < n; ++k) {
      int piv = k;
      double best = std::abs(A[k * n + k]);
      for (int i = k + 1; i < n; ++i)
        if (std::abs(A[i * n + i]) > best) {
          best = std::abs(A[i * n + i]);
          piv = i;
        }
      if (piv != k) {
        for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[piv * n + j]);
        for (int i = 0; i < n; ++i) std::swap(A[i * n + k], A[i * n + piv]);
        for (int j = 0; j < k; ++j) std::swap(L[k * n + j], L[piv * n + j]);
        std::swap(perm[k], perm[piv]);
      }
      const double dk = A[k * n + k];
      Dg[k] = dk;
      L[k * n + k] = 1.0;
      for (int i = k + 1; i < n; ++i) {
        const double lik = dk != 0.0 ? A[i * n + k] / dk : 0.0;
        L[i * n + k] = lik;
      }
      for (int i = k + 1; i < n; ++i)
        for (int j = k + 1; j <= i; ++j) {
          A[i * n + j] -= L[i * n + k] * dk * L[j * n + k];
          A[j * n + i] = A[i * n + j];
        }
    }
  }
  std::vector<double> solve(const std::vector<double>& b) const {
    std::vector<double> y(n);
    for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < i; ++j) y[i] -= L[i * n + j] * y[j];
    for (int i = 0; i < n; ++i) y[i] = Dg[i] != 0.0 ? y[i] / Dg[i] : 0.0;
    for (int i = n - 1; i >= 0; --i)
      for (int j = i + 1; j < n; ++j) y[i] -= L[j * n + i] * y[j];
    std::vector<double> x(n);
    for (int i = 0; i < n; ++i) x[perm[i]] = y[i];
    return x;
  }
};

}  // namespace

// proj/src/fourier_fit.cpp:67-105 (with the Gram solver of :25-40)
Coeffs fit_mmse(const std::vector<cd>& target, const Grid& grid, int kind) {
  const std::vector<double> q = nodes_of(grid.K);
  if (target.size() != q.size())
    throw std::invalid_argument("fit_mmse: target must be sampled on [-K, K]");
  for (const cd& v : target)
    if (!std::isfinite(v.real()) || !std::isfinite(v.imag()))
      throw std::invalid_argument("fit_mmse: target must be finite");
  const size_t R = q.size();
  const int n = static_cast<int>(grid.size());
  const std::vector<double> D = design(grid, q);
  std::vector<double> G(static_cast<size_t>(n) * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double acc = 0.0;
      const double* ci = &D[static_cast<size_t>(i) * R];
      const double* cj = &D[static_cast<size_t>(j) * R];
      for (size_t r = 0; r < R; ++r) acc += ci[r] * cj[r];
      G[i * n + j] = G[j * n + i] = acc;
    }
  const std::vector<double> ev = sym_eigenvalues(G, n);
  const double lo = *std::min_element(ev.begin(), ev.end());
  const double hi = *std::max_element(ev.begin(), ev.end());
  if (!(lo > 0.0) || hi / lo > 1e12)
    throw FitDegenerate("fit_mmse: Gram matrix condition estimate exceeds 1e12");
  const Ldlt ldlt(G, n);
  std::vector<double> bre(n, 0.0), bim(n, 0.0);
  for (int c = 0; c < n; ++c) {
    const double* col = &D[static_cast<size_t>(c) * R];
    double sr = 0.0, si = 0.0;
    for (size_t r = 0; r < R; ++r) {
      sr += col[r] * target[r].real();
      si += col[r] * target[r].imag();
    }
    bre[c] = sr;
    bim[c] = si;
  }
  const std::vector<double> re = ldlt.solve(bre), im = ldlt.solve(bim);
  Coeffs out;
  out.kind = kind;
  out.grid = grid;
  const size_t nc = grid.cos_p.size();
  for (size_t i = 0; i < nc; ++i) out.cc.emplace_back(re[i], im[i]);
  for (size_t i = nc; i < static_cast<size_t>(n); ++i) out.sc.emplace_back(re[i], im[i]);
  double rn = 0.0, tn = 0.0;
  for (size_t r = 0; r < R; ++r) {
    double fr = 0.0, fi = 0.0;
    for (int c = 0; c < n; ++c) {
      fr += D[static_cast<size_t>(c) * R + r] * re[c];
      fi += D[static_cast<size_t>(c) * R + r] * im[c];
    }
    rn += std::norm(cd(fr, fi) - target[r]);
    tn += std::norm(target[r]);
  }
  out.fit_rmse = tn > 0.0 ? std::sqrt(rn / tn) * 100.0 : 0.0;
  return out;
}

// proj/src/fourier_fit.cpp:107-129
std::vector<cd> reconstruct(const Coeffs& c, const std::vector<double>& q) {
  std::vector<double> re(q.size(), 0.0), im(q.size(), 0.0);
  for (size_t i = 0; i < c.grid.cos_p.size(); ++i) {
    const double bp = c.grid.beta * c.grid.cos_p[i];
    for (size_t r = 0; r < q.size(); ++r) {
      const double b = std::cos(bp * q[r]);
      re[r] += c.cc[i].real() * b;
      im[r] += c.cc[i].imag() * b;
    }
  }
  for (size_t i = 0; i < c.grid.sin_p.size(); ++i) {
    const double bp = c.grid.beta * c.grid.sin_p[i];
    for (size_t r = 0; r < q.size(); ++r) {
      const double b = std::sin(bp * q[r]);
      re[r] += c.sc[i].real() * b;
      im[r] += c.sc[i].imag() * b;
    }
  }
  std::vector<cd> out(q.size());
  for (size_t r = 0; r < q.size(); ++r) out[r] = cd(re[r], im[r]);
  return out;
}

// proj/src/fourier_fit.cpp:131-161
Bundle fit_gaussian_bundle(const GaussP& params, int P, double beta) {
  if (P < 1) throw std::invalid_argument("fit_gaussian_bundle: P must be >= 1");
  std::vector<int> co(P + 1), so(P);
  for (int p = 0; p <= P; ++p) co[p] = p;
  for (int p = 1; p <= P; ++p) so[p - 1] = p;
  const Grid cg(params.K, beta, co, {});
  const Grid sg(params.K, beta, {}, so);
  const std::vector<double> q = nodes_of(params.K);
  std::vector<cd> g(q.size()), gd(q.size()), gdd(q.size());
  for (size_t i = 0; i < q.size(); ++i) {
    g[i] = gauss(params, q[i]);
    gd[i] = gauss_d(params, q[i]);
    gdd[i] = gauss_dd(params, q[i]);
  }
  const Coeffs fa = fit_mmse(g, cg, kGaussCos);
  const Coeffs fb = fit_mmse(gd, sg, kGaussDerivSin);
  const Coeffs fd = fit_mmse(gdd, cg, kGaussDeriv2Cos);
  Bundle b;
  b.params = params;
  b.beta = beta;
  b.P = P;
  for (const cd& v : fa.cc) b.a.push_back(v.real());
  for (const cd& v : fb.sc) b.b.push_back(v.real());
  for (const cd& v : fd.cc) b.d.push_back(v.real());
  b.rmse_g = fa.fit_rmse;
  b.rmse_gd = fb.fit_rmse;
  b.rmse_gdd = fd.fit_rmse;
  return b;
}

namespace {
std::vector<double> cos_series(const std::vector<double>& c, double beta, const std::vector<double>& q) {
  std::vector<double> out(q.size(), 0.0);
  for (size_t p = 0; p < c.size(); ++p) {
    const double bp = beta * static_cast<double>(p);
    for (size_t r = 0; r < q.size(); ++r) out[r] += c[p] * std::cos(bp * q[r]);
  }
  return out;
}
std::vector<double> sin_series(const std::vector<double>& c, double beta, const std::vector<double>& q) {
  std::vector<double> out(q.size(), 0.0);
  for (size_t p = 0; p < c.size(); ++p) {
    const double bp = beta * static_cast<double>(p + 1);
    for (size_t r = 0; r < q.size(); ++r) out[r] += c[p] * std::sin(bp * q[r]);
  }
  return out;
}

// proj/src/fourier_fit.cpp:226-238 — attenuation compensation, support [-K+n0, K+n0].
Taps asft_weight(const std::vector<cd>& series, double sigma, int K, int n0) {
  const double g = 1.0 / (2.0 * sigma * sigma);
  const double alpha = 2.0 * g * n0;
  const double pref = std::exp(-alpha * alpha / (4.0 * g));
  Taps t;
  t.lo = -K + n0;
  t.taps.resize(series.size());
  for (int i = 0; i <= 2 * K; ++i) t.taps[i] = series[i] * (pref * std::exp(-alpha * (i - K)));
  return t;
}

double rmse_against(const Taps& taps, int half, const std::function<cd(double)>& truth) {
  std::vector<cd> approx(2 * static_cast<size_t>(half) + 1, cd(0, 0)), exact(approx.size());
  const int64_t hi = taps.lo + static_cast<int64_t>(taps.taps.size()) - 1;
  for (int n = -half; n <= half; ++n) {
    exact[n + half] = truth(n);
    if (n >= taps.lo && n <= hi) approx[n + half] = taps.taps[n - taps.lo];
  }
  return relative_rmse(approx, exact);
}
}  // namespace

// proj/src/fourier_fit.cpp:184-211
Taps gauss_effective_taps(const Bundle& b, GKind kind, int n0) {
  const int K = b.params.K;
  const double g = b.params.gamma();
  const double alpha = 2.0 * g * n0;
  const double pref = std::exp(-alpha * alpha / (4.0 * g));
  const std::vector<double> q = nodes_of(K);
  std::vector<double> mix;
  switch (kind) {
    case GKind::Value:
      mix = cos_series(b.a, b.beta, q);
      break;
    case GKind::Deriv1: {
      mix = sin_series(b.b, b.beta, q);
      if (n0 != 0) {
        const std::vector<double> ca = cos_series(b.a, b.beta, q);
        for (size_t i = 0; i < q.size(); ++i) mix[i] -= alpha * ca[i];
      }
      break;
    }
    case GKind::Deriv2: {
      mix = cos_series(b.d, b.beta, q);
      if (n0 != 0) {
        const std::vector<double> ca = cos_series(b.a, b.beta, q);
        const std::vector<double> sb = sin_series(b.b, b.beta, q);
        for (size_t i = 0; i < q.size(); ++i) mix[i] += alpha * alpha * ca[i] - 2.0 * alpha * sb[i];
      }
      break;
    }
  }
  Taps t;
  t.lo = -K + n0;
  t.taps.resize(q.size());
  for (size_t i = 0; i < q.size(); ++i)
    t.taps[i] = n0 != 0 ? mix[i] * (pref * std::exp(-alpha * q[i])) : mix[i];
  return t;
}

// proj/src/fourier_fit.cpp:240-247
Taps morlet_direct_effective_taps(const Coeffs& c, const MorletP& p, int n0) {
  const int K = c.grid.K;
  const std::vector<cd> s = reconstruct(c, nodes_of(K));
  if (n0 == 0) return Taps{s, -K};
  return asft_weight(s, p.sigma, K, n0);
}

// proj/src/fourier_fit.cpp:249-261
Taps morlet_multiply_effective_taps(const Coeffs& env, const MorletP& p, int n0) {
  const int K = env.grid.K;
  const std::vector<double> q = nodes_of(K);
  const std::vector<cd> e = reconstruct(env, q);
  std::vector<cd> s(q.size());
  for (size_t i = 0; i < q.size(); ++i) {
    const double ph = p.xi * (q[i] + static_cast<double>(n0)) / p.sigma;
    s[i] = e[i].real() * cd(std::cos(ph) - p.kappa(), std::sin(ph));
  }
  if (n0 == 0) return Taps{s, -K};
  return asft_weight(s, p.sigma, K, n0);
}

// proj/src/fourier_fit.cpp:278-291
double gauss_kernel_rmse(const Bundle& b, GKind kind, int n0) {
  const Taps t = gauss_effective_taps(b, kind, n0);
  const GaussP& p = b.params;
  const int half = 3 * p.K;
  switch (kind) {
    case GKind::Value: return rmse_against(t, half, [&](double n) { return cd(gauss(p, n)); });
    case GKind::Deriv1: return rmse_against(t, half, [&](double n) { return cd(gauss_d(p, n)); });
    case GKind::Deriv2: return rmse_against(t, half, [&](double n) { return cd(gauss_dd(p, n)); });
  }
  return 0.0;
}

// proj/src/fourier_fit.cpp:293-340
Coeffs fit_morlet_direct(const MorletP& p, int ps, int pd, double beta, int n0) {
  if (ps < 0 || pd < 1) throw std::invalid_argument("fit_morlet_direct: need P_S >= 0, P_D >= 1");
  const int K = p.K;
  std::vector<int> co, so;
  for (int o = ps; o < ps + pd; ++o) {
    co.push_back(o);
    if (o > 0) so.push_back(o);
  }
  const std::vector<double> q = nodes_of(K);
  const Grid grid(K, beta, co, so);
  if (n0 == 0) {
    // even real part on cosines, odd imaginary part on sines (stored as i*l_p)
    std::vector<cd> re(q.size()), im(q.size()), tgt(q.size());
    for (size_t i = 0; i < q.size(); ++i) {
      tgt[i] = morlet(p, q[i]);
      re[i] = tgt[i].real();
      im[i] = tgt[i].imag();
    }
    Coeffs out;
    out.kind = kMorletDirect;
    out.grid = grid;
    out.sigma = p.sigma;
    out.xi = p.xi;
    out.n0 = n0;
    out.cc = fit_mmse(re, Grid(K, beta, co, {}), kMorletDirect).cc;
    if (!so.empty()) {
      const Coeffs fs = fit_mmse(im, Grid(K, beta, {}, so), kMorletDirect);
      for (const cd& v : fs.sc) out.sc.emplace_back(0.0, v.real());
    }
    out.fit_rmse = relative_rmse(reconstruct(out, q), tgt);
    return out;
  }
  // ASFT: carrier-advanced target on the full cos+sin basis (:270-276, :332-339)
  const double scale = p.cxi() / (std::pow(M_PI, 0.25) * std::sqrt(p.sigma));
  std::vector<cd> tgt(q.size());
  for (size_t i = 0; i < q.size(); ++i) {
    const double env = scale * std::exp(-p.gamma() * (q[i] * q[i]));
    const double ph = p.xi * (q[i] + static_cast<double>(n0)) / p.sigma;
    tgt[i] = env * cd(std::cos(ph) - p.kappa(), std::sin(ph));
  }
  Coeffs out = fit_mmse(tgt, grid, kMorletDirect);
  out.sigma = p.sigma;
  out.xi = p.xi;
  out.n0 = n0;
  return out;
}

// proj/src/fourier_fit.cpp:342-355
Coeffs fit_morlet_envelope(const MorletP& p, int P, double beta) {
  if (P < 1) throw std::invalid_argument("fit_morlet_envelope: P must be >= 1");
  std::vector<int> co(P + 1);
  for (int o = 0; o <= P; ++o) co[o] = o;
  const Grid grid(p.K, beta, co, {});
  const std::vector<double> q = nodes_of(p.K);
  const double scale = p.cxi() / (std::pow(M_PI, 0.25) * std::sqrt(p.sigma));
  std::vector<cd> env(q.size());
  for (size_t i = 0; i < q.size(); ++i) env[i] = scale * std::exp(-p.gamma() * (q[i] * q[i]));
  Coeffs out = fit_mmse(env, grid, kMorletMultiply);
  out.sigma = p.sigma;
  out.xi = p.xi;
  return out;
}

// proj/src/fourier_fit.cpp:357-377
double morlet_direct_kernel_rmse(const MorletP& p, int ps, int pd, int n0, Coeffs* out) {
  const Coeffs c = fit_morlet_direct(p, ps, pd, M_PI / p.K, n0);
  const Taps t = morlet_direct_effective_taps(c, p, n0);
  const double r = rmse_against(t, 5 * p.K, [&](double n) { return morlet(p, n); });
  if (out) *out = c;
  return r;
}

double morlet_multiply_kernel_rmse(const MorletP& p, int pm, int n0, Coeffs* out) {
  const Coeffs e = fit_morlet_envelope(p, pm, M_PI / p.K);
  const Taps t = morlet_multiply_effective_taps(e, p, n0);
  const double r = rmse_against(t, 5 * p.K, [&](double n) { return morlet(p, n); });
  if (out) *out = e;
  return r;
}

// proj/src/fourier_fit.cpp:379-393 — exhaustive scan, ties toward smaller P_S.
int select_optimal_ps(const MorletP& p, int pd, int n0) {
  if (pd < 1) throw std::invalid_argument("select_optimal_ps: P_D must be >= 1");
  const int hi = static_cast<int>(std::ceil(p.K * p.xi / (M_PI * p.sigma))) + pd;
  // The true kernel on [-5K, 5K] is the same for every candidate: evaluate it once.
  const int half = 5 * p.K;
  std::vector<cd> truth(2 * static_cast<size_t>(half) + 1);
  for (int n = -half; n <= half; ++n) truth[n + half] = morlet(p, n);
  int best_ps = 0;
  double best = -1.0;
  for (int ps = 0; ps <= hi; ++ps) {
    const Coeffs c = fit_morlet_direct(p, ps, pd, M_PI / p.K, n0);
    const Taps t = morlet_direct_effective_taps(c, p, n0);
    std::vector<cd> approx(truth.size(), cd(0, 0));
    const int64_t thi = t.lo + static_cast<int64_t>(t.taps.size()) - 1;
    for (int n = -half; n <= half; ++n)
      if (n >= t.lo && n <= thi) approx[n + half] = t.taps[n - t.lo];
    const double r = relative_rmse(approx, truth);
    if (best < 0.0 || r < best - 1e-12) {
      best = r;
      best_ps = ps;
    }
  }
  return best_ps;
}

// proj/src/fourier_fit.cpp:395-438 — 33-point prescan + golden section to 1e-4 relative.
template <typename F>
BetaTune tune_beta(F&& f, int K) {
  const double base = M_PI / K, lo = 0.5 * base, hi = 1.5 * base;
  constexpr int kScan = 33;
  auto at = [&](int i) { return lo + (hi - lo) * i / (kScan - 1); };
  int bi = 0;
  double bv = 0.0;
  for (int i = 0; i < kScan; ++i) {
    const double v = f(at(i));
    if (i == 0 || v < bv) {
      bv = v;
      bi = i;
    }
  }
  double a = at(std::max(0, bi - 1)), b = at(std::min(kScan - 1, bi + 1));
  const double ip = (std::sqrt(5.0) - 1.0) / 2.0;
  double c = b - ip * (b - a), d = a + ip * (b - a);
  double fc = f(c), fd = f(d);
  while (b - a > 1e-4 * b) {
    if (fc < fd) {
      b = d;
      d = c;
      fd = fc;
      c = b - ip * (b - a);
      fc = f(c);
    } else {
      a = c;
      c = d;
      fc = fd;
      d = a + ip * (b - a);
      fd = f(d);
    }
  }
  BetaTune r;
  r.beta = 0.5 * (a + b);
  r.rmse = f(r.beta);
  return r;
}

BetaTune tune_beta_callback(double (*f)(double, void*), void* user, int K) {
  return tune_beta([&](double beta) { return f(beta, user); }, K);
}

BetaTune tune_beta_gauss(const GaussP& p, int P, int n0) {
  return tune_beta(
      [&](double beta) { return gauss_kernel_rmse(fit_gaussian_bundle(p, P, beta), GKind::Value, n0); },
      p.K);
}

// ------------------------------------------------------------------ spec factories
// proj/src/transforms.cpp:16-49, :53-120, :122-242
namespace {
void check_shift(double sigma, int n0) {
  if (n0 < 0) throw std::invalid_argument("TransformSpec: n0 must be >= 0");
  if (n0 > sigma / 4.0) throw std::invalid_argument("TransformSpec: n0 must stay <= sigma/4");
}
double shift_alpha(double sigma, int n0) { return 2.0 * (1.0 / (2.0 * sigma * sigma)) * n0; }
int oracle_K(double sigma) { return static_cast<int>(std::floor(3.0 * sigma + 1e-9)); }
}  // namespace

Abbrev parse_abbreviation(const std::string& s) {
  if (s == "GCT3") return {TKind::TruncGauss, 0, 0};
  if (s == "MCT3") return {TKind::TruncMorlet, 0, 0};
  auto bad = [&]() -> Abbrev { throw std::invalid_argument("unrecognized filter abbreviation: " + s); };
  if (s.size() < 3) return bad();
  const char fam = s[0], meth = s[1];
  if ((fam != 'G' && fam != 'M') || (meth != 'D' && meth != 'M')) return bad();
  if (fam == 'G' && meth == 'M') return bad();
  size_t pos = 2;
  int n0 = 0;
  if (s[pos] == 'S') {
    ++pos;
    size_t dg = 0;
    while (pos + dg < s.size() && std::isdigit(static_cast<unsigned char>(s[pos + dg]))) ++dg;
    if (dg == 0) return bad();
    n0 = std::stoi(s.substr(pos, dg));
    pos += dg;
    if (n0 < 1) return bad();
  }
  if (pos >= s.size() || s[pos] != 'P') return bad();
  ++pos;
  if (pos >= s.size()) return bad();
  for (size_t i = pos; i < s.size(); ++i)
    if (!std::isdigit(static_cast<unsigned char>(s[i]))) return bad();
  const int order = std::stoi(s.substr(pos));
  if (order < 1) return bad();
  Abbrev a;
  a.n0 = n0;
  a.order = order;
  a.kind = fam == 'G' ? TKind::Gauss : (meth == 'D' ? TKind::MorletDirect : TKind::MorletMultiply);
  return a;
}

std::string encode_abbreviation(TKind k, int n0, int order) {
  switch (k) {
    case TKind::TruncGauss: return "GCT3";
    case TKind::TruncMorlet: return "MCT3";
    case TKind::Gauss:
    case TKind::GaussD:
    case TKind::GaussDD: {
      std::string t = "GD";
      if (n0 > 0) t += "S" + std::to_string(n0);
      t += "P" + std::to_string(order);
      if (k == TKind::GaussD) t += ":d1";
      if (k == TKind::GaussDD) t += ":d2";
      return t;
    }
    case TKind::MorletDirect:
    case TKind::MorletMultiply: {
      std::string t = k == TKind::MorletDirect ? "MD" : "MM";
      if (n0 > 0) t += "S" + std::to_string(n0);
      t += "P" + std::to_string(order);
      return t;
    }
  }
  return "?";
}

Spec make_gauss_spec(double sigma, GKind kind, int P, int n0, const Options& o) {
  check_shift(sigma, n0);
  const int K = o.has_K ? o.K : GaussP::default_K(sigma);
  const GaussP params(sigma, K);
  Spec s;
  s.kind = kind == GKind::Value ? TKind::Gauss : (kind == GKind::Deriv1 ? TKind::GaussD : TKind::GaussDD);
  s.has_gauss = true;
  s.gparams = params;
  s.max_order = P;
  s.n0 = n0;
  s.alpha = shift_alpha(sigma, n0);
  s.strategy = o.strategy;
  s.precision = o.precision;
  if (o.has_beta)
    s.beta = o.beta;
  else if (o.tune)
    s.beta = tune_beta_gauss(params, P, n0).beta;
  else
    s.beta = M_PI / K;
  s.bundle = fit_gaussian_bundle(params, P, s.beta);
  s.has_bundle = true;
  s.kernel_rmse = gauss_kernel_rmse(s.bundle, kind, n0);
  s.abbrev = encode_abbreviation(s.kind, n0, P);
  return s;
}

Spec make_morlet_direct_spec(double sigma, double xi, int pd, int n0, const Options& o) {
  check_shift(sigma, n0);
  const int K = o.has_K ? o.K : GaussP::default_K(sigma);
  const MorletP params(sigma, xi, K);
  Spec s;
  s.kind = TKind::MorletDirect;
  s.has_morlet = true;
  s.mparams = params;
  s.pd = pd;
  s.ps = o.has_ps ? o.ps : -1;
  if (s.ps < 0) s.ps = select_optimal_ps(params, pd, n0);
  s.n0 = n0;
  s.alpha = shift_alpha(sigma, n0);
  s.strategy = o.strategy;
  s.precision = o.precision;
  s.beta = o.has_beta ? o.beta : M_PI / K;
  s.morlet = fit_morlet_direct(params, s.ps, pd, s.beta, n0);
  s.has_mcoef = true;
  s.kernel_rmse = rmse_against(morlet_direct_effective_taps(s.morlet, params, n0), 5 * K,
                               [&](double n) { return morlet(params, n); });
  s.abbrev = encode_abbreviation(s.kind, n0, pd);
  return s;
}

Spec make_morlet_multiply_spec(double sigma, double xi, int pm, int n0, const Options& o) {
  check_shift(sigma, n0);
  const int K = o.has_K ? o.K : GaussP::default_K(sigma);
  const MorletP params(sigma, xi, K);
  Spec s;
  s.kind = TKind::MorletMultiply;
  s.has_morlet = true;
  s.mparams = params;
  s.max_order = pm;
  s.n0 = n0;
  s.alpha = shift_alpha(sigma, n0);
  s.strategy = o.strategy;
  s.precision = o.precision;
  s.beta = o.has_beta ? o.beta : M_PI / K;
  s.envelope = fit_morlet_envelope(params, pm, s.beta);
  s.has_env = true;
  s.kernel_rmse = rmse_against(morlet_multiply_effective_taps(s.envelope, params, n0), 5 * K,
                               [&](double n) { return morlet(params, n); });
  s.abbrev = encode_abbreviation(s.kind, n0, pm);
  return s;
}

Spec make_transform_spec(const std::string& a, double sigma, double xi, const Options& o) {
  const Abbrev info = parse_abbreviation(a);
  switch (info.kind) {
    case TKind::Gauss: return make_gauss_spec(sigma, GKind::Value, info.order, info.n0, o);
    case TKind::MorletDirect: return make_morlet_direct_spec(sigma, xi, info.order, info.n0, o);
    case TKind::MorletMultiply: return make_morlet_multiply_spec(sigma, xi, info.order, info.n0, o);
    case TKind::TruncGauss: {
      Spec s;
      s.kind = TKind::TruncGauss;
      s.has_gauss = true;
      s.gparams = GaussP(sigma, oracle_K(sigma));
      s.abbrev = "GCT3";
      return s;
    }
    case TKind::TruncMorlet: {
      Spec s;
      s.kind = TKind::TruncMorlet;
      s.has_morlet = true;
      s.mparams = MorletP(sigma, xi, oracle_K(sigma));
      s.abbrev = "MCT3";
      return s;
    }
    default: throw std::invalid_argument("unsupported abbreviation: " + a);
  }
}

// proj/src/transforms.cpp:461-477
Taps effective_kernel(const Spec& s) {
  switch (s.kind) {
    case TKind::Gauss: return gauss_effective_taps(s.bundle, GKind::Value, s.n0);
    case TKind::GaussD: return gauss_effective_taps(s.bundle, GKind::Deriv1, s.n0);
    case TKind::GaussDD: return gauss_effective_taps(s.bundle, GKind::Deriv2, s.n0);
    case TKind::MorletDirect: return morlet_direct_effective_taps(s.morlet, s.mparams, s.n0);
    case TKind::MorletMultiply: return morlet_multiply_effective_taps(s.envelope, s.mparams, s.n0);
    case TKind::TruncGauss: return sample_gauss(s.gparams);
    case TKind::TruncMorlet: return sample_morlet(s.mparams);
  }
  throw std::invalid_argument("effective_kernel: unknown kind");
}

// ------------------------------------------------------------------ coefficient files
// "sft-coefficients v1" text format (proj/src/coeff_io.cpp:11-101): one "set" header
// line with key=value fields, "coeff cos|sin p re im" lines, "end".
namespace {
const char* kind_name(int k) {
  switch (k) {
    case kGaussCos: return "GaussCos";
    case kGaussDerivSin: return "GaussDerivSin";
    case kGaussDeriv2Cos: return "GaussDeriv2Cos";
    case kMorletDirect: return "MorletDirect";
    case kMorletMultiply: return "MorletMultiply";
  }
  return "?";
}
int kind_from_name(const std::string& n) {
  for (int k = kGaussCos; k <= kMorletMultiply; ++k)
    if (n == kind_name(k)) return k;
  throw std::invalid_argument("unknown coefficient kind: " + n);
}
std::string g17(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}
}  // namespace

std::string write_coefficient_sets(const std::vector<Coeffs>& sets) {
  std::string o = "sft-coefficients v1\n";
  for (const Coeffs& c : sets) {
    o += "set kind=" + std::string(kind_name(c.kind)) + " K=" + std::to_string(c.grid.K) + " beta=" + g17(c.grid.beta) +
         " sigma=" + g17(c.sigma) + " xi=" + g17(c.xi) + " n0=" + std::to_string(c.n0) + " fit_rmse=" + g17(c.fit_rmse) +
         "\n";
    for (size_t i = 0; i < c.grid.cos_p.size(); ++i)
      o += "coeff cos " + std::to_string(c.grid.cos_p[i]) + " " + g17(c.cc[i].real()) + " " + g17(c.cc[i].imag()) + "\n";
    for (size_t i = 0; i < c.grid.sin_p.size(); ++i)
      o += "coeff sin " + std::to_string(c.grid.sin_p[i]) + " " + g17(c.sc[i].real()) + " " + g17(c.sc[i].imag()) + "\n";
    o += "end\n";
  }
  return o;
}

std::vector<Coeffs> read_coefficient_sets(const std::string& text) {
  std::istringstream is(text);
  std::string line;
  if (!std::getline(is, line) || line != "sft-coefficients v1")
    throw std::invalid_argument("coefficient file: bad or missing version header");
  std::vector<Coeffs> sets;
  while (std::getline(is, line)) {
    if (line.empty()) continue;
    std::istringstream head(line);
    std::string tok;
    head >> tok;
    if (tok != "set") throw std::invalid_argument("coefficient file: expected 'set', got: " + line);
    std::map<std::string, std::string> f;
    while (head >> tok) {
      const auto eq = tok.find('=');
      if (eq == std::string::npos) throw std::invalid_argument("coefficient file: malformed field: " + tok);
      f[tok.substr(0, eq)] = tok.substr(eq + 1);
    }
    auto need = [&](const char* k) -> const std::string& {
      auto it = f.find(k);
      if (it == f.end()) throw std::invalid_argument(std::string("coefficient file: missing field ") + k);
      return it->second;
    };
    Coeffs c;
    c.kind = kind_from_name(need("kind"));
    const int K = std::stoi(need("K"));
    const double beta = std::stod(need("beta"));
    std::vector<int> co, so;
    while (std::getline(is, line) && line != "end") {
      std::istringstream row(line);
      std::string tag, basis;
      int p = 0;
      double re = 0.0, im = 0.0;
      row >> tag >> basis >> p >> re >> im;
      if (tag != "coeff" || row.fail())
        throw std::invalid_argument("coefficient file: malformed coefficient line: " + line);
      if (basis == "cos") {
        co.push_back(p);
        c.cc.emplace_back(re, im);
      } else if (basis == "sin") {
        so.push_back(p);
        c.sc.emplace_back(re, im);
      } else {
        throw std::invalid_argument("coefficient file: unknown basis: " + basis);
      }
    }
    c.grid = Grid(K, beta, co, so);
    c.fit_rmse = std::stod(need("fit_rmse"));
    c.sigma = std::stod(need("sigma"));
    c.xi = std::stod(need("xi"));
    c.n0 = std::stoi(need("n0"));
    sets.push_back(std::move(c));
  }
  return sets;
}

// A MorletDirect spec from a stored coefficient set (the CLI's --coeffs path,
// proj/src/cli.cpp:224-280): parameters from the set's provenance, kernel RMSE
// recomputed on [-5K, 5K] when requested.
Spec morlet_direct_spec_from_coeffs(const Coeffs& c, int precision, int strategy, bool recompute_rmse) {
  if (c.kind != kMorletDirect) throw std::invalid_argument("coefficient set is not MorletDirect");
  if (c.grid.cos_p.empty()) throw std::invalid_argument("coefficient set has no cosine orders");
  check_shift(c.sigma, c.n0);
  Spec s;
  s.kind = TKind::MorletDirect;
  s.has_morlet = true;
  s.mparams = MorletP(c.sigma, c.xi, c.grid.K);
  s.ps = c.grid.cos_p.front();
  s.pd = static_cast<int>(c.grid.cos_p.size());
  s.n0 = c.n0;
  s.alpha = shift_alpha(c.sigma, c.n0);
  s.strategy = strategy;
  s.precision = precision;
  s.beta = c.grid.beta;
  s.morlet = c;
  s.has_mcoef = true;
  if (recompute_rmse)
    s.kernel_rmse = rmse_against(morlet_direct_effective_taps(c, s.mparams, c.n0), 5 * c.grid.K,
                                 [&](double n) { return morlet(s.mparams, n); });
  s.abbrev = encode_abbreviation(s.kind, c.n0, s.pd);
  return s;
}

}  // namespace sftb
