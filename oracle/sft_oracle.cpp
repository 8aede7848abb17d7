// ============================================================================
// TEST INFRASTRUCTURE ONLY — NOT PART OF THE PRODUCT.
//
// CPU restatement of the reference SFT/ASFT hot path (arXiv 2110.11866
// reference library, /root/reference/proj). Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load this library,
// and only as the checker or the timed CPU baseline. The product path
// (paper_2110_11866_b200/, libsftgpu.so) never links or calls it.
//
// The reference itself cannot be built here (it needs Eigen3, absent; see
// DESIGN.md "Oracle"), so this file restates, function by function, the
// algorithms of:
//   proj/include/sft/signal.hpp:35-45, proj/src/signal.cpp:9-51   (signal, generators)
//   proj/src/engine.cpp:12-337                                     (3 strategies + sliding-sum route)
//   proj/include/sft/sliding_sum.hpp:89-234, proj/src/sliding_sum.cpp (flat + blocked8 + cost model)
//   proj/src/kernels.cpp:35-51, proj/include/sft/kernels.hpp:54-73 (truncated convolution, kernels)
//   proj/src/transforms.cpp:279-428                                (coefficient combine)
//   proj/src/fourier_fit.cpp:184-261 (effective taps, via series evaluation)
// keeping the reference's fp64 phase evaluation (std::cos/std::sin of omega*j),
// loop orders and Scalar casts so results agree to rounding (~1e-15 relative).
// Parity pins: tests/test_oracle_pins.py checks this file against every
// known-answer assertion of proj/tests/test_engine.cpp, test_transforms.cpp,
// test_sliding_sum.cpp, test_kernels.cpp, test_signal.cpp and the numbers
// printed in proj/test_output.txt.
// ============================================================================

#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

using i64 = std::int64_t;
using cd = std::complex<double>;

enum Boundary { kZero = 0, kClamp = 1 };
enum Strategy { kKernelIntegral = 0, kRecursive1 = 1, kRecursive2 = 2 };
enum Precision { kSingle = 0, kDouble = 1 };

thread_local std::string g_err;

struct Sig {
  const double* x;
  i64 n;
  int boundary;
  // proj/include/sft/signal.hpp:35-45
  double at(i64 j) const {
    if (j >= 0 && j < n) return x[j];
    if (boundary == kZero) return 0.0;
    return j < 0 ? x[0] : x[n - 1];
  }
};

struct Cfg {
  int K;
  double beta;
  int integer_order;
  int p;
  double omega;
  double alpha;
  int n0;
  int strategy;
  int precision;
  int window_2k1;
  // proj/include/sft/engine.hpp:38
  double angular() const { return integer_order ? beta * p : omega; }
  // proj/include/sft/engine.hpp:51-59
  void validate() const {
    if (K < 1) throw std::invalid_argument("SftConfig: K must be >= 1");
    if (!(beta > 0.0) && integer_order) throw std::invalid_argument("SftConfig: beta must be > 0");
    if (alpha < 0.0) throw std::invalid_argument("SftConfig: alpha must be >= 0");
    if (integer_order && p < 0) throw std::invalid_argument("OrderSpec: p must be >= 0");
    if (!integer_order && strategy != kKernelIntegral)
      throw std::invalid_argument(
          "SftConfig: real-frequency components require the kernel-integral strategy");
  }
};

// proj/include/sft/parallel.hpp:13-32 — contiguous chunks, one std::thread each.
template <typename Fn>
void parallel_chunks(i64 lo, i64 hi, int workers, Fn&& body) {
  const i64 count = hi - lo;
  if (count <= 0) return;
  if (workers <= 1 || count == 1) {
    body(lo, hi);
    return;
  }
  const int used = static_cast<int>(std::min<i64>(workers, count));
  const i64 chunk = (count + used - 1) / used;
  std::vector<std::thread> pool;
  for (int w = 0; w < used; ++w) {
    const i64 a = lo + w * chunk;
    const i64 b = std::min(hi, a + chunk);
    if (a >= b) break;
    pool.emplace_back([&body, a, b] { body(a, b); });
  }
  for (auto& t : pool) t.join();
}

// Ring of complex states indexed by absolute position (proj/src/engine.cpp:12-31).
template <typename T>
struct PosRing {
  i64 first;
  std::vector<T> buf;
  PosRing(i64 first_pos, i64 cap) : first(first_pos), buf(static_cast<size_t>(cap), T{}) {}
  size_t slot(i64 pos) const { return static_cast<size_t>((pos - first) % static_cast<i64>(buf.size())); }
  void put(i64 pos, T v) { buf[slot(pos)] = v; }
  T get(i64 pos) const { return pos < first ? T{} : buf[slot(pos)]; }
};

// Output convention (proj/src/engine.cpp:33-45): c = Re, s = -Im, stored as double.
template <typename S>
inline void emit(double* c, double* s, i64 idx, std::complex<S> v) {
  c[idx] = static_cast<double>(v.real());
  s[idx] = -static_cast<double>(v.imag());
}

// ---------------------------------------------------------------- Recursive1/2
// proj/src/engine.cpp:53-120
template <typename S>
void run_recursive(const Sig& sig, const Cfg& cfg, i64 lo, i64 hi, double* c, double* s,
                   double* max_state) {
  using C = std::complex<S>;
  const int k = cfg.K;
  const double w = cfg.angular();
  const double dec = std::exp(-cfg.alpha);
  const C z(static_cast<S>(dec * std::cos(w)), static_cast<S>(-dec * std::sin(w)));
  const S two_c = static_cast<S>(2.0 * dec * std::cos(w));
  const S dec2 = static_cast<S>(dec * dec);
  const C zc(z.real(), -z.imag());
  auto zpow = [&](double cnt) {
    const double m = std::exp(-cfg.alpha * cnt);
    return C(static_cast<S>(m * std::cos(w * cnt)), static_cast<S>(-m * std::sin(w * cnt)));
  };
  const C z2k = zpow(2.0 * k);
  const C z2k1 = zpow(2.0 * k + 1.0);
  const double um = std::exp(cfg.alpha * k);
  const C unwind(static_cast<S>(um * std::cos(w * k)), static_cast<S>(um * std::sin(w * k)));

  const i64 start = lo - k - (2 * static_cast<i64>(k) + 1);
  PosRing<C> ring(start, 2 * static_cast<i64>(k) + 2);
  S xprev = S(0);
  C v1{}, v2{};
  double peak = 0.0;
  for (i64 m = start; m <= hi + k; ++m) {
    const S xm = static_cast<S>(sig.at(m));
    C v;
    if (cfg.strategy == kRecursive1) {
      v = C(z.real() * v1.real() - z.imag() * v1.imag() + xm,
            z.real() * v1.imag() + z.imag() * v1.real());
    } else {
      v = C(two_c * v1.real() - dec2 * v2.real() + xm - zc.real() * xprev,
            two_c * v1.imag() - dec2 * v2.imag() - zc.imag() * xprev);
    }
    v2 = v1;
    v1 = v;
    xprev = xm;
    ring.put(m, v);
    if (max_state) peak = std::max(peak, static_cast<double>(std::abs(v)));
    if (m >= lo + k) {
      const i64 n = m - k;
      C win;
      if (cfg.window_2k1)
        win = v - z2k1 * ring.get(m - 2 * k - 1);
      else
        win = v - z2k * ring.get(m - 2 * k) + z2k * static_cast<S>(sig.at(n - k));
      emit(c, s, n - lo, unwind * win);
    }
  }
  if (max_state) *max_state = peak;
}

// proj/src/engine.cpp:122-134 — fp64 phase, cast to Scalar.
template <typename S>
inline std::complex<S> modulated(const Sig& sig, double w, i64 j) {
  const double xj = sig.at(j);
  return {static_cast<S>(xj * std::cos(w * static_cast<double>(j))),
          static_cast<S>(xj * std::sin(w * static_cast<double>(j)))};
}

template <typename S>
inline std::complex<S> demodulate(double w, i64 n, std::complex<S> v) {
  const S cn = static_cast<S>(std::cos(w * static_cast<double>(n)));
  const S sn = static_cast<S>(std::sin(w * static_cast<double>(n)));
  return {v.real() * cn + v.imag() * sn, v.imag() * cn - v.real() * sn};
}

// ---------------------------------------------------------------- kernel integral
// proj/src/engine.cpp:136-181
template <typename S>
void run_kernel_integral(const Sig& sig, const Cfg& cfg, i64 lo, i64 hi, double* c, double* s,
                         double* max_state) {
  using C = std::complex<S>;
  const int k = cfg.K;
  const double w = cfg.angular();
  double peak = 0.0;
  if (cfg.alpha == 0.0) {
    // prefix u[m] from lo-K-1; window = u[m] - u[m-2K-1], output n = m-K
    const i64 start = lo - k - 1;
    PosRing<C> ring(start, 2 * static_cast<i64>(k) + 2);
    C u{};
    for (i64 m = start; m <= hi + k; ++m) {
      u += modulated<S>(sig, w, m);
      ring.put(m, u);
      if (max_state) peak = std::max(peak, static_cast<double>(std::abs(u)));
      if (m >= lo + k) {
        const i64 n = m - k;
        const C win = u - ring.get(m - 2 * k - 1);
        emit(c, s, n - lo, demodulate<S>(w, n, win));
      }
    }
  } else {
    // attenuated in-window recurrence, exact explicit initial window
    const S dec = static_cast<S>(std::exp(-cfg.alpha));
    const S leave = static_cast<S>(std::exp(-(2.0 * k + 1.0) * cfg.alpha));
    const S gain = static_cast<S>(std::exp(cfg.alpha * k));
    const i64 first = lo + k;
    C win{};
    for (int lag = 2 * k; lag >= 0; --lag) win = dec * win + modulated<S>(sig, w, first - lag);
    for (i64 m = first; m <= hi + k; ++m) {
      if (m > first)
        win = dec * win + modulated<S>(sig, w, m) - leave * modulated<S>(sig, w, m - 2 * k - 1);
      if (max_state) peak = std::max(peak, static_cast<double>(std::abs(win)));
      const i64 n = m - k;
      emit(c, s, n - lo, gain * demodulate<S>(w, n, win));
    }
  }
  if (max_state) *max_state = peak;
}

// ---------------------------------------------------------------- sliding sums
inline int bit_of(std::uint64_t m, unsigned r) { return static_cast<int>((m >> r) & 1ULL); }

struct RoundRec {
  int round, stage, r, bit;
  i64 active, adds;
};

// proj/include/sft/sliding_sum.hpp:32-60
struct Plan {
  i64 n = 0, L = 0;
  int rounds = 0;
  i64 padded = 0;
  static int stages_for(i64 L) {
    int st = 0;
    for (i64 rest = L; rest > 0; rest /= 8) ++st;
    return st;
  }
  static Plan make(i64 n, i64 L) {
    if (n < 1) throw std::invalid_argument("SlidingSumPlan: N must be >= 1");
    if (L < 1 || L > n) throw std::invalid_argument("SlidingSumPlan: need 1 <= L <= N");
    Plan p;
    p.n = n;
    p.L = L;
    p.rounds = 1;
    while ((i64{1} << p.rounds) <= L) ++p.rounds;
    i64 floor8 = 1;
    for (int t = 0; t < stages_for(L); ++t) floor8 *= 8;
    p.padded = 1;
    while (p.padded < n || p.padded < floor8) p.padded *= 8;
    return p;
  }
};

// Algorithm 1 (proj/include/sft/sliding_sum.hpp:89-121): log-depth doubling over double buffers.
template <typename T>
std::vector<T> sliding_flat(const T* f, i64 n, i64 L, int workers, std::vector<RoundRec>* trace) {
  const Plan plan = Plan::make(n, L);
  std::vector<T> g(f, f + n), h(static_cast<size_t>(n), T{}), g2(static_cast<size_t>(n)),
      h2(static_cast<size_t>(n));
  for (int r = 0; r < plan.rounds; ++r) {
    const i64 sh = i64{1} << r;
    const int fold = bit_of(static_cast<std::uint64_t>(L), static_cast<unsigned>(r));
    parallel_chunks(0, n, workers, [&](i64 a, i64 b) {
      for (i64 i = a; i < b; ++i) {
        const T gi = i + sh < n ? g[i + sh] : T{};
        g2[i] = g[i] + gi;
        if (fold) {
          const T hi = i + sh < n ? h[i + sh] : T{};
          h2[i] = g[i] + hi;
        } else {
          h2[i] = h[i];
        }
      }
    });
    g.swap(g2);
    h.swap(h2);
    if (trace) trace->push_back({r, 0, r, fold, n, n * (1 + fold)});
  }
  h.resize(static_cast<size_t>(n - L + 1));
  return h;
}

// proj/include/sft/sliding_sum.hpp:127-139
inline void layout8(i64 index, int stages, i64* row, i64* col) {
  i64 div = 1;
  for (int t = 0; t < stages; ++t) div *= 8;
  i64 rem = index % div;
  i64 c = 0;
  for (int t = 0; t < stages; ++t) {
    c = c * 8 + rem % 8;
    rem /= 8;
  }
  *row = index / div;
  *col = c;
}

// Algorithms 2-3 (proj/include/sft/sliding_sum.hpp:144-234): (16,8) tiles, three rounds
// per base-8 digit of L, transposed write-back.
template <typename T>
std::vector<T> sliding_blocked8(const T* f, i64 n, i64 L, int workers,
                                std::vector<RoundRec>* trace) {
  const Plan plan = Plan::make(n, L);
  const i64 P = plan.padded;
  std::vector<T> ga(P, T{}), ha(P, T{}), gb(P, T{}), hb(P, T{});
  for (i64 i = 0; i < n; ++i) ga[i] = f[i];
  i64 rest = L;
  int stage = 0, gr = 0;
  i64 rows = P, cols = 1;
  while (rest > 0) {
    const i64 out_rows = rows / 8;
    const i64 bx_count = (rows + 63) / 64;
    const i64 blocks = bx_count * cols;
    parallel_chunks(0, blocks, workers, [&](i64 a, i64 b) {
      T S[16][8], Tt[16][8], Sn[16][8], Tn[16][8];
      for (i64 id = a; id < b; ++id) {
        const i64 bx = id / cols, col = id % cols;
        for (int xt = 0; xt < 16; ++xt)
          for (int yt = 0; yt < 8; ++yt) {
            const i64 row = xt + 8 * yt + 64 * bx;
            const bool in = row < rows;
            S[xt][yt] = in ? ga[row * cols + col] : T{};
            Tt[xt][yt] = in ? ha[row * cols + col] : T{};
          }
        for (int r = 0; r < 3; ++r) {
          const int fold = bit_of(static_cast<std::uint64_t>(rest), static_cast<unsigned>(r));
          const int reach = 1 << r;
          for (int xt = 0; xt < 16; ++xt)
            for (int yt = 0; yt < 8; ++yt) {
              if (xt < 16 - reach) {
                Tn[xt][yt] = fold ? T(S[xt][yt] + Tt[xt + reach][yt]) : Tt[xt][yt];
                Sn[xt][yt] = S[xt][yt] + S[xt + reach][yt];
              } else {
                Tn[xt][yt] = Tt[xt][yt];
                Sn[xt][yt] = S[xt][yt];
              }
            }
          for (int xt = 0; xt < 16; ++xt)
            for (int yt = 0; yt < 8; ++yt) {
              S[xt][yt] = Sn[xt][yt];
              Tt[xt][yt] = Tn[xt][yt];
            }
        }
        for (int xt = 0; xt < 8; ++xt)
          for (int yt = 0; yt < 8; ++yt) {
            const i64 orow = yt + 8 * bx;
            if (orow >= out_rows) continue;
            const i64 ocol = xt + 8 * col;
            gb[orow * (cols * 8) + ocol] = S[xt][yt];
            hb[orow * (cols * 8) + ocol] = Tt[xt][yt];
          }
      }
    });
    if (trace) {
      for (int r = 0; r < 3; ++r) {
        const int fold = bit_of(static_cast<std::uint64_t>(rest), static_cast<unsigned>(r));
        const i64 active = static_cast<i64>(16 - (1 << r)) * 8 * blocks;
        trace->push_back({gr + r, stage, r, fold, active, active * (1 + fold)});
      }
    }
    gr += 3;
    ga.swap(gb);
    ha.swap(hb);
    rows = out_rows;
    cols *= 8;
    rest /= 8;
    ++stage;
  }
  std::vector<T> out(static_cast<size_t>(n - L + 1));
  for (i64 i = 0; i < static_cast<i64>(out.size()); ++i) {
    i64 row, col;
    layout8(i, stage, &row, &col);
    out[i] = ha[row * cols + col];
  }
  return out;
}

// proj/src/engine.cpp:183-219 — materialise the (midpoint-rebased) modulated sequence,
// sliding-sum it with L=2K+1, demodulate and un-rebase.
template <typename S>
void run_sliding_route(const Sig& sig, const Cfg& cfg, i64 lo, i64 hi, double* c, double* s,
                       int workers, double* max_state) {
  using C = std::complex<S>;
  const int k = cfg.K;
  const double w = cfg.angular();
  const i64 count = hi - lo + 1;
  const i64 len = count + 2 * static_cast<i64>(k);
  const double mid = 0.5 * static_cast<double>(lo + hi);
  if (cfg.alpha * (0.5 * static_cast<double>(count) + k) > 600.0)
    throw std::invalid_argument(
        "sft_via_sliding_sum: alpha * N / 2 too large for the attenuated phased sequence");
  std::vector<C> f(static_cast<size_t>(len));
  for (i64 i = 0; i < len; ++i) {
    const i64 j = lo - k + i;
    const double wt = cfg.alpha == 0.0 ? 1.0 : std::exp(cfg.alpha * (static_cast<double>(j) - mid));
    const double xj = sig.at(j) * wt;
    f[i] = C(static_cast<S>(xj * std::cos(w * static_cast<double>(j))),
             static_cast<S>(xj * std::sin(w * static_cast<double>(j))));
  }
  const std::vector<C> sums = sliding_flat<C>(f.data(), len, 2 * static_cast<i64>(k) + 1, workers,
                                              nullptr);
  double peak = 0.0;
  for (i64 n = lo; n <= hi; ++n) {
    const C v = sums[n - lo];
    if (max_state) peak = std::max(peak, static_cast<double>(std::abs(v)));
    const double sc = cfg.alpha == 0.0 ? 1.0 : std::exp(-cfg.alpha * (static_cast<double>(n) - mid));
    emit(c, s, n - lo, static_cast<S>(sc) * demodulate<S>(w, n, v));
  }
  if (max_state) *max_state = peak;
}

// proj/src/engine.cpp:221-251
template <typename S>
void route(const Sig& sig, const Cfg& cfg, i64 lo, i64 hi, double* c, double* s, double* ms) {
  if (cfg.strategy == kRecursive1 || cfg.strategy == kRecursive2) {
    run_recursive<S>(sig, cfg, lo, hi, c, s, ms);
  } else if (cfg.precision == kSingle && cfg.alpha == 0.0) {
    run_sliding_route<S>(sig, cfg, lo, hi, c, s, 1, ms);
  } else {
    run_kernel_integral<S>(sig, cfg, lo, hi, c, s, ms);
  }
}

void components(const Sig& sig, const Cfg& cfg, i64 lo, i64 hi, double* c, double* s,
                double* ms = nullptr) {
  cfg.validate();
  if (lo > hi) throw std::invalid_argument("components_over: empty range");
  if (cfg.precision == kSingle)
    route<float>(sig, cfg, lo, hi, c, s, ms);
  else
    route<double>(sig, cfg, lo, hi, c, s, ms);
}

// ---------------------------------------------------------------- combine (transforms.cpp)
struct Comp {
  std::vector<double> c, s;
};

Cfg base_cfg(int K, double beta, double alpha, int n0, int strategy, int precision) {
  Cfg cfg{};
  cfg.K = K;
  cfg.beta = beta;
  cfg.integer_order = 1;
  cfg.alpha = alpha;
  cfg.n0 = n0;
  cfg.strategy = strategy;
  cfg.precision = precision;
  cfg.window_2k1 = 0;
  return cfg;
}

// Accumulate only nonzero parts, sequentially over orders (transforms.cpp:355-373, :415-441).
struct Acc {
  std::vector<double> re, im;
  explicit Acc(i64 n) : re(static_cast<size_t>(n), 0.0), im(static_cast<size_t>(n), 0.0) {}
  void add(cd coef, const std::vector<double>& v) {
    if (coef.real() != 0.0)
      for (size_t i = 0; i < v.size(); ++i) re[i] += coef.real() * v[i];
    if (coef.imag() != 0.0)
      for (size_t i = 0; i < v.size(); ++i) im[i] += coef.imag() * v[i];
  }
};

}  // namespace orc

// ============================================================================ C ABI
using namespace orc;

#define ORC_TRY(...)                                    \
  try {                                                 \
    __VA_ARGS__;                                               \
    return 0;                                           \
  } catch (const std::invalid_argument& e) {            \
    g_err = e.what();                                   \
    return 2;                                           \
  } catch (const std::exception& e) {                   \
    g_err = e.what();                                   \
    return 1;                                           \
  }

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// proj/src/signal.cpp:9-51 (splitmix64; uniform in [-1,1]; chirp with 8 cycles).
int orc_make_test_signal(int kind, i64 n, std::uint64_t seed, double* out) {
  ORC_TRY({
    if (n < 1) throw std::invalid_argument("make_test_signal: N must be >= 1");
    switch (kind) {
      case 0:  // Impulse
        for (i64 i = 0; i < n; ++i) out[i] = 0.0;
        out[n / 2] = 1.0;
        break;
      case 1:  // Constant
        for (i64 i = 0; i < n; ++i) out[i] = 1.0;
        break;
      case 2: {  // Chirp
        const double inv = 1.0 / (static_cast<double>(n) * static_cast<double>(n));
        for (i64 i = 0; i < n; ++i)
          out[i] = std::sin(2.0 * M_PI * 8.0 * static_cast<double>(i * i) * inv);
        break;
      }
      case 3: {  // SeededNoise
        std::uint64_t st = seed;
        for (i64 i = 0; i < n; ++i) {
          st += 0x9e3779b97f4a7c15ULL;
          std::uint64_t z = st;
          z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
          z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
          z ^= z >> 31;
          out[i] = 2.0 * (static_cast<double>(z >> 11) * 0x1.0p-53) - 1.0;
        }
        break;
      }
      default:
        throw std::invalid_argument("make_test_signal: unknown kind");
    }
  })
}

// components_over (proj/src/engine.cpp:255-258) incl. the alpha checks of
// sft_components/asft_components when mode = 1/2 (:260-269).
int orc_components(const double* x, i64 n, int boundary, int K, double beta, int integer_order,
                   int p, double omega, double alpha, int strategy, int precision, int window_2k1,
                   i64 lo, i64 hi, int mode, double* c, double* s, double* max_state) {
  ORC_TRY({
    if (n < 1) throw std::invalid_argument("Signal: need at least one sample");
    Sig sig{x, n, boundary};
    Cfg cfg{K, beta, integer_order, p, omega, alpha, 0, strategy, precision, window_2k1};
    if (mode == 1 && cfg.alpha != 0.0)
      throw std::invalid_argument("sft_components: alpha must be 0 (use asft_components)");
    if (mode == 2 && !(cfg.alpha > 0.0))
      throw std::invalid_argument("asft_components: alpha must be > 0");
    components(sig, cfg, lo, hi, c, s, max_state);
  })
}

// sft_via_sliding_sum (proj/src/engine.cpp:323-337)
int orc_sft_via_sliding_sum(const double* x, i64 n, int boundary, int K, double beta,
                            int integer_order, int p, double omega, double alpha, int precision,
                            int workers, double* c, double* s) {
  ORC_TRY({
    Sig sig{x, n, boundary};
    Cfg cfg{K, beta, integer_order, p, omega, alpha, 0, kKernelIntegral, precision, 0};
    cfg.validate();
    if (precision == kSingle)
      run_sliding_route<float>(sig, cfg, 0, n - 1, c, s, workers, nullptr);
    else
      run_sliding_route<double>(sig, cfg, 0, n - 1, c, s, workers, nullptr);
  })
}

// sliding_window_state (proj/src/engine.cpp:271-302): prefix route vs in-window recurrence.
int orc_sliding_window_state(const double* x, i64 n, int boundary, int K, double beta, int p,
                             double* prefix_re, double* prefix_im, double* rec_re,
                             double* rec_im) {
  ORC_TRY({
    Sig sig{x, n, boundary};
    Cfg cfg{K, beta, 1, p, 0.0, 0.0, 0, kKernelIntegral, kDouble, 0};
    cfg.validate();
    const double w = cfg.angular();
    PosRing<cd> ring(-1 - K, 2 * static_cast<i64>(K) + 2);
    cd u{}, win{};
    for (int lag = 2 * K; lag >= 0; --lag) win += modulated<double>(sig, w, K - lag);
    for (i64 m = -K - 1; m <= n - 1 + K; ++m) {
      u += modulated<double>(sig, w, m);
      ring.put(m, u);
      if (m >= K) {
        const i64 j = m - K;
        if (m > K) win += modulated<double>(sig, w, m) - modulated<double>(sig, w, m - 2 * K - 1);
        const cd pv = u - ring.get(m - 2 * K - 1);
        prefix_re[j] = pv.real();
        prefix_im[j] = pv.imag();
        rec_re[j] = win.real();
        rec_im[j] = win.imag();
      }
    }
  })
}

// stability_probe (proj/src/engine.cpp:304-321)
int orc_stability_probe(const double* x, i64 n, int boundary, int K, double beta, int p,
                        double alpha, int strategy, double* max_state, double* max_err,
                        double* ref_scale, double* abs_err) {
  ORC_TRY({
    Sig sig{x, n, boundary};
    Cfg lo{K, beta, 1, p, 0.0, alpha, 0, strategy, kSingle, 0};
    Cfg hi = lo;
    hi.precision = kDouble;
    std::vector<double> c1(n), s1(n), c2(n), s2(n);
    components(sig, lo, 0, n - 1, c1.data(), s1.data(), max_state);
    components(sig, hi, 0, n - 1, c2.data(), s2.data(), nullptr);
    double scale = 0.0, worst = 0.0;
    for (i64 i = 0; i < n; ++i) {
      abs_err[i] = std::max(std::abs(c1[i] - c2[i]), std::abs(s1[i] - s2[i]));
      worst = std::max(worst, abs_err[i]);
      scale = std::max(scale, std::max(std::abs(c2[i]), std::abs(s2[i])));
    }
    *ref_scale = scale;
    *max_err = scale > 0.0 ? worst / scale : worst;
  })
}

// Sliding sums over int64 / double (Algorithms 1-3). trace_out: 6 int64 per round.
int orc_sliding_sum_i64(const i64* f, i64 n, i64 L, int blocked, int workers, i64* out,
                        i64* trace_out, int* trace_rounds) {
  ORC_TRY({
    std::vector<RoundRec> tr;
    const std::vector<i64> h = blocked ? sliding_blocked8<i64>(f, n, L, workers, &tr)
                                       : sliding_flat<i64>(f, n, L, workers, &tr);
    std::memcpy(out, h.data(), h.size() * sizeof(i64));
    if (trace_rounds) *trace_rounds = static_cast<int>(tr.size());
    if (trace_out)
      for (size_t r = 0; r < tr.size(); ++r) {
        trace_out[6 * r + 0] = tr[r].round;
        trace_out[6 * r + 1] = tr[r].stage;
        trace_out[6 * r + 2] = tr[r].r;
        trace_out[6 * r + 3] = tr[r].bit;
        trace_out[6 * r + 4] = tr[r].active;
        trace_out[6 * r + 5] = tr[r].adds;
      }
  })
}

int orc_sliding_sum_f64(const double* f, i64 n, i64 L, int blocked, int workers, double* out) {
  ORC_TRY({
    const std::vector<double> h = blocked ? sliding_blocked8<double>(f, n, L, workers, nullptr)
                                          : sliding_flat<double>(f, n, L, workers, nullptr);
    std::memcpy(out, h.data(), h.size() * sizeof(double));
  })
}

// SlidingSumPlan::make + cost_model (proj/src/sliding_sum.cpp:7-40).
int orc_sliding_plan(i64 n, i64 L, int blocked, i64* rounds, i64* padded, i64* stages,
                     i64* parallel_steps, i64* total_adds) {
  ORC_TRY({
    const Plan plan = Plan::make(n, L);
    *rounds = plan.rounds;
    *padded = plan.padded;
    *stages = Plan::stages_for(L);
    i64 adds = 0;
    if (!blocked) {
      *parallel_steps = plan.rounds;
      for (int r = 0; r < plan.rounds; ++r)
        adds += plan.n * (1 + bit_of(static_cast<std::uint64_t>(L), static_cast<unsigned>(r)));
    } else {
      *parallel_steps = 3 * Plan::stages_for(L);
      i64 rows = plan.padded, cols = 1, rest = L;
      while (rest > 0) {
        const i64 blocks = ((rows + 63) / 64) * cols;
        for (int r = 0; r < 3; ++r) {
          const int fold = bit_of(static_cast<std::uint64_t>(rest), static_cast<unsigned>(r));
          const i64 active = static_cast<i64>(16 - (1 << r)) * 8 * blocks;
          adds += active * (1 + fold);
        }
        rows /= 8;
        cols *= 8;
        rest /= 8;
      }
    }
    *total_adds = adds;
  })
}

// truncated_convolution (proj/src/kernels.cpp:35-51): out[n] = sum_j taps[j] x[n-(lo+j)].
int orc_truncated_convolution(const double* x, i64 n, int boundary, const double* taps_re,
                              const double* taps_im, i64 ntaps, i64 tap_lo, int workers,
                              double* out_re, double* out_im) {
  ORC_TRY({
    if (ntaps < 1) throw std::invalid_argument("truncated_convolution: empty kernel");
    Sig sig{x, n, boundary};
    parallel_chunks(0, n, workers, [&](i64 a, i64 b) {
      for (i64 i = a; i < b; ++i) {
        cd acc(0.0, 0.0);
        for (i64 j = 0; j < ntaps; ++j) acc += cd(taps_re[j], taps_im[j]) * sig.at(i - (tap_lo + j));
        out_re[i] = acc.real();
        out_im[i] = acc.imag();
      }
    });
  })
}

// gauss_smooth combine (proj/src/transforms.cpp:279-335). kind 0/1/2 = G/GD/GDD.
// a: P+1 (cos, orders 0..P); b: P (sin, orders 1..P); d: P+1.
int orc_gauss_smooth(const double* x, i64 n, int boundary, int kind, int K, double beta,
                     int n0, double alpha, double gamma, int strategy, int precision, int P,
                     const double* a, const double* b, const double* d, int workers,
                     double* out) {
  ORC_TRY({
    Sig sig{x, n, boundary};
    const i64 lo = -static_cast<i64>(n0), hi = n - 1 - n0;
    const double pref = n0 == 0 ? 1.0 : std::exp(-alpha * alpha / (4.0 * gamma));
    std::vector<Comp> comps(P + 1);
    parallel_chunks(0, P + 1, workers, [&](i64 a0, i64 b0) {
      for (i64 p = a0; p < b0; ++p) {
        Cfg cfg = base_cfg(K, beta, alpha, n0, strategy, precision);
        cfg.p = static_cast<int>(p);
        comps[p].c.resize(n);
        comps[p].s.resize(n);
        components(sig, cfg, lo, hi, comps[p].c.data(), comps[p].s.data());
      }
    });
    std::vector<double> acc(static_cast<size_t>(n), 0.0);
    for (int p = 0; p <= P; ++p) {
      double wc = 0.0, ws = 0.0;
      const double ap = a[p], bp = p >= 1 ? b[p - 1] : 0.0, dp = d[p];
      if (kind == 0) {
        wc = ap;
      } else if (kind == 1) {
        ws = bp;
        if (n0 != 0) wc = -alpha * ap;
      } else {
        wc = dp;
        if (n0 != 0) {
          wc += alpha * alpha * ap;
          ws = -2.0 * alpha * bp;
        }
      }
      if (wc != 0.0)
        for (i64 i = 0; i < n; ++i) acc[i] += wc * comps[p].c[i];
      if (ws != 0.0)
        for (i64 i = 0; i < n; ++i) acc[i] += ws * comps[p].s[i];
    }
    for (i64 i = 0; i < n; ++i) out[i] = acc[i] * pref;
  })
}

// morlet_direct_transform combine (proj/src/transforms.cpp:337-371).
// Complex coefficients as interleaved (re, im). sin orders must be a subsequence
// of cos orders in the same order (as fit_morlet_direct produces).
int orc_morlet_direct(const double* x, i64 n, int boundary, int K, double beta, int n0,
                      double alpha, double gamma, int strategy, int precision, int nc,
                      const int* cos_orders, const double* cos_coeffs, int ns,
                      const int* sin_orders, const double* sin_coeffs, int workers,
                      double* out) {
  ORC_TRY({
    Sig sig{x, n, boundary};
    const i64 lo = -static_cast<i64>(n0), hi = n - 1 - n0;
    const double pref = n0 == 0 ? 1.0 : std::exp(-alpha * alpha / (4.0 * gamma));
    std::vector<Comp> comps(nc);
    parallel_chunks(0, nc, workers, [&](i64 a0, i64 b0) {
      for (i64 i = a0; i < b0; ++i) {
        Cfg cfg = base_cfg(K, beta, alpha, n0, strategy, precision);
        cfg.p = cos_orders[i];
        comps[i].c.resize(n);
        comps[i].s.resize(n);
        components(sig, cfg, lo, hi, comps[i].c.data(), comps[i].s.data());
      }
    });
    Acc acc(n);
    int si = 0;
    for (int ci = 0; ci < nc; ++ci) {
      acc.add(cd(cos_coeffs[2 * ci], cos_coeffs[2 * ci + 1]), comps[ci].c);
      if (si < ns && sin_orders[si] == cos_orders[ci]) {
        acc.add(cd(sin_coeffs[2 * si], sin_coeffs[2 * si + 1]), comps[ci].s);
        ++si;
      }
    }
    for (i64 i = 0; i < n; ++i) {
      out[2 * i] = acc.re[i] * pref;
      out[2 * i + 1] = acc.im[i] * pref;
    }
  })
}

// morlet_multiply_transform combine (proj/src/transforms.cpp:373-428). env: P+1 real
// envelope cos coefficients (orders 0..P).
int orc_morlet_multiply(const double* x, i64 n, int boundary, int K, double beta, int n0,
                        double alpha, double sigma, double xi, int strategy, int precision,
                        int P, const double* env, int workers, double* out) {
  ORC_TRY({
    Sig sig{x, n, boundary};
    const i64 lo = -static_cast<i64>(n0), hi = n - 1 - n0;
    const double gamma = 1.0 / (2.0 * sigma * sigma);
    const double pref = n0 == 0 ? 1.0 : std::exp(-alpha * alpha / (4.0 * gamma));
    const double kappa = std::exp(-0.5 * xi * xi);
    const i64 nreal = 2 * static_cast<i64>(P) + 1;
    std::vector<Comp> comps(static_cast<size_t>(nreal + P + 1));
    parallel_chunks(0, static_cast<i64>(comps.size()), workers, [&](i64 a0, i64 b0) {
      for (i64 i = a0; i < b0; ++i) {
        Cfg cfg = base_cfg(K, beta, alpha, n0, strategy, precision);
        if (i < nreal) {
          const int p = static_cast<int>(i) - P;
          cfg.strategy = kKernelIntegral;
          cfg.integer_order = 0;
          cfg.omega = xi / sigma + beta * p;
        } else {
          cfg.p = static_cast<int>(i - nreal);
        }
        comps[i].c.resize(n);
        comps[i].s.resize(n);
        components(sig, cfg, lo, hi, comps[i].c.data(), comps[i].s.data());
      }
    });
    const cd carrier = n0 == 0 ? cd(1.0, 0.0)
                               : cd(std::cos(xi * n0 / sigma), std::sin(xi * n0 / sigma));
    Acc acc(n);
    for (int p = -P; p <= P; ++p) {
      const double ap = env[std::abs(p)];
      const double apr = p == 0 ? ap : 0.5 * ap;
      acc.add(carrier * apr, comps[p + P].c);
      acc.add(carrier * apr * cd(0, 1), comps[p + P].s);
    }
    for (int p = 0; p <= P; ++p) acc.add(cd(-kappa * env[p], 0.0), comps[nreal + p].c);
    for (i64 i = 0; i < n; ++i) {
      out[2 * i] = acc.re[i] * pref;
      out[2 * i + 1] = acc.im[i] * pref;
    }
  })
}

// Analytic kernels (proj/include/sft/kernels.hpp:54-73).
double orc_gauss(double sigma, double t) {
  const double g = 1.0 / (2.0 * sigma * sigma);
  return std::sqrt(g / M_PI) * std::exp(-g * t * t);
}
double orc_gauss_d(double sigma, double t) {
  const double g = 1.0 / (2.0 * sigma * sigma);
  return -2.0 * g * t * orc_gauss(sigma, t);
}
double orc_gauss_dd(double sigma, double t) {
  const double g = 1.0 / (2.0 * sigma * sigma);
  return (4.0 * g * g * t * t - 2.0 * g) * orc_gauss(sigma, t);
}
void orc_morlet(double sigma, double xi, double t, double* re, double* im) {
  const double kap = std::exp(-0.5 * xi * xi);
  const double cxi = 1.0 / std::sqrt(1.0 + std::exp(-xi * xi) - 2.0 * std::exp(-0.75 * xi * xi));
  const double env = cxi / (std::pow(M_PI, 0.25) * std::sqrt(sigma)) *
                     std::exp(-t * t / (2.0 * sigma * sigma));
  const double ph = xi * t / sigma;
  *re = env * (std::cos(ph) - kap);
  *im = env * std::sin(ph);
}

// Effective kernels (proj/src/fourier_fit.cpp:184-261, proj/src/transforms.cpp:461-477):
// series of cos/sin orders with complex coefficients on q in [-K, K], attenuation-
// weighted prefactor*e^{-alpha q} and support shifted to [-K+n0, K+n0] for ASFT.
int orc_series_taps(int K, double beta, int nc, const int* cos_orders, const double* cos_coeffs,
                    int ns, const int* sin_orders, const double* sin_coeffs, int n0,
                    double gamma, double* taps_re, double* taps_im, i64* tap_lo) {
  ORC_TRY({
    const double alpha = 2.0 * gamma * n0;
    const double pref = std::exp(-alpha * alpha / (4.0 * gamma));
    for (int i = 0; i <= 2 * K; ++i) {
      const double q = -K + i;
      double re = 0.0, im = 0.0;
      for (int c = 0; c < nc; ++c) {
        const double bs = std::cos(beta * cos_orders[c] * q);
        re += cos_coeffs[2 * c] * bs;
        im += cos_coeffs[2 * c + 1] * bs;
      }
      for (int c = 0; c < ns; ++c) {
        const double bs = std::sin(beta * sin_orders[c] * q);
        re += sin_coeffs[2 * c] * bs;
        im += sin_coeffs[2 * c + 1] * bs;
      }
      if (n0 != 0) {
        const double wgt = pref * std::exp(-alpha * q);
        re *= wgt;
        im *= wgt;
      }
      taps_re[i] = re;
      taps_im[i] = im;
    }
    *tap_lo = -K + n0;
  })
}

// morlet_multiply_effective_taps (proj/src/fourier_fit.cpp:240-255)
int orc_multiply_taps(int K, double beta, int P, const double* env, double sigma, double xi,
                      int n0, double* taps_re, double* taps_im, i64* tap_lo) {
  ORC_TRY({
    const double gamma = 1.0 / (2.0 * sigma * sigma);
    const double alpha = 2.0 * gamma * n0;
    const double pref = std::exp(-alpha * alpha / (4.0 * gamma));
    const double kap = std::exp(-0.5 * xi * xi);
    for (int i = 0; i <= 2 * K; ++i) {
      const double q = -K + i;
      double e = 0.0;
      for (int p = 0; p <= P; ++p) e += env[p] * std::cos(beta * p * q);
      const double ph = xi * (q + static_cast<double>(n0)) / sigma;
      double re = e * (std::cos(ph) - kap), im = e * std::sin(ph);
      if (n0 != 0) {
        const double wgt = pref * std::exp(-alpha * q);
        re *= wgt;
        im *= wgt;
      }
      taps_re[i] = re;
      taps_im[i] = im;
    }
    *tap_lo = -K + n0;
  })
}

}  // extern "C"
