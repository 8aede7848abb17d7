/*
 * sftgpu.h — C ABI of the B200-native SFT/ASFT hot path (libsftgpu.so).
 *
 * Drop-in boundary for the reference library's transform path
 * (/root/reference/proj, arXiv 2110.11866). Plain C types only: pointers, sizes,
 * ints, doubles. Device pointers are CUDA global-memory addresses on the current
 * device; `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 * Every entry point returns an sftgpu_status; on failure sftgpu_last_error()
 * returns a thread-local message. There is no CPU fallback: when no CUDA device
 * is present the execute functions fail with SFTGPU_ECUDA.
 *
 * Reference interfaces each entry point replaces (file:line under proj/):
 *   sftgpu_make_gauss_spec          make_gauss_spec            src/transforms.cpp:122-148
 *   sftgpu_make_morlet_direct_spec  make_morlet_direct_spec    src/transforms.cpp:151-182
 *   sftgpu_make_morlet_multiply_spec make_morlet_multiply_spec src/transforms.cpp:184-213
 *   sftgpu_make_transform_spec      make_transform_spec        src/transforms.cpp:215-242
 *   sftgpu_parse_abbreviation       parse_abbreviation         src/transforms.cpp:53-95
 *   sftgpu_encode_abbreviation      encode_abbreviation        src/transforms.cpp:97-120
 *   sftgpu_effective_kernel         effective_kernel           src/transforms.cpp:461-477
 *   sftgpu_select_optimal_ps        select_optimal_ps          src/fourier_fit.cpp:379-393
 *   sftgpu_tune_beta_gauss          tune_beta_gauss            src/fourier_fit.cpp:440-447
 *   sftgpu_fit_gaussian_bundle      fit_gaussian_bundle        src/fourier_fit.cpp:131-161
 *   sftgpu_fit_morlet_direct        fit_morlet_direct          src/fourier_fit.cpp:293-340
 *   sftgpu_fit_morlet_envelope      fit_morlet_envelope        src/fourier_fit.cpp:342-355
 *   sftgpu_fit_mmse                 fit_mmse                   src/fourier_fit.cpp:67-105
 *   sftgpu_transform_plan_create +
 *   sftgpu_transform_execute        gauss_smooth / morlet_direct_transform /
 *                                   morlet_multiply_transform / apply_transform
 *                                                              src/transforms.cpp:279-459
 *   sftgpu_components_plan_create +
 *   sftgpu_components_execute       components_over / sft_components /
 *                                   asft_components / sft_via_sliding_sum
 *                                                              src/engine.cpp:255-269, :323-337
 *   sftgpu_components_replay        recursive_components (Recursive1/2 with the
 *                                   reference's rounding)      src/engine.cpp:53-120
 *   sftgpu_generate_signal          make_test_signal           src/signal.cpp:24-51
 *   sftgpu_truncated_convolution    truncated_convolution      src/kernels.cpp:35-51
 */
#ifndef SFTGPU_H
#define SFTGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SFTGPU_OK = 0,
  SFTGPU_EINVAL = 1,   /* std::invalid_argument in the reference */
  SFTGPU_ECUDA = 2,    /* CUDA runtime / launch failure, or no device */
  SFTGPU_ENOMEM = 3,   /* device or host allocation failure */
  SFTGPU_EDEGENERATE = 4, /* FitDegenerateError (Gram condition > 1e12) */
  SFTGPU_EINTERNAL = 5
} sftgpu_status;

/* BoundaryPolicy (include/sft/signal.hpp:12) */
enum { SFTGPU_BOUNDARY_ZERO = 0, SFTGPU_BOUNDARY_CLAMP = 1 };
/* Precision (include/sft/signal.hpp:15): device arrays are float / double. */
enum { SFTGPU_SINGLE = 0, SFTGPU_DOUBLE = 1 };
/* Strategy (include/sft/engine.hpp:16). Accepted for API parity; every strategy
 * executes the same fused window-recurrence scan on the GPU (results agree with
 * the reference's strategies to rounding). */
enum { SFTGPU_KERNEL_INTEGRAL = 0, SFTGPU_RECURSIVE1 = 1, SFTGPU_RECURSIVE2 = 2 };
/* TransformKind (include/sft/transforms.hpp:11-19) */
enum {
  SFTGPU_GAUSS = 0,
  SFTGPU_GAUSS_D = 1,
  SFTGPU_GAUSS_DD = 2,
  SFTGPU_MORLET_DIRECT = 3,
  SFTGPU_MORLET_MULTIPLY = 4,
  SFTGPU_TRUNC_CONV_GAUSS = 5,  /* GCT3 */
  SFTGPU_TRUNC_CONV_MORLET = 6  /* MCT3 */
};
/* GaussKind (include/sft/fourier_fit.hpp:101) */
enum { SFTGPU_GK_VALUE = 0, SFTGPU_GK_DERIV1 = 1, SFTGPU_GK_DERIV2 = 2 };
/* CoeffKind (include/sft/fourier_fit.hpp:49) */
enum {
  SFTGPU_CK_GAUSS_COS = 0,
  SFTGPU_CK_GAUSS_DERIV_SIN = 1,
  SFTGPU_CK_GAUSS_DERIV2_COS = 2,
  SFTGPU_CK_MORLET_DIRECT = 3,
  SFTGPU_CK_MORLET_MULTIPLY = 4
};
/* make_test_signal kinds (include/sft/signal.hpp:47) */
enum { SFTGPU_SIG_IMPULSE = 0, SFTGPU_SIG_CONSTANT = 1, SFTGPU_SIG_CHIRP = 2, SFTGPU_SIG_NOISE = 3 };

#define SFTGPU_MAX_COEFFS 64

/* TransformOptions (include/sft/transforms.hpp:43-50). has_* = 0 means "unset". */
typedef struct {
  int has_half_width;
  int half_width;
  int has_beta;
  double beta;
  int tune_beta;
  int has_ps;
  int ps;
  int strategy;
  int precision;
} sftgpu_options;

/* CoefficientSet (include/sft/fourier_fit.hpp:56-68); coefficients are complex,
 * stored interleaved (re, im). */
typedef struct {
  int kind;
  int half_width;
  double beta;
  int n_cos;
  int n_sin;
  int cos_orders[SFTGPU_MAX_COEFFS];
  int sin_orders[SFTGPU_MAX_COEFFS];
  double cos_coeffs[2 * SFTGPU_MAX_COEFFS];
  double sin_coeffs[2 * SFTGPU_MAX_COEFFS];
  double fit_rmse_percent;
  double sigma;
  double xi;
  int n0;
} sftgpu_coeffs;

/* GaussianFitBundle (include/sft/fourier_fit.hpp:88-99): a (P+1), b (P), d (P+1). */
typedef struct {
  double sigma;
  int half_width;
  double beta;
  int max_order;
  double a[SFTGPU_MAX_COEFFS];
  double b[SFTGPU_MAX_COEFFS];
  double d[SFTGPU_MAX_COEFFS];
  double fit_rmse_g;
  double fit_rmse_gd;
  double fit_rmse_gdd;
} sftgpu_gauss_bundle;

/* TransformSpec (include/sft/transforms.hpp:23-41). Exactly one of the
 * coefficient members is meaningful, selected by `kind`. */
typedef struct {
  int kind;
  double sigma;
  double xi;        /* Morlet kinds */
  int half_width;   /* K */
  int max_order;    /* P (Gauss) or P_M (multiply) */
  int ps;           /* direct-method start order */
  int pd;           /* direct-method order count */
  double beta;
  int n0;
  double alpha;
  int strategy;
  int precision;
  char abbreviation[32];
  double kernel_rmse_percent;
  sftgpu_gauss_bundle gauss;   /* Gauss kinds */
  sftgpu_coeffs morlet;        /* MorletDirect */
  sftgpu_coeffs envelope;      /* MorletMultiply */
} sftgpu_spec;

/* SftConfig (include/sft/engine.hpp:41-60) for the components entry points. */
typedef struct {
  int half_width;
  double beta;
  int integer_order; /* 1: omega = beta * p; 0: omega given (real frequency) */
  int p;
  double omega;
  double alpha;
  int n0;
  int strategy;
  int precision;
  int window_2k1;
} sftgpu_config;

typedef struct sftgpu_plan sftgpu_plan;

const char* sftgpu_last_error(void);
const char* sftgpu_version(void);

/* ---------------- host precompute (coefficient fitting; untimed in the reference) */
int sftgpu_parse_abbreviation(const char* abbrev, int* kind, int* n0, int* order);
int sftgpu_encode_abbreviation(int kind, int n0, int order, char* out, int out_len);
int sftgpu_make_transform_spec(const char* abbrev, double sigma, double xi,
                               const sftgpu_options* opt, sftgpu_spec* out);
int sftgpu_make_gauss_spec(double sigma, int gauss_kind, int max_order, int n0,
                           const sftgpu_options* opt, sftgpu_spec* out);
int sftgpu_make_morlet_direct_spec(double sigma, double xi, int pd, int n0,
                                   const sftgpu_options* opt, sftgpu_spec* out);
int sftgpu_make_morlet_multiply_spec(double sigma, double xi, int pm, int n0,
                                     const sftgpu_options* opt, sftgpu_spec* out);
/* taps buffers hold 2*K+1 complex values (interleaved); *tap_lo receives the support start. */
int sftgpu_effective_kernel(const sftgpu_spec* spec, double* taps, int64_t taps_capacity,
                            int64_t* n_taps, int64_t* tap_lo);
int sftgpu_fit_mmse(const double* target_re_im, int half_width, double beta, int n_cos,
                    const int* cos_orders, int n_sin, const int* sin_orders, int coeff_kind,
                    sftgpu_coeffs* out);
int sftgpu_fit_gaussian_bundle(double sigma, int half_width, int max_order, double beta,
                               sftgpu_gauss_bundle* out);
int sftgpu_fit_morlet_direct(double sigma, double xi, int half_width, int ps, int pd,
                             double beta, int n0, sftgpu_coeffs* out);
int sftgpu_fit_morlet_envelope(double sigma, double xi, int half_width, int max_order,
                               double beta, sftgpu_coeffs* out);
int sftgpu_select_optimal_ps(double sigma, double xi, int half_width, int pd, int n0, int* ps);
int sftgpu_morlet_direct_kernel_rmse(double sigma, double xi, int half_width, int ps, int pd,
                                     int n0, double* rmse);
int sftgpu_morlet_multiply_kernel_rmse(double sigma, double xi, int half_width, int pm,
                                       int n0, double* rmse);
int sftgpu_gauss_kernel_rmse(const sftgpu_gauss_bundle* b, int gauss_kind, int n0,
                             double* rmse);
int sftgpu_tune_beta_gauss(double sigma, int half_width, int max_order, int n0,
                           double* beta, double* rmse);
/* tune_beta (src/fourier_fit.cpp:395-438): 33-point prescan of rmse_of_beta over
 * [0.5 pi/K, 1.5 pi/K], then golden section to 1e-4 relative. */
int sftgpu_tune_beta(double (*rmse_of_beta)(double beta, void* user), void* user, int half_width,
                     double* beta, double* rmse);
/* reconstruct (src/fourier_fit.cpp:107-129): the fitted series at n points, complex
 * values interleaved (re, im) into out_re_im[2n]. */
int sftgpu_reconstruct(const sftgpu_coeffs* coeffs, const double* points, int64_t n, double* out_re_im);

/* Coefficient files, "sft-coefficients v1" text format
 * (replaces write_coefficient_sets / read_coefficient_sets, src/coeff_io.cpp:21-101). */
int sftgpu_write_coefficient_sets(const char* path, const sftgpu_coeffs* sets, int n_sets);
int sftgpu_read_coefficient_sets(const char* path, sftgpu_coeffs* sets, int capacity, int* n_sets);
/* MorletDirect spec from a stored coefficient set (the CLI's --coeffs substitution,
 * src/cli.cpp:224-280); kernel RMSE recomputed when recompute_rmse != 0. */
int sftgpu_make_morlet_direct_spec_from_coeffs(const sftgpu_coeffs* set, int precision, int strategy,
                                               int recompute_rmse, sftgpu_spec* out);

/* ---------------- device execution (the hot path) */
/* Transform plan for `batch` signals of `n` samples each, laid out
 * [batch][ld_x] in device memory of the spec's precision (float/double).
 * Output: [batch][ld_out] real (Gauss kinds) or complex interleaved (Morlet kinds),
 * same precision. The plan owns its look-back workspace; it is bound to one
 * stream at a time (like a cuFFT plan). */
int sftgpu_transform_plan_create(const sftgpu_spec* spec, int64_t n, int64_t batch,
                                 int boundary, sftgpu_plan** plan);
/* Output range [out_begin, out_begin + out_count) of signals of n samples: the plan
 * reads the samples it needs (window halo K + n0 on each side, boundary policy at the
 * signal ends) from the full signal and writes out_count outputs. Used to shard one
 * long signal by chunk across GPUs without any cross-GPU carry. */
int sftgpu_transform_plan_create_range(const sftgpu_spec* spec, int64_t n, int64_t batch, int boundary,
                                       int64_t out_begin, int64_t out_count, sftgpu_plan** plan);
/* As _range, with an execution-mode hint: 0 auto, 1 sequential (one CTA per
 * (signal, chunk), chunks start from their own warm-up), 2 decoupled look-back,
 * 3 tensor cores (K4: chunked scan as tcgen05 3xTF32 GEMMs; fp32 transforms with <= 8
 * orders sharing one injection constant, else SFTGPU_EINVAL). Auto picks K4 for such
 * transforms when they span >= 4 x 148 tiles of 4096 outputs (SFTGPU_NO_TC=1 disables). */
int sftgpu_transform_plan_create_ex(const sftgpu_spec* spec, int64_t n, int64_t batch, int boundary,
                                    int64_t out_begin, int64_t out_count, int mode_hint, sftgpu_plan** plan);
/* Multi-scale plan (scalogram, BASELINE config 5): n_specs transforms of ONE signal of n
 * samples, output rows s = 0..n_specs-1 ([n_specs][ld_out] real or [n_specs][ld_out][2]
 * complex), each over output range [out_begin, out_begin + out_count). One persistent
 * tensor-core (K4) launch walks every scale's fixed chunks, balanced over the SMs by cost,
 * instead of one launch per scale (replaces the reference's per-scale
 * apply_transform / morlet_direct_transform calls, proj/src/transforms.cpp:337-371).
 * Every spec must be fp32 and K4-eligible with the same number of orders and output kind
 * (all Morlet-direct specs of a scalogram are); at most 128 specs per plan. Executed with
 * sftgpu_transform_execute (x: the one signal) or sftgpu_transform_execute_host. */
int sftgpu_multiscale_plan_create(const sftgpu_spec* specs, int n_specs, int64_t n, int boundary,
                                  int64_t out_begin, int64_t out_count, sftgpu_plan** plan);
int sftgpu_transform_execute(sftgpu_plan* plan, const void* x, int64_t ld_x, void* out,
                             int64_t ld_out, void* stream);
/* Same, from/to HOST memory of the plan's precision (host<->device copies included;
 * pinned memory recommended). Synchronises `stream` before returning. Large tensor-core
 * (K4) plans pipeline sub-batches of signals through the plan's copy-in / compute /
 * copy-out streams inside the call, so the copies of one sub-batch overlap the kernel
 * of the next. */
int sftgpu_transform_execute_host(sftgpu_plan* plan, const void* x_host, void* out_host,
                                  void* stream);
/* Pipelined variant for streams of host buffers: enqueues H2D of x_host, the transform
 * and D2H into out_host on the plan's internal copy-in / compute / copy-out streams
 * (three staging slots) and returns without waiting, so the copy-in of the next call,
 * this call's kernel and the previous call's copy-out overlap. x_host must hold its data
 * when the call is made (it is not ordered after work queued on `stream`); `stream`
 * waits for this call's D2H: after cudaStreamSynchronize(stream) (or
 * sftgpu_plan_synchronize) out_host holds the result. x_host must stay valid and
 * out_host untouched until then; host buffers must be pinned for the copies to overlap.
 * Do not interleave with sftgpu_transform_execute on the same plan while calls are in
 * flight (they share the look-back workspace). */
int sftgpu_transform_execute_host_async(sftgpu_plan* plan, const void* x_host, void* out_host,
                                        void* stream);
/* Blocks until every pipelined call on the plan has finished. */
int sftgpu_plan_synchronize(sftgpu_plan* plan);
/* One transform of one fp64 HOST signal, the signature the reference's drop-in calls
 * need (apply_transform / gauss_smooth / morlet_direct_transform /
 * morlet_multiply_transform, proj/include/sft/transforms.hpp:86-102, which take an
 * Eigen::ArrayXd signal and return ArrayXcd values): x_host = n doubles, out_host = n
 * doubles (real output) or 2n (complex, interleaved re/im); *complex_out tells which.
 * Plans are cached inside the library per (spec, n, boundary, device), so repeated
 * calls reuse one plan, its device buffers and its pinned staging (single-precision
 * specs convert fp64 <-> fp32 on the host, into / out of that staging). Thread-safe (one
 * call at a time per cached plan). */
int sftgpu_transform_oneshot(const sftgpu_spec* spec, int64_t n, int boundary, const double* x_host,
                             double* out_host, int* complex_out);
/* Drops every cached one-shot plan (frees their device and pinned buffers). */
void sftgpu_oneshot_cache_clear(void);
/* 1 if the transform output is complex, 0 if real. */
int sftgpu_plan_output_is_complex(const sftgpu_plan* plan);
/* Plan geometry: info[0..10] = {sequential, direct-convolution, positions per thread,
 * positions per tile, warm-up tiles, chunks per signal, CTAs per launch, launches,
 * orders evaluated, injection group mode of the first launch (0 shared real, 1 split,
 * 2 per order, 3 shared complex), tensor-core kernel K4}. */
int sftgpu_plan_describe(const sftgpu_plan* plan, int64_t* info, int n_info);
/* Number of kernel launches one execute issues. */
int sftgpu_plan_launches_per_execute(const sftgpu_plan* plan);

/* Component plan: n_orders configs sharing K, alpha, precision; output range
 * [lo, hi]; c and s are [n_orders][batch][hi-lo+1] (plan precision).
 * mode: 0 components_over, 1 sft_components (requires alpha == 0, lo=0, hi=n-1),
 * 2 asft_components (requires alpha > 0, lo=0, hi=n-1). */
int sftgpu_components_plan_create(const sftgpu_config* cfgs, int n_orders, int64_t n,
                                  int64_t batch, int boundary, int64_t lo, int64_t hi,
                                  int mode, sftgpu_plan** plan);
int sftgpu_components_execute(sftgpu_plan* plan, const void* x, void* c, void* s,
                              void* stream);

/* Same, from/to HOST memory of the plan's precision; synchronises `stream`. */
int sftgpu_components_execute_host(sftgpu_plan* plan, const void* x_host, void* c_host, void* s_host,
                                   void* stream);

void sftgpu_plan_destroy(sftgpu_plan* plan);

/* Device splitmix64 signal generator, bit-identical to make_test_signal
 * (batch signals with seeds seed+i). dtype: SFTGPU_SINGLE/DOUBLE. */
int sftgpu_generate_signal(int kind, int64_t n, uint64_t seed, int64_t batch, int dtype,
                           void* out, void* stream);

/* GPU direct truncated convolution (GCT3/MCT3 and the exactness oracle):
 * out[n] = sum_j taps[j] x[n - (tap_lo + j)], double precision, complex taps
 * interleaved, complex output interleaved. All pointers device. */
int sftgpu_truncated_convolution(const double* x, int64_t n, int boundary,
                                 const double* taps, int64_t n_taps, int64_t tap_lo,
                                 double* out, void* stream);
/* The paper's data-parallel sliding sum h[n] = sum_{k<L} f[n+k], n in [0, N-L]
 * (sliding_sum_flat / sliding_sum_blocked8, include/sft/sliding_sum.hpp:89-234): Algorithm 1
 * (flat doubling) or Algorithms 2-3 (blocked8, (16,8) tiles) as GPU kernels with the reference's
 * exact addition trees (bit-identical for int64 and fp64). Device buffers; synchronous.
 * info (plan + cost model, src/sliding_sum.cpp:7-40): {rounds R, padded size, blocked stages,
 * parallel steps, total adds}. */
enum { SFTGPU_SS_I64 = 0, SFTGPU_SS_F64 = 1, SFTGPU_SS_C128 = 2 };
int sftgpu_sliding_sum_plan(int64_t n, int64_t L, int blocked, int64_t* info);
int sftgpu_sliding_sum(int dtype, int blocked, const void* f, int64_t n, int64_t L, void* out, void* stream);
/* sft_via_sliding_sum (src/engine.cpp:183-219, 323-337): the components of one SftConfig
 * over the whole signal by the reference's sliding-sum route, on the GPU: the rebased
 * phased sequence, the K5 flat window sums (paper Algorithm 1, complex128), rescale and
 * phase removal. HOST fp64 signal in, c = Re / s = -Im out (n each); synchronous. The
 * same argument checks as the reference (alpha * N / 2 > 600 rejected). */
int sftgpu_sft_via_sliding_sum(const sftgpu_config* cfg, const double* x_host, int64_t n, int boundary,
                               double* c_host, double* s_host);

/* The reference's recursive strategies with the reference's own rounding (K7,
 * src/engine.cpp:53-120 recursive_components, dispatched from :221-243): Recursive1
 * (v = z v + x) or Recursive2 (the real second-order form), each step in the reference's
 * operation order without FMA contraction (pass 1, one GPU thread per order, filter states
 * in HBM), then the 2K or 2K+1 truncation window, the z^{-K} unwind and the sink (pass 2,
 * parallel). Bit-identical to the reference's components_over for these strategies, in
 * Single (float arithmetic) and Double. The kernel-integral window recurrence (K1, every
 * strategy through sftgpu_components_plan_create) is the fast path and the more accurate
 * one; this entry is for callers who need the reference's numbers exactly.
 * cfgs: n_orders configs with strategy SFTGPU_RECURSIVE1/2 (any K / alpha / precision mix);
 * HOST fp64 signal in; c = Re, s = -Im out, [n_orders][hi - lo + 1]; max_state (NULL or
 * [n_orders]) = the peak |filter state| over the chain, the quantity stability_probe
 * reports (src/engine.cpp:101, :304-312; the root of the peak |v|^2 in fp64, which may
 * differ from the reference's hypot in the Scalar precision in the last bits); synchronous. */
int sftgpu_components_replay(const sftgpu_config* cfgs, int n_orders, const double* x_host, int64_t n,
                             int boundary, int64_t lo, int64_t hi, double* c_host, double* s_host,
                             double* max_state);

/* Host-memory variants (device buffers managed internally; synchronous). */
int sftgpu_sliding_sum_host(int dtype, int blocked, const void* f_host, int64_t n, int64_t L, void* out_host);
int sftgpu_generate_signal_host(int kind, int64_t n, uint64_t seed, double* out_host);
int sftgpu_truncated_convolution_host(const double* x_host, int64_t n, int boundary,
                                      const double* taps_host, int64_t n_taps, int64_t tap_lo,
                                      double* out_host);

#ifdef __cplusplus
}
#endif

#endif /* SFTGPU_H */
