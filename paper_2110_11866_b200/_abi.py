"""ctypes binding of include/sftgpu.h (libsftgpu.so, built in-tree by build.py).

Loading fails loudly when the library is missing: there is no Python or CPU
fallback for the transform path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsftgpu.so")
# A/B experiments may point the package at another build of the same ABI.
LIB_PATH = os.environ.get("SFTGPU_LIB", LIB_PATH)

MAX_COEFFS = 64

OK, EINVAL, ECUDA, ENOMEM, EDEGENERATE, EINTERNAL = range(6)


class Options(C.Structure):
    _fields_ = [
        ("has_half_width", C.c_int),
        ("half_width", C.c_int),
        ("has_beta", C.c_int),
        ("beta", C.c_double),
        ("tune_beta", C.c_int),
        ("has_ps", C.c_int),
        ("ps", C.c_int),
        ("strategy", C.c_int),
        ("precision", C.c_int),
    ]


class Coeffs(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("half_width", C.c_int),
        ("beta", C.c_double),
        ("n_cos", C.c_int),
        ("n_sin", C.c_int),
        ("cos_orders", C.c_int * MAX_COEFFS),
        ("sin_orders", C.c_int * MAX_COEFFS),
        ("cos_coeffs", C.c_double * (2 * MAX_COEFFS)),
        ("sin_coeffs", C.c_double * (2 * MAX_COEFFS)),
        ("fit_rmse_percent", C.c_double),
        ("sigma", C.c_double),
        ("xi", C.c_double),
        ("n0", C.c_int),
    ]


class GaussBundle(C.Structure):
    _fields_ = [
        ("sigma", C.c_double),
        ("half_width", C.c_int),
        ("beta", C.c_double),
        ("max_order", C.c_int),
        ("a", C.c_double * MAX_COEFFS),
        ("b", C.c_double * MAX_COEFFS),
        ("d", C.c_double * MAX_COEFFS),
        ("fit_rmse_g", C.c_double),
        ("fit_rmse_gd", C.c_double),
        ("fit_rmse_gdd", C.c_double),
    ]


class Spec(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("sigma", C.c_double),
        ("xi", C.c_double),
        ("half_width", C.c_int),
        ("max_order", C.c_int),
        ("ps", C.c_int),
        ("pd", C.c_int),
        ("beta", C.c_double),
        ("n0", C.c_int),
        ("alpha", C.c_double),
        ("strategy", C.c_int),
        ("precision", C.c_int),
        ("abbreviation", C.c_char * 32),
        ("kernel_rmse_percent", C.c_double),
        ("gauss", GaussBundle),
        ("morlet", Coeffs),
        ("envelope", Coeffs),
    ]


class Config(C.Structure):
    _fields_ = [
        ("half_width", C.c_int),
        ("beta", C.c_double),
        ("integer_order", C.c_int),
        ("p", C.c_int),
        ("omega", C.c_double),
        ("alpha", C.c_double),
        ("n0", C.c_int),
        ("strategy", C.c_int),
        ("precision", C.c_int),
        ("window_2k1", C.c_int),
    ]


# Every symbol include/sftgpu.h declares, with its ctypes signature.
_P, _I, _D, _I64, _U64 = C.c_void_p, C.c_int, C.c_double, C.c_int64, C.c_uint64
SIGNATURES = {
    "sftgpu_last_error": ([], C.c_char_p),
    "sftgpu_version": ([], C.c_char_p),
    "sftgpu_parse_abbreviation": ([C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)], _I),
    "sftgpu_encode_abbreviation": ([_I, _I, _I, C.c_char_p, _I], _I),
    "sftgpu_make_transform_spec": ([C.c_char_p, _D, _D, C.POINTER(Options), C.POINTER(Spec)], _I),
    "sftgpu_make_gauss_spec": ([_D, _I, _I, _I, C.POINTER(Options), C.POINTER(Spec)], _I),
    "sftgpu_make_morlet_direct_spec": ([_D, _D, _I, _I, C.POINTER(Options), C.POINTER(Spec)], _I),
    "sftgpu_make_morlet_multiply_spec": ([_D, _D, _I, _I, C.POINTER(Options), C.POINTER(Spec)], _I),
    "sftgpu_effective_kernel": ([C.POINTER(Spec), _P, _I64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], _I),
    "sftgpu_fit_mmse": ([_P, _I, _D, _I, _P, _I, _P, _I, C.POINTER(Coeffs)], _I),
    "sftgpu_fit_gaussian_bundle": ([_D, _I, _I, _D, C.POINTER(GaussBundle)], _I),
    "sftgpu_fit_morlet_direct": ([_D, _D, _I, _I, _I, _D, _I, C.POINTER(Coeffs)], _I),
    "sftgpu_fit_morlet_envelope": ([_D, _D, _I, _I, _D, C.POINTER(Coeffs)], _I),
    "sftgpu_select_optimal_ps": ([_D, _D, _I, _I, _I, C.POINTER(C.c_int)], _I),
    "sftgpu_morlet_direct_kernel_rmse": ([_D, _D, _I, _I, _I, _I, C.POINTER(C.c_double)], _I),
    "sftgpu_morlet_multiply_kernel_rmse": ([_D, _D, _I, _I, _I, C.POINTER(C.c_double)], _I),
    "sftgpu_gauss_kernel_rmse": ([C.POINTER(GaussBundle), _I, _I, C.POINTER(C.c_double)], _I),
    "sftgpu_tune_beta_gauss": ([_D, _I, _I, _I, C.POINTER(C.c_double), C.POINTER(C.c_double)], _I),
    "sftgpu_write_coefficient_sets": ([C.c_char_p, C.POINTER(Coeffs), _I], _I),
    "sftgpu_read_coefficient_sets": ([C.c_char_p, C.POINTER(Coeffs), _I, C.POINTER(C.c_int)], _I),
    "sftgpu_make_morlet_direct_spec_from_coeffs": ([C.POINTER(Coeffs), _I, _I, _I, C.POINTER(Spec)], _I),
    "sftgpu_transform_plan_create": ([C.POINTER(Spec), _I64, _I64, _I, C.POINTER(_P)], _I),
    "sftgpu_transform_plan_create_range": ([C.POINTER(Spec), _I64, _I64, _I, _I64, _I64, C.POINTER(_P)], _I),
    "sftgpu_transform_plan_create_ex": ([C.POINTER(Spec), _I64, _I64, _I, _I64, _I64, _I, C.POINTER(_P)], _I),
    "sftgpu_transform_oneshot": ([C.POINTER(Spec), _I64, _I, C.c_void_p, C.c_void_p, C.POINTER(_I)], _I),
    "sftgpu_oneshot_cache_clear": ([], None),
    "sftgpu_multiscale_plan_create": ([C.POINTER(Spec), _I, _I64, _I, _I64, _I64, C.POINTER(_P)], _I),
    "sftgpu_plan_describe": ([_P, C.POINTER(C.c_int64), _I], _I),
    "sftgpu_transform_execute": ([_P, _P, _I64, _P, _I64, _P], _I),
    "sftgpu_transform_execute_host": ([_P, _P, _P, _P], _I),
    "sftgpu_transform_execute_host_async": ([_P, _P, _P, _P], _I),
    "sftgpu_plan_synchronize": ([_P], _I),
    "sftgpu_plan_output_is_complex": ([_P], _I),
    "sftgpu_plan_launches_per_execute": ([_P], _I),
    "sftgpu_components_plan_create": ([C.POINTER(Config), _I, _I64, _I64, _I, _I64, _I64, _I, C.POINTER(_P)], _I),
    "sftgpu_components_execute": ([_P, _P, _P, _P, _P], _I),
    "sftgpu_components_execute_host": ([_P, _P, _P, _P, _P], _I),
    "sftgpu_plan_destroy": ([_P], None),
    "sftgpu_generate_signal_host": ([_I, _I64, _U64, _P], _I),
    "sftgpu_truncated_convolution_host": ([_P, _I64, _I, _P, _I64, _I64, _P], _I),
    "sftgpu_sliding_sum_plan": ([_I64, _I64, _I, C.POINTER(C.c_int64)], _I),
    "sftgpu_sliding_sum": ([_I, _I, _P, _I64, _I64, _P, _P], _I),
    "sftgpu_sliding_sum_host": ([_I, _I, C.c_void_p, _I64, _I64, C.c_void_p], _I),
    "sftgpu_tune_beta": ([C.CFUNCTYPE(C.c_double, C.c_double, C.c_void_p), C.c_void_p, _I, C.POINTER(C.c_double),
                          C.POINTER(C.c_double)], _I),
    "sftgpu_reconstruct": ([C.POINTER(Coeffs), C.c_void_p, _I64, C.c_void_p], _I),
    "sftgpu_sft_via_sliding_sum": ([C.POINTER(Config), C.c_void_p, _I64, _I, C.c_void_p, C.c_void_p], _I),
    "sftgpu_components_replay": ([C.POINTER(Config), _I, C.c_void_p, _I64, _I, _I64, _I64, C.c_void_p, C.c_void_p,
                                  C.c_void_p], _I),
    "sftgpu_generate_signal": ([_I, _I64, _U64, _I64, _I, _P, _P], _I),
    "sftgpu_truncated_convolution": ([_P, _I64, _I, _P, _I64, _I64, _P, _P], _I),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2110_11866_b200.build` "
                "(there is no CPU fallback for the SFT/ASFT path)"
            )
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


class SftGpuError(RuntimeError):
    """CUDA / internal failure reported by libsftgpu."""


class FitDegenerateError(RuntimeError):
    """Gram matrix condition estimate exceeds 1e12 (proj/src/fourier_fit.cpp:37-38)."""


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().sftgpu_last_error().decode()
    if rc == EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == EDEGENERATE:
        raise FitDegenerateError(msg)
    if rc == ENOMEM:
        raise MemoryError(msg)
    raise SftGpuError(msg)
