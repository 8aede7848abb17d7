"""TEST INFRASTRUCTURE ONLY — the reference library itself, compiled from its own sources
under /root/reference/proj by ``oracle/ref.mk`` (mini-Eigen / mini-doctest shims in
``oracle/ref_shim``) into ``oracle/_ref/libsftref.so``, called through the C bridge
``oracle/ref_bridge.cpp``.

Used by ``tests/`` (to pin the restated oracle and the GPU path to the literal
reference) and by ``bench.py``'s reference arm / cpu_baseline leg (the timed CPU
reference). The product package never imports it. On the GPU box /root/reference is
absent: the prebuilt ``oracle/_ref`` (git-ignored, shipped with the snapshot) is used.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/proj"
OUT = os.path.join(_HERE, "_ref")
LIB_PATH = os.path.join(OUT, "libsftref.so")
TESTS_BIN = os.path.join(OUT, "ref_tests")
ACCEPTANCE_BIN = os.path.join(OUT, "acceptance")
_lib = None

KERNEL_INTEGRAL, RECURSIVE1, RECURSIVE2 = 0, 1, 2
SINGLE, DOUBLE = 0, 1


class RefError(RuntimeError):
    pass


class RefInvalidArgument(ValueError):
    pass


def source_available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "src"))


def build(jobs: int | None = None) -> str:
    """Compile the reference (only where its sources exist; elsewhere the prebuilt
    oracle/_ref is used as is)."""
    if source_available():
        subprocess.check_call(["make", "-s", f"-j{jobs or os.cpu_count() or 4}", "-f",
                               os.path.join(_HERE, "ref.mk"), f"REF={REF_SRC}"])
    if not os.path.exists(LIB_PATH):
        raise RefError("oracle/_ref/libsftref.so is not built and the reference sources are absent")
    return LIB_PATH


def available() -> bool:
    return os.path.exists(LIB_PATH) or source_available()


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        d, i, i64, u64, P = C.c_double, C.c_int, C.c_int64, C.c_uint64, C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_make_transform_spec.argtypes = [C.c_char_p, d, d, i, i, i, d, i, i, i, i, i, C.POINTER(P)]
        L.ref_spec_free.argtypes = [P]
        L.ref_spec_free.restype = None
        L.ref_spec_set_engine.argtypes = [P, i, i]
        L.ref_spec_info.argtypes = [P, P]
        L.ref_apply_transform.argtypes = [P, P, i64, i, i, P]
        L.ref_effective_kernel.argtypes = [P, P, i64, C.POINTER(i64), C.POINTER(i64)]
        L.ref_spec_gauss_coeffs.argtypes = [P, i, C.POINTER(i), P, P, P]
        L.ref_spec_morlet_coeffs.argtypes = [P, i, i, C.POINTER(i), P, P, C.POINTER(i), P, P]
        L.ref_components.argtypes = [P, i64, i, i, d, i, i, d, d, i, i, i, i64, i64, i, P, P]
        L.ref_make_test_signal.argtypes = [i, i64, u64, P]
        L.ref_sliding_sum_flat_i64.argtypes = [P, i64, i64, P]
        _lib = L
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().ref_last_error().decode()
    if rc == 1:
        raise RefInvalidArgument(msg)
    raise RefError(msg)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Spec:
    """An ``sft::TransformSpec`` built by the reference's own factory
    (``make_transform_spec``, proj/src/transforms.cpp)."""

    def __init__(self, abbrev: str, sigma: float, xi: float, *, half_width=None, beta=None, tune_beta=False,
                 ps=None, strategy=RECURSIVE2, precision=DOUBLE):
        h = C.c_void_p()
        _check(lib().ref_make_transform_spec(abbrev.encode(), sigma, xi, int(half_width is not None),
                                             half_width or 0, int(beta is not None), beta or 0.0, int(tune_beta),
                                             int(ps is not None), ps or 0, strategy, precision, C.byref(h)))
        self._h = h
        self._free = lib().ref_spec_free
        info = np.zeros(11)
        _check(lib().ref_spec_info(h, _p(info)))
        (self.kind, self.half_width, self.beta, self.n0, self.alpha, self.ps, self.pd, self.max_order,
         self.kernel_rmse_percent, self.sigma, self.xi) = (
            int(info[0]), int(info[1]), info[2], int(info[3]), info[4], int(info[5]), int(info[6]), int(info[7]),
            info[8], info[9], info[10])
        self.strategy, self.precision = strategy, precision

    def set_engine(self, strategy: int, precision: int) -> "Spec":
        _check(lib().ref_spec_set_engine(self._h, strategy, precision))
        self.strategy, self.precision = strategy, precision
        return self

    def gauss_coeffs(self):
        P = C.c_int()
        a, b, d = np.zeros(64), np.zeros(64), np.zeros(64)
        _check(lib().ref_spec_gauss_coeffs(self._h, 64, C.byref(P), _p(a), _p(b), _p(d)))
        p = P.value
        return a[:p + 1].copy(), b[:p].copy(), d[:p + 1].copy()

    def morlet_coeffs(self, envelope: bool = False):
        nc, ns = C.c_int(), C.c_int()
        co, so = np.zeros(64, dtype=np.int32), np.zeros(64, dtype=np.int32)
        cc, sc = np.zeros(128), np.zeros(128)
        _check(lib().ref_spec_morlet_coeffs(self._h, 1 if envelope else 0, 64, C.byref(nc), _p(co), _p(cc),
                                            C.byref(ns), _p(so), _p(sc)))
        n, m = nc.value, ns.value
        return (co[:n].tolist(), cc[:2 * n:2] + 1j * cc[1:2 * n:2], so[:m].tolist(), sc[:2 * m:2] + 1j * sc[1:2 * m:2])

    def effective_kernel(self):
        n, lo = C.c_int64(), C.c_int64()
        _check(lib().ref_effective_kernel(self._h, None, 0, C.byref(n), C.byref(lo)))
        buf = np.zeros(2 * n.value)
        _check(lib().ref_effective_kernel(self._h, _p(buf), n.value, C.byref(n), C.byref(lo)))
        return buf[0::2] + 1j * buf[1::2], lo.value

    def __del__(self):
        if getattr(self, "_h", None) and getattr(self, "_free", None):
            self._free(self._h)
            self._h = None


def apply_transform(spec: Spec, x, boundary: int = 1, workers: int = 1) -> np.ndarray:
    """``sft::apply_transform`` (proj/src/transforms.cpp:444-459): complex128[n]."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    out = np.zeros(2 * x.size)
    _check(lib().ref_apply_transform(spec._h, _p(x), x.size, boundary, workers, _p(out)))
    return out[0::2] + 1j * out[1::2]


def components(x, boundary, K, beta, p=0, omega=None, alpha=0.0, strategy=RECURSIVE2, precision=DOUBLE,
               window_2k1=False, lo=0, hi=None, sliding_route=False):
    """``sft::components_over`` or, with ``sliding_route``, ``sft::sft_via_sliding_sum``
    (proj/src/engine.cpp:255-337): (c, s)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if hi is None:
        hi = x.size - 1
    if sliding_route:
        lo, hi = 0, x.size - 1
    n = hi - lo + 1
    c, s = np.zeros(n), np.zeros(n)
    _check(lib().ref_components(_p(x), x.size, boundary, K, beta, int(omega is None), p, float(omega or 0.0), alpha,
                                strategy, precision, int(window_2k1), lo, hi, int(sliding_route), _p(c), _p(s)))
    return c, s


def make_test_signal(kind: int, n: int, seed: int) -> np.ndarray:
    out = np.zeros(n)
    _check(lib().ref_make_test_signal(kind, n, seed, _p(out)))
    return out


def sliding_sum_flat_i64(f, window: int) -> np.ndarray:
    f = np.ascontiguousarray(np.asarray(f, dtype=np.int64))
    out = np.zeros(f.size - window + 1, dtype=np.int64)
    _check(lib().ref_sliding_sum_flat_i64(_p(f), f.size, window, _p(out)))
    return out
