"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the SFT/ASFT hot path.

ctypes wrapper over ``oracle/_build/liboracle.so`` (built from ``oracle/sft_oracle.cpp``,
a plain-C++ restatement of the reference library at /root/reference/proj; see the
header of that file for the file:line map). Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package, and only as the checker or the timed CPU baseline. The product package
``paper_2110_11866_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

ZERO, CLAMP = 0, 1
KERNEL_INTEGRAL, RECURSIVE1, RECURSIVE2 = 0, 1, 2
SINGLE, DOUBLE = 0, 1
IMPULSE, CONSTANT, CHIRP, SEEDED_NOISE = 0, 1, 2, 3


def build() -> str:
    """The restated oracle, and the reference compiled from its own sources (oracle/ref.mk)
    where those sources exist (elsewhere the prebuilt oracle/_ref is used)."""
    subprocess.check_call(["make", "-s", "-C", _HERE])
    from . import ref

    if ref.source_available():
        ref.build()
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "sft_oracle.cpp")
        ):
            build()
        L = C.CDLL(_LIB_PATH)
        d, i, i64, u64 = C.c_double, C.c_int, C.c_int64, C.c_uint64
        P = C.c_void_p
        L.orc_last_error.restype = C.c_char_p
        L.orc_make_test_signal.argtypes = [i, i64, u64, P]
        L.orc_components.argtypes = [P, i64, i, i, d, i, i, d, d, i, i, i, i64, i64, i, P, P, P]
        L.orc_sft_via_sliding_sum.argtypes = [P, i64, i, i, d, i, i, d, d, i, i, P, P]
        L.orc_sliding_window_state.argtypes = [P, i64, i, i, d, i, P, P, P, P]
        L.orc_stability_probe.argtypes = [P, i64, i, i, d, i, d, i, P, P, P, P]
        L.orc_sliding_sum_i64.argtypes = [P, i64, i64, i, i, P, P, P]
        L.orc_sliding_sum_f64.argtypes = [P, i64, i64, i, i, P]
        L.orc_sliding_plan.argtypes = [i64, i64, i, P, P, P, P, P]
        L.orc_truncated_convolution.argtypes = [P, i64, i, P, P, i64, i64, i, P, P]
        L.orc_gauss_smooth.argtypes = [P, i64, i, i, i, d, i, d, d, i, i, i, P, P, P, i, P]
        L.orc_morlet_direct.argtypes = [P, i64, i, i, d, i, d, d, i, i, i, P, P, i, P, P, i, P]
        L.orc_morlet_multiply.argtypes = [P, i64, i, i, d, i, d, d, d, i, i, i, P, i, P]
        for f in ("orc_gauss", "orc_gauss_d", "orc_gauss_dd"):
            getattr(L, f).argtypes = [d, d]
            getattr(L, f).restype = d
        L.orc_morlet.argtypes = [d, d, d, P, P]
        L.orc_series_taps.argtypes = [i, d, i, P, P, i, P, P, i, d, P, P, P]
        L.orc_multiply_taps.argtypes = [i, d, i, P, d, d, i, P, P, P]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


class OracleInvalidArgument(ValueError):
    pass


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 2:
        raise OracleInvalidArgument(msg)
    raise OracleError(msg)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def make_test_signal(kind: int, n: int, seed: int) -> np.ndarray:
    out = np.empty(max(n, 1), dtype=np.float64)
    _check(lib().orc_make_test_signal(kind, n, seed, _p(out)))
    return out


@dataclass
class Cfg:
    """SftConfig (proj/include/sft/engine.hpp:41-60)."""

    K: int
    beta: float
    p: int = 0
    omega: float | None = None  # real-frequency order when set
    alpha: float = 0.0
    strategy: int = RECURSIVE2
    precision: int = DOUBLE
    window_2k1: bool = False


def components_over(x, boundary: int, cfg: Cfg, lo: int, hi: int, mode: int = 0, want_state=False):
    x = _f64(x)
    n = hi - lo + 1
    c = np.zeros(max(n, 1))
    s = np.zeros(max(n, 1))
    ms = np.zeros(1)
    io = 0 if cfg.omega is not None else 1
    _check(
        lib().orc_components(
            _p(x), x.size, boundary, cfg.K, cfg.beta, io, cfg.p,
            float(cfg.omega or 0.0), cfg.alpha, cfg.strategy, cfg.precision,
            int(cfg.window_2k1), lo, hi, mode, _p(c), _p(s), _p(ms) if want_state else None,
        )
    )
    if want_state:
        return c, s, float(ms[0])
    return c, s


def sft_components(x, boundary, cfg):
    return components_over(x, boundary, cfg, 0, len(x) - 1, mode=1)


def asft_components(x, boundary, cfg):
    return components_over(x, boundary, cfg, 0, len(x) - 1, mode=2)


def sft_via_sliding_sum(x, boundary, cfg: Cfg, workers: int = 1):
    x = _f64(x)
    c = np.zeros(x.size)
    s = np.zeros(x.size)
    io = 0 if cfg.omega is not None else 1
    _check(
        lib().orc_sft_via_sliding_sum(
            _p(x), x.size, boundary, cfg.K, cfg.beta, io, cfg.p, float(cfg.omega or 0.0),
            cfg.alpha, cfg.precision, workers, _p(c), _p(s),
        )
    )
    return c, s


def sliding_window_state(x, boundary, K, beta, p):
    x = _f64(x)
    a, b, cc, d = (np.zeros(x.size) for _ in range(4))
    _check(lib().orc_sliding_window_state(_p(x), x.size, boundary, K, beta, p, _p(a), _p(b), _p(cc), _p(d)))
    return a + 1j * b, cc + 1j * d


def stability_probe(x, boundary, K, beta, p, alpha, strategy):
    x = _f64(x)
    ms, me, rs = np.zeros(1), np.zeros(1), np.zeros(1)
    ae = np.zeros(x.size)
    _check(lib().orc_stability_probe(_p(x), x.size, boundary, K, beta, p, alpha, strategy, _p(ms), _p(me), _p(rs), _p(ae)))
    return dict(max_state_magnitude=ms[0], max_component_error=me[0], reference_scale=rs[0], abs_error=ae)


def sliding_sum(f, L: int, blocked: bool = False, workers: int = 1, trace: bool = False):
    f = np.asarray(f)
    n = f.size
    if f.dtype == np.int64:
        f = np.ascontiguousarray(f)
        out = np.zeros(max(n - L + 1, 1), dtype=np.int64)
        tr = np.zeros(6 * 256, dtype=np.int64)
        nr = C.c_int(0)
        _check(lib().orc_sliding_sum_i64(_p(f), n, L, int(blocked), workers, _p(out), _p(tr), C.byref(nr)))
        if trace:
            return out, tr[: 6 * nr.value].reshape(-1, 6)
        return out
    f = _f64(f)
    out = np.zeros(max(n - L + 1, 1))
    _check(lib().orc_sliding_sum_f64(_p(f), n, L, int(blocked), workers, _p(out)))
    return out


def sliding_plan(n: int, L: int, blocked: bool = False) -> dict:
    vals = [C.c_int64(0) for _ in range(5)]
    _check(lib().orc_sliding_plan(n, L, int(blocked), *[C.byref(v) for v in vals]))
    keys = ("rounds", "padded_size", "blocked_stages", "parallel_steps", "total_adds")
    return {k: v.value for k, v in zip(keys, vals)}


def truncated_convolution(x, boundary: int, taps, tap_lo: int, workers: int = 1) -> np.ndarray:
    x = _f64(x)
    taps = np.asarray(taps, dtype=np.complex128)
    tr, ti = _f64(taps.real), _f64(taps.imag)
    ore, oim = np.zeros(x.size), np.zeros(x.size)
    _check(lib().orc_truncated_convolution(_p(x), x.size, boundary, _p(tr), _p(ti), taps.size, tap_lo, workers, _p(ore), _p(oim)))
    return ore + 1j * oim


def gauss_smooth(x, boundary, kind, K, beta, n0, alpha, gamma, strategy, precision, a, b, d, workers=1):
    x = _f64(x)
    a, b, d = _f64(a), _f64(b), _f64(d)
    P = a.size - 1
    out = np.zeros(x.size)
    _check(lib().orc_gauss_smooth(_p(x), x.size, boundary, kind, K, beta, n0, alpha, gamma, strategy, precision, P, _p(a), _p(b), _p(d), workers, _p(out)))
    return out


def morlet_direct(x, boundary, K, beta, n0, alpha, gamma, strategy, precision, cos_orders, cos_coeffs, sin_orders, sin_coeffs, workers=1):
    x = _f64(x)
    co = np.ascontiguousarray(cos_orders, dtype=np.int32)
    so = np.ascontiguousarray(sin_orders, dtype=np.int32)
    cc = _f64(np.column_stack([np.real(cos_coeffs), np.imag(cos_coeffs)]).ravel()) if len(co) else np.zeros(2)
    sc = _f64(np.column_stack([np.real(sin_coeffs), np.imag(sin_coeffs)]).ravel()) if len(so) else np.zeros(2)
    out = np.zeros(2 * x.size)
    _check(lib().orc_morlet_direct(_p(x), x.size, boundary, K, beta, n0, alpha, gamma, strategy, precision, co.size, _p(co), _p(cc), so.size, _p(so), _p(sc), workers, _p(out)))
    return out[0::2] + 1j * out[1::2]


def morlet_multiply(x, boundary, K, beta, n0, alpha, sigma, xi, strategy, precision, env, workers=1):
    x = _f64(x)
    env = _f64(env)
    out = np.zeros(2 * x.size)
    _check(lib().orc_morlet_multiply(_p(x), x.size, boundary, K, beta, n0, alpha, sigma, xi, strategy, precision, env.size - 1, _p(env), workers, _p(out)))
    return out[0::2] + 1j * out[1::2]


def gauss(sigma, t):
    return lib().orc_gauss(sigma, t)


def gauss_d(sigma, t):
    return lib().orc_gauss_d(sigma, t)


def gauss_dd(sigma, t):
    return lib().orc_gauss_dd(sigma, t)


def morlet(sigma, xi, t):
    re, im = C.c_double(0), C.c_double(0)
    lib().orc_morlet(sigma, xi, t, C.byref(re), C.byref(im))
    return complex(re.value, im.value)


def series_taps(K, beta, cos_orders, cos_coeffs, sin_orders, sin_coeffs, n0, gamma):
    co = np.ascontiguousarray(cos_orders, dtype=np.int32)
    so = np.ascontiguousarray(sin_orders, dtype=np.int32)
    cc = _f64(np.column_stack([np.real(cos_coeffs), np.imag(cos_coeffs)]).ravel()) if len(co) else np.zeros(2)
    sc = _f64(np.column_stack([np.real(sin_coeffs), np.imag(sin_coeffs)]).ravel()) if len(so) else np.zeros(2)
    tr, ti = np.zeros(2 * K + 1), np.zeros(2 * K + 1)
    lo = C.c_int64(0)
    _check(lib().orc_series_taps(K, beta, co.size, _p(co), _p(cc), so.size, _p(so), _p(sc), n0, gamma, _p(tr), _p(ti), C.byref(lo)))
    return tr + 1j * ti, lo.value


def multiply_taps(K, beta, env, sigma, xi, n0):
    env = _f64(env)
    tr, ti = np.zeros(2 * K + 1), np.zeros(2 * K + 1)
    lo = C.c_int64(0)
    _check(lib().orc_multiply_taps(K, beta, env.size - 1, _p(env), sigma, xi, n0, _p(tr), _p(ti), C.byref(lo)))
    return tr + 1j * ti, lo.value
