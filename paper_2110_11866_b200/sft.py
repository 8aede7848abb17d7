"""Python mirror of the reference library's public API for the SFT/ASFT path
(namespace ``sft`` in /root/reference/proj/include/sft/*.hpp), executed on the B200
through libsftgpu's C ABI.

Same names, argument meaning and error behaviour as the reference:
``std::invalid_argument`` -> ``ValueError``, ``FitDegenerateError`` ->
``FitDegenerateError``; results are host arrays (``numpy``) like the reference's
Eigen arrays. Device execution uses torch only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import FitDegenerateError, SftGpuError, check, lib

__all__ = [
    "BoundaryPolicy", "Precision", "Strategy", "TransformKind", "GaussKind", "TestSignalKind",
    "Signal", "make_test_signal", "generate_signals", "OrderSpec", "SftConfig", "components_replay", "ComponentSeq", "TransformOptions",
    "TransformSpec", "TransformResult", "KernelTaps", "AbbrevInfo", "GaussianFitBundle",
    "CoefficientSet", "parse_abbreviation", "encode_abbreviation", "make_transform_spec",
    "make_gauss_spec", "make_morlet_direct_spec", "make_morlet_multiply_spec", "gauss_smooth",
    "morlet_direct_transform", "morlet_multiply_transform", "truncated_reference", "apply_transform",
    "effective_kernel", "components_over", "sft_components", "asft_components", "sft_via_sliding_sum",
    "truncated_convolution", "fit_gaussian_bundle", "fit_morlet_direct", "fit_morlet_envelope",
    "fit_mmse", "select_optimal_ps", "tune_beta_gauss", "gauss_kernel_rmse",
    "morlet_direct_kernel_rmse", "morlet_multiply_kernel_rmse", "TransformPlan", "MultiScalePlan", "ComponentsPlan",
    "reconstruct", "tune_beta", "WindowState", "sliding_window_state", "StabilityReport", "stability_probe",
    "CostReport", "cost_model", "MethodOpCounts", "sft_method_counts", "conv_method_counts",
    "FitDegenerateError", "SftGpuError", "write_coefficient_sets", "read_coefficient_sets",
    "morlet_direct_spec_from_coeffs", "sliding_sum_plan", "sliding_sum_flat", "sliding_sum_blocked8",
]


class BoundaryPolicy(enum.IntEnum):  # include/sft/signal.hpp:12
    Zero = 0
    Clamp = 1


class Precision(enum.IntEnum):  # include/sft/signal.hpp:15
    Single = 0
    Double = 1


class Strategy(enum.IntEnum):  # include/sft/engine.hpp:16
    KernelIntegral = 0
    Recursive1 = 1
    Recursive2 = 2


class TransformKind(enum.IntEnum):  # include/sft/transforms.hpp:11-19
    Gauss = 0
    GaussD = 1
    GaussDD = 2
    MorletDirect = 3
    MorletMultiply = 4
    TruncConvGauss = 5
    TruncConvMorlet = 6


class GaussKind(enum.IntEnum):  # include/sft/fourier_fit.hpp:101
    Value = 0
    Deriv1 = 1
    Deriv2 = 2


class TestSignalKind(enum.IntEnum):  # include/sft/signal.hpp:47
    Impulse = 0
    Constant = 1
    Chirp = 2
    SeededNoise = 3


# ------------------------------------------------------------------ signal
class Signal:
    """Finite real sample sequence + boundary policy (include/sft/signal.hpp:19-32)."""

    def __init__(self, samples, boundary: BoundaryPolicy = BoundaryPolicy.Clamp):
        arr = np.ascontiguousarray(np.asarray(samples, dtype=np.float64))
        if arr.ndim != 1 or arr.size < 1:
            raise ValueError("Signal: need at least one sample")
        if not np.all(np.isfinite(arr)):
            raise ValueError("Signal: samples must be finite")
        self.samples = arr
        self.boundary = BoundaryPolicy(boundary)

    def size(self) -> int:
        return int(self.samples.size)

    def __len__(self) -> int:
        return self.size()


_TORCH = None


def _torch():
    """torch, once a CUDA device is known to exist (checked once: torch.cuda.is_available()
    queries the driver and costs microseconds on the streaming path)."""
    global _TORCH
    if _TORCH is None:
        import torch

        if not torch.cuda.is_available():
            raise SftGpuError("no CUDA device available (libsftgpu has no CPU fallback)")
        _TORCH = torch
    return _TORCH


def _stream_ptr(torch):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def make_test_signal(kind: TestSignalKind, n: int, seed: int, boundary=BoundaryPolicy.Clamp) -> Signal:
    """Deterministic generators (proj/src/signal.cpp:24-51), generated on the device
    by the splitmix64 kernel (K2) and copied back; noise is bit-identical."""
    if n < 1:
        raise ValueError("make_test_signal: N must be >= 1")
    torch = _torch()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    check(lib().sftgpu_generate_signal(int(kind), n, seed, 1, 1, C.c_void_p(out.data_ptr()), _stream_ptr(torch)))
    return Signal(out.cpu().numpy(), boundary)


def generate_signals(kind: TestSignalKind, n: int, seed: int, batch: int = 1, precision=Precision.Single):
    """Device batch generator: [batch][n] tensor, signal i seeded with seed+i."""
    torch = _torch()
    dt = torch.float32 if precision == Precision.Single else torch.float64
    out = torch.empty((batch, n), dtype=dt, device="cuda")
    check(lib().sftgpu_generate_signal(int(kind), n, seed, batch, int(precision), C.c_void_p(out.data_ptr()), _stream_ptr(torch)))
    return out


# ------------------------------------------------------------------ engine types
@dataclass
class OrderSpec:  # include/sft/engine.hpp:18-39
    integer_order: bool = True
    p: int = 0
    omega: float = 0.0

    @staticmethod
    def order(p: int) -> "OrderSpec":
        if p < 0:
            raise ValueError("OrderSpec: p must be >= 0")
        return OrderSpec(True, p, 0.0)

    @staticmethod
    def frequency(omega: float) -> "OrderSpec":
        return OrderSpec(False, 0, float(omega))

    def angular(self, beta: float) -> float:
        return beta * self.p if self.integer_order else self.omega


@dataclass
class SftConfig:  # include/sft/engine.hpp:41-60
    half_width: int
    beta: float
    order: OrderSpec = field(default_factory=OrderSpec)
    alpha: float = 0.0
    n0: int = 0
    strategy: Strategy = Strategy.Recursive2
    precision: Precision = Precision.Double
    window_2k1: bool = False

    def _c(self) -> _abi.Config:
        return _abi.Config(
            self.half_width, self.beta, int(self.order.integer_order), self.order.p, self.order.omega,
            self.alpha, self.n0, int(self.strategy), int(self.precision), int(self.window_2k1),
        )


@dataclass
class ComponentSeq:  # include/sft/engine.hpp:65-68
    c: np.ndarray
    s: np.ndarray


class ComponentsPlan:
    """Device plan for component sequences of several orders sharing K/alpha/precision:
    c, s are [n_orders][batch][hi-lo+1]."""

    def __init__(self, cfgs, n: int, batch: int, boundary, lo: int, hi: int, mode: int = 0):
        arr = (_abi.Config * len(cfgs))(*[c._c() for c in cfgs])
        h = C.c_void_p()
        check(lib().sftgpu_components_plan_create(arr, len(cfgs), n, batch, int(boundary), lo, hi, mode, C.byref(h)))
        self._h = h
        self._destroy = lib().sftgpu_plan_destroy
        self.n_orders, self.n, self.batch, self.count = len(cfgs), n, batch, hi - lo + 1
        self.precision = Precision(cfgs[0].precision)
        self.device = _torch().cuda.current_device()

    def execute(self, x, c, s, stream=None):
        torch = _torch()
        dt = torch.float32 if self.precision == Precision.Single else torch.float64
        _check_device_buffer(x, dt, self.batch * self.n, self.device, "x")
        for name, t in (("c", c), ("s", s)):
            _check_device_buffer(t, dt, self.n_orders * self.batch * self.count, self.device, name)
        st = C.c_void_p(stream) if stream is not None else _stream_ptr(torch)
        check(lib().sftgpu_components_execute(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(c.data_ptr()), C.c_void_p(s.data_ptr()), st))

    def __del__(self):
        # the destroy entry point is bound at creation: module globals may already be
        # torn down when this runs at interpreter exit
        if getattr(self, "_h", None) and getattr(self, "_destroy", None):
            self._destroy(self._h)
            self._h = None


def _components(sig: Signal, cfgs, lo: int, hi: int, mode: int):
    torch = _torch()
    plan = ComponentsPlan(cfgs, sig.size(), 1, sig.boundary, lo, hi, mode)
    dt = torch.float32 if plan.precision == Precision.Single else torch.float64
    x = torch.from_numpy(sig.samples).to(device="cuda", dtype=dt)
    c = torch.empty((len(cfgs), plan.count), dtype=dt, device="cuda")
    s = torch.empty_like(c)
    plan.execute(x, c, s)
    torch.cuda.synchronize()
    return c.double().cpu().numpy(), s.double().cpu().numpy()


def components_replay(sig: Signal, cfgs, lo: int, hi: int, want_state: bool = False):
    """proj/src/engine.cpp:53-120 (recursive_components): Recursive1 / Recursive2 replayed on
    the GPU with the reference's own operation order (K7, ``sftgpu_components_replay``), so
    the result is bit-identical to the reference's. (c, s) as [n_cfgs][hi - lo + 1], plus
    the per-config peak |filter state| (engine.cpp:101) with ``want_state``."""
    cfgs = list(cfgs)
    n = sig.size()
    count = hi - lo + 1 if hi >= lo else 0
    x = np.ascontiguousarray(sig.samples, dtype=np.float64)
    c = np.empty((len(cfgs), max(count, 1)), dtype=np.float64)
    s = np.empty_like(c)
    arr = (_abi.Config * len(cfgs))(*[cf._c() for cf in cfgs])
    peak = np.zeros(len(cfgs), dtype=np.float64)
    check(lib().sftgpu_components_replay(arr, len(cfgs), x.ctypes.data_as(C.c_void_p), n, int(sig.boundary), lo, hi,
                                         c.ctypes.data_as(C.c_void_p), s.ctypes.data_as(C.c_void_p),
                                         peak.ctypes.data_as(C.c_void_p)))
    return (c, s, peak) if want_state else (c, s)


def _one(sig: Signal, cfg: SftConfig, lo: int, hi: int, mode: int, exact: bool) -> ComponentSeq:
    # Recursive strategies replay the reference's recurrence (bit-identical) unless the
    # caller asks for the window-recurrence scan (K1, faster and more accurate)
    if exact and cfg.strategy != Strategy.KernelIntegral and cfg.order.integer_order:
        if mode == 1 and cfg.alpha != 0.0:
            raise ValueError("sft_components: alpha must be 0 (use asft_components)")
        if mode == 2 and not cfg.alpha > 0.0:
            raise ValueError("asft_components: alpha must be > 0")
        c, s = components_replay(sig, [cfg], lo, hi)
    else:
        c, s = _components(sig, [cfg], lo, hi, mode)
    return ComponentSeq(c[0], s[0])


def components_over(sig: Signal, cfg: SftConfig, lo: int, hi: int, exact: bool = True) -> ComponentSeq:
    """proj/src/engine.cpp:255-258 (signed output range, boundary-extended reads).
    Recursive1/2 configs run the reference's recurrence on the GPU (K7, bit-identical);
    ``exact=False`` runs every strategy on the window-recurrence scan (K1)."""
    return _one(sig, cfg, lo, hi, 0, exact)


def sft_components(sig: Signal, cfg: SftConfig, exact: bool = True) -> ComponentSeq:
    """proj/src/engine.cpp:260-264 (requires alpha == 0)."""
    return _one(sig, cfg, 0, sig.size() - 1, 1, exact)


def asft_components(sig: Signal, cfg: SftConfig, exact: bool = True) -> ComponentSeq:
    """proj/src/engine.cpp:266-269 (requires alpha > 0)."""
    return _one(sig, cfg, 0, sig.size() - 1, 2, exact)


def sft_via_sliding_sum(sig: Signal, cfg: SftConfig, workers: int = 1) -> ComponentSeq:
    """proj/src/engine.cpp:183-219, 323-337: the kernel-integral components by the
    reference's sliding-sum route, on the GPU (``sftgpu_sft_via_sliding_sum``): the
    rebased attenuated phased sequence, the K5 flat window sums (paper Algorithm 1,
    complex128), rescale and phase removal. ``workers`` is accepted for API parity."""
    n = sig.size()
    x = np.ascontiguousarray(sig.samples, dtype=np.float64)
    c = np.empty(n, dtype=np.float64)
    s = np.empty(n, dtype=np.float64)
    raw = cfg._c()
    check(lib().sftgpu_sft_via_sliding_sum(C.byref(raw), x.ctypes.data_as(C.c_void_p), n, int(sig.boundary),
                                           c.ctypes.data_as(C.c_void_p), s.ctypes.data_as(C.c_void_p)))
    return ComponentSeq(c, s)


# ------------------------------------------------------------------ fits / specs
@dataclass
class CoefficientSet:  # include/sft/fourier_fit.hpp:56-68
    kind: int
    half_width: int
    beta: float
    cos_orders: list
    sin_orders: list
    cos_coeffs: np.ndarray
    sin_coeffs: np.ndarray
    fit_rmse_percent: float
    sigma: float = 0.0
    xi: float = 0.0
    n0: int = 0

    @staticmethod
    def _from(c: _abi.Coeffs) -> "CoefficientSet":
        cc = np.array(c.cos_coeffs[: 2 * c.n_cos]).reshape(-1, 2) if c.n_cos else np.zeros((0, 2))
        sc = np.array(c.sin_coeffs[: 2 * c.n_sin]).reshape(-1, 2) if c.n_sin else np.zeros((0, 2))
        return CoefficientSet(
            c.kind, c.half_width, c.beta, list(c.cos_orders[: c.n_cos]), list(c.sin_orders[: c.n_sin]),
            cc[:, 0] + 1j * cc[:, 1], sc[:, 0] + 1j * sc[:, 1], c.fit_rmse_percent, c.sigma, c.xi, c.n0,
        )

    def _c(self) -> _abi.Coeffs:
        c = _abi.Coeffs()
        c.kind, c.half_width, c.beta = int(self.kind), int(self.half_width), float(self.beta)
        c.n_cos, c.n_sin = len(self.cos_orders), len(self.sin_orders)
        for i, p in enumerate(self.cos_orders):
            c.cos_orders[i] = int(p)
            c.cos_coeffs[2 * i], c.cos_coeffs[2 * i + 1] = float(np.real(self.cos_coeffs[i])), float(np.imag(self.cos_coeffs[i]))
        for i, p in enumerate(self.sin_orders):
            c.sin_orders[i] = int(p)
            c.sin_coeffs[2 * i], c.sin_coeffs[2 * i + 1] = float(np.real(self.sin_coeffs[i])), float(np.imag(self.sin_coeffs[i]))
        c.fit_rmse_percent, c.sigma, c.xi, c.n0 = float(self.fit_rmse_percent), float(self.sigma), float(self.xi), int(self.n0)
        return c


@dataclass
class GaussianFitBundle:  # include/sft/fourier_fit.hpp:88-99
    sigma: float
    half_width: int
    beta: float
    max_order: int
    a: np.ndarray
    b: np.ndarray
    d: np.ndarray
    fit_rmse_g: float
    fit_rmse_gd: float
    fit_rmse_gdd: float

    @staticmethod
    def _from(b: _abi.GaussBundle) -> "GaussianFitBundle":
        P = b.max_order
        return GaussianFitBundle(
            b.sigma, b.half_width, b.beta, P, np.array(b.a[: P + 1]), np.array(b.b[:P]), np.array(b.d[: P + 1]),
            b.fit_rmse_g, b.fit_rmse_gd, b.fit_rmse_gdd,
        )


@dataclass
class TransformOptions:  # include/sft/transforms.hpp:43-50
    half_width: int | None = None
    beta: float | None = None
    tune_beta: bool = False
    ps: int | None = None
    strategy: Strategy = Strategy.Recursive2
    precision: Precision = Precision.Double

    def _c(self) -> _abi.Options:
        return _abi.Options(
            int(self.half_width is not None), self.half_width or 0, int(self.beta is not None), self.beta or 0.0,
            int(self.tune_beta), int(self.ps is not None), self.ps or 0, int(self.strategy), int(self.precision),
        )


@dataclass
class AbbrevInfo:
    kind: TransformKind
    n0: int = 0
    order: int = 0


class TransformSpec:
    """Fully resolved transform (include/sft/transforms.hpp:23-41), backed by the
    C ``sftgpu_spec``; fields are readable and the engine knobs writable."""

    def __init__(self, raw: _abi.Spec):
        self._raw = raw

    kind = property(lambda s: TransformKind(s._raw.kind))
    sigma = property(lambda s: s._raw.sigma)
    xi = property(lambda s: s._raw.xi)
    half_width = property(lambda s: s._raw.half_width)
    max_order = property(lambda s: s._raw.max_order)
    ps = property(lambda s: s._raw.ps)
    pd = property(lambda s: s._raw.pd)
    beta = property(lambda s: s._raw.beta)
    abbreviation = property(lambda s: s._raw.abbreviation.decode())
    kernel_rmse_percent = property(lambda s: s._raw.kernel_rmse_percent)

    def _rw(name):  # noqa: N805
        return property(lambda s: getattr(s._raw, name), lambda s, v: setattr(s._raw, name, v))

    n0 = _rw("n0")
    alpha = _rw("alpha")
    strategy = property(lambda s: Strategy(s._raw.strategy), lambda s, v: setattr(s._raw, "strategy", int(v)))
    precision = property(lambda s: Precision(s._raw.precision), lambda s, v: setattr(s._raw, "precision", int(v)))

    @property
    def gauss_coeffs(self):
        return GaussianFitBundle._from(self._raw.gauss) if self.kind <= TransformKind.GaussDD else None

    @property
    def morlet_coeffs(self):
        return CoefficientSet._from(self._raw.morlet) if self.kind == TransformKind.MorletDirect else None

    @property
    def envelope_coeffs(self):
        return CoefficientSet._from(self._raw.envelope) if self.kind == TransformKind.MorletMultiply else None

    def copy(self) -> "TransformSpec":
        raw = _abi.Spec()
        C.pointer(raw)[0] = self._raw
        return TransformSpec(raw)


def parse_abbreviation(abbrev: str) -> AbbrevInfo:
    k, n0, o = C.c_int(), C.c_int(), C.c_int()
    check(lib().sftgpu_parse_abbreviation(abbrev.encode(), C.byref(k), C.byref(n0), C.byref(o)))
    return AbbrevInfo(TransformKind(k.value), n0.value, o.value)


def encode_abbreviation(kind: TransformKind, n0: int, order: int) -> str:
    buf = C.create_string_buffer(32)
    check(lib().sftgpu_encode_abbreviation(int(kind), n0, order, buf, 32))
    return buf.value.decode()


def _opts(options):
    return (options or TransformOptions())._c()


def make_transform_spec(abbrev: str, sigma: float, xi: float, options: TransformOptions | None = None) -> TransformSpec:
    raw = _abi.Spec()
    o = _opts(options)
    check(lib().sftgpu_make_transform_spec(abbrev.encode(), sigma, xi, C.byref(o), C.byref(raw)))
    return TransformSpec(raw)


def make_gauss_spec(sigma, kind: GaussKind, max_order: int, n0: int, options=None) -> TransformSpec:
    raw = _abi.Spec()
    o = _opts(options)
    check(lib().sftgpu_make_gauss_spec(sigma, int(kind), max_order, n0, C.byref(o), C.byref(raw)))
    return TransformSpec(raw)


def make_morlet_direct_spec(sigma, xi, pd: int, n0: int, options=None) -> TransformSpec:
    raw = _abi.Spec()
    o = _opts(options)
    check(lib().sftgpu_make_morlet_direct_spec(sigma, xi, pd, n0, C.byref(o), C.byref(raw)))
    return TransformSpec(raw)


def make_morlet_multiply_spec(sigma, xi, pm: int, n0: int, options=None) -> TransformSpec:
    raw = _abi.Spec()
    o = _opts(options)
    check(lib().sftgpu_make_morlet_multiply_spec(sigma, xi, pm, n0, C.byref(o), C.byref(raw)))
    return TransformSpec(raw)


def write_coefficient_sets(path: str, sets) -> None:
    """"sft-coefficients v1" file (proj/src/coeff_io.cpp:21-42); ``sets`` are
    TransformSpec (their fitted set) or raw ``_abi.Coeffs``."""
    raws = []
    for s_ in sets:
        if isinstance(s_, TransformSpec):
            k = s_.kind
            raws.append(s_._raw.morlet if k == TransformKind.MorletDirect else s_._raw.envelope)
        else:
            raws.append(s_)
    arr = (_abi.Coeffs * max(1, len(raws)))(*raws)
    check(lib().sftgpu_write_coefficient_sets(path.encode(), arr, len(raws)))


def read_coefficient_sets(path: str):
    """Raw coefficient sets from an "sft-coefficients v1" file (coeff_io.cpp:44-101)."""
    n = C.c_int()
    check(lib().sftgpu_read_coefficient_sets(path.encode(), None, 0, C.byref(n)))
    arr = (_abi.Coeffs * max(1, n.value))()
    check(lib().sftgpu_read_coefficient_sets(path.encode(), arr, n.value, C.byref(n)))
    return [arr[i] for i in range(n.value)]


def morlet_direct_spec_from_coeffs(raw: "_abi.Coeffs", precision=Precision.Double, strategy=Strategy.Recursive2,
                                   recompute_rmse: bool = True) -> TransformSpec:
    """A MorletDirect spec from a stored coefficient set (proj/src/cli.cpp:224-280)."""
    spec = _abi.Spec()
    check(lib().sftgpu_make_morlet_direct_spec_from_coeffs(C.byref(raw), int(precision), int(strategy),
                                                           int(recompute_rmse), C.byref(spec)))
    return TransformSpec(spec)


def sliding_sum_plan(n: int, window: int, blocked: bool = False) -> dict:
    """SlidingSumPlan::make + cost_model (proj/include/sft/sliding_sum.hpp:32-60,
    proj/src/sliding_sum.cpp:7-40)."""
    info = (C.c_int64 * 5)()
    check(lib().sftgpu_sliding_sum_plan(n, window, int(blocked), info))
    keys = ("rounds", "padded_size", "blocked_stages", "parallel_steps", "total_adds")
    return dict(zip(keys, list(info)))


def _sliding(f, window: int, blocked: bool):
    torch = _torch()
    a = np.ascontiguousarray(np.asarray(f))
    if a.dtype == np.int64:
        dt, code = torch.int64, 0
    elif np.iscomplexobj(a):
        a = a.astype(np.complex128)
        dt, code = torch.complex128, 2
    else:
        a = a.astype(np.float64)
        dt, code = torch.float64, 1
    n = a.size
    x = torch.from_numpy(a).to("cuda")
    out = torch.empty(max(1, n - window + 1), dtype=dt, device="cuda")
    check(lib().sftgpu_sliding_sum(code, int(blocked), C.c_void_p(x.data_ptr()), n, window,
                                   C.c_void_p(out.data_ptr()), _stream_ptr(torch)))
    return out.cpu().numpy()


def sliding_sum_flat(f, window: int, workers: int = 1):
    """Algorithm 1 on the GPU (proj/include/sft/sliding_sum.hpp:89-121): h[n] = sum_{k<L} f[n+k],
    same addition tree as the reference (bit-identical for int64 / float64)."""
    return _sliding(f, window, False)


def sliding_sum_blocked8(f, window: int, workers: int = 1):
    """Algorithms 2-3 on the GPU ((16,8) shared-memory tiles, proj/include/sft/sliding_sum.hpp:144-234)."""
    return _sliding(f, window, True)


@dataclass
class KernelTaps:  # include/sft/kernels.hpp:76-81
    taps: np.ndarray
    lo: int

    def hi(self) -> int:
        return self.lo + self.taps.size - 1


def effective_kernel(spec: TransformSpec) -> KernelTaps:
    n, lo = C.c_int64(), C.c_int64()
    check(lib().sftgpu_effective_kernel(C.byref(spec._raw), None, 0, C.byref(n), C.byref(lo)))
    buf = np.zeros(2 * n.value)
    check(lib().sftgpu_effective_kernel(C.byref(spec._raw), buf.ctypes.data_as(C.c_void_p), n.value, C.byref(n), C.byref(lo)))
    return KernelTaps(buf[0::2] + 1j * buf[1::2], lo.value)


def fit_gaussian_bundle(sigma: float, half_width: int, max_order: int, beta: float) -> GaussianFitBundle:
    b = _abi.GaussBundle()
    check(lib().sftgpu_fit_gaussian_bundle(sigma, half_width, max_order, beta, C.byref(b)))
    return GaussianFitBundle._from(b)


def fit_morlet_direct(sigma, xi, half_width, ps, pd, beta, n0=0) -> CoefficientSet:
    c = _abi.Coeffs()
    check(lib().sftgpu_fit_morlet_direct(sigma, xi, half_width, ps, pd, beta, n0, C.byref(c)))
    return CoefficientSet._from(c)


def fit_morlet_envelope(sigma, xi, half_width, max_order, beta) -> CoefficientSet:
    c = _abi.Coeffs()
    check(lib().sftgpu_fit_morlet_envelope(sigma, xi, half_width, max_order, beta, C.byref(c)))
    return CoefficientSet._from(c)


def fit_mmse(target, half_width: int, beta: float, cos_orders, sin_orders, kind: int = 0) -> CoefficientSet:
    t = np.asarray(target, dtype=np.complex128)
    buf = np.ascontiguousarray(np.column_stack([t.real, t.imag]).ravel())
    co = np.ascontiguousarray(cos_orders, dtype=np.int32)
    so = np.ascontiguousarray(sin_orders, dtype=np.int32)
    c = _abi.Coeffs()
    check(lib().sftgpu_fit_mmse(buf.ctypes.data_as(C.c_void_p), half_width, beta, co.size, co.ctypes.data_as(C.c_void_p),
                                so.size, so.ctypes.data_as(C.c_void_p), kind, C.byref(c)))
    return CoefficientSet._from(c)


def reconstruct(coeffs: CoefficientSet, points) -> np.ndarray:
    """proj/src/fourier_fit.cpp:107-129: the fitted series at arbitrary points."""
    q = np.ascontiguousarray(points, dtype=np.float64)
    out = np.empty(2 * q.size, dtype=np.float64)
    raw = coeffs._c()
    check(lib().sftgpu_reconstruct(C.byref(raw), q.ctypes.data_as(C.c_void_p), q.size, out.ctypes.data_as(C.c_void_p)))
    return out.view(np.complex128)


def tune_beta(rmse_of_beta, half_width: int):
    """proj/src/fourier_fit.cpp:395-438: 33-point prescan over [0.5 pi/K, 1.5 pi/K] plus
    golden section to 1e-4 relative, on any RMSE profile. Returns (beta, rmse)."""
    cb = C.CFUNCTYPE(C.c_double, C.c_double, C.c_void_p)(lambda b, _u: float(rmse_of_beta(b)))
    beta, rmse = C.c_double(), C.c_double()
    check(lib().sftgpu_tune_beta(cb, None, half_width, C.byref(beta), C.byref(rmse)))
    return beta.value, rmse.value


@dataclass
class WindowState:  # include/sft/engine.hpp:82-88
    via_prefix: np.ndarray
    via_recurrence: np.ndarray


def sliding_window_state(sig: Signal, cfg: SftConfig) -> WindowState:
    """proj/src/engine.cpp:270-300: u_{(2K+1)}[n+K] by the sliding-sum route (K5) and by
    the window-recurrence scan (K1), both on the GPU, output phase re-applied. Plain SFT."""
    if cfg.alpha != 0.0:
        raise ValueError("sliding_window_state: plain SFT only")
    k = SftConfig(cfg.half_width, cfg.beta, cfg.order, 0.0, cfg.n0, Strategy.KernelIntegral, Precision.Double,
                  cfg.window_2k1)
    a, b = sft_via_sliding_sum(sig, k), sft_components(sig, k)
    omega = cfg.beta * cfg.order.p if cfg.order.integer_order else cfg.order.omega
    ph = np.exp(1j * omega * np.arange(sig.size()))
    return WindowState(ph * (a.c - 1j * a.s), ph * (b.c - 1j * b.s))


@dataclass
class StabilityReport:  # include/sft/engine.hpp:94-100
    max_state_magnitude: float
    max_component_error: float
    reference_scale: float
    abs_error: np.ndarray


def stability_probe(sig: Signal, cfg: SftConfig) -> StabilityReport:
    """proj/src/engine.cpp:302-320: cfg at single precision against double (both GPU).
    max_state_magnitude: the peak |filter state| of the single-precision recurrence for the
    recursive strategies (K7, as the reference), else the peak |window state| of the scan."""
    n = sig.size()
    mk = lambda p: SftConfig(cfg.half_width, cfg.beta, cfg.order, cfg.alpha, cfg.n0, cfg.strategy, p,  # noqa: E731
                             cfg.window_2k1)
    if cfg.strategy != Strategy.KernelIntegral and cfg.order.integer_order:
        # recursive strategies: the reference's own single-precision recurrence (K7) and
        # its peak filter-state magnitude
        c, s, peak = components_replay(sig, [mk(Precision.Single)], 0, n - 1, want_state=True)
        lo = ComponentSeq(c[0], s[0])
        max_state = float(peak[0])
    else:
        lo = components_over(sig, mk(Precision.Single), 0, n - 1)
        max_state = float(np.hypot(lo.c, lo.s).max())
    ref = components_over(sig, mk(Precision.Double), 0, n - 1)
    err = np.maximum(np.abs(lo.c - ref.c), np.abs(lo.s - ref.s))
    scale = float(max(np.abs(ref.c).max(), np.abs(ref.s).max()))
    return StabilityReport(max_state, float(err.max() / scale if scale > 0 else err.max()), scale, err)


@dataclass
class CostReport:  # include/sft/sliding_sum.hpp:236-243
    parallel_steps: int
    outer_iterations: int
    total_adds: int
    total_mults: int
    predicted_regime: str


def cost_model(n: int, window: int, blocked: bool = False, core_budget: int = 1) -> CostReport:
    """proj/src/sliding_sum.cpp:7-40 for SlidingSumPlan::make(n, window, variant, M)."""
    p = sliding_sum_plan(n, window, blocked)
    regime = "O(log2 L) parallel time (M >= N)" if core_budget >= n else "O(N log2 L / M) parallel time (M < N)"
    return CostReport(p["parallel_steps"], p["blocked_stages"] if blocked else 1, p["total_adds"], 0, regime)


@dataclass
class MethodOpCounts:  # include/sft/sliding_sum.hpp:248-256
    mults: int
    adds: int
    regime: str


def sft_method_counts(n: int, orders: int, half_width: int, core_budget: int) -> MethodOpCounts:
    """proj/src/sliding_sum.cpp:42-52."""
    reg = "O(P log2 K) time (M >= N)" if core_budget >= n else "O(N P log2 K / M) time (M < N)"
    return MethodOpCounts(7 * n * orders, n * orders * (2 * half_width + 1), reg)


def conv_method_counts(n: int, sigma: float, core_budget: int) -> MethodOpCounts:
    """proj/src/sliding_sum.cpp:54-64."""
    w = int(round(6.0 * sigma)) + 1
    reg = "O(log2 sigma) time (M >= N(6 sigma + 1))" if core_budget >= n * w else "O(N sigma log2 sigma / M) time"
    return MethodOpCounts(n * w, n * w, reg)


def select_optimal_ps(sigma, xi, half_width, pd, n0=0) -> int:
    ps = C.c_int()
    check(lib().sftgpu_select_optimal_ps(sigma, xi, half_width, pd, n0, C.byref(ps)))
    return ps.value


def tune_beta_gauss(sigma, half_width, max_order, n0=0):
    b, r = C.c_double(), C.c_double()
    check(lib().sftgpu_tune_beta_gauss(sigma, half_width, max_order, n0, C.byref(b), C.byref(r)))
    return b.value, r.value


def gauss_kernel_rmse(bundle_spec: TransformSpec, kind: GaussKind, n0: int) -> float:
    r = C.c_double()
    check(lib().sftgpu_gauss_kernel_rmse(C.byref(bundle_spec._raw.gauss), int(kind), n0, C.byref(r)))
    return r.value


def morlet_direct_kernel_rmse(sigma, xi, half_width, ps, pd, n0) -> float:
    r = C.c_double()
    check(lib().sftgpu_morlet_direct_kernel_rmse(sigma, xi, half_width, ps, pd, n0, C.byref(r)))
    return r.value


def morlet_multiply_kernel_rmse(sigma, xi, half_width, pm, n0) -> float:
    r = C.c_double()
    check(lib().sftgpu_morlet_multiply_kernel_rmse(sigma, xi, half_width, pm, n0, C.byref(r)))
    return r.value


# ------------------------------------------------------------------ transforms
@dataclass
class TransformResult:  # include/sft/transforms.hpp:74-81
    values: np.ndarray
    complex_valued: bool
    abbreviation: str
    strategy: Strategy
    precision: Precision
    kernel_rmse_percent: float


def _host_ptr(a) -> int:
    """Address of a host buffer (numpy array or CPU torch tensor) without building a
    ctypes view: ndarray.ctypes costs microseconds per call on the streaming path."""
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.__array_interface__["data"][0]


def _check_device_buffer(t, dtype, need: int, device: int, name: str) -> None:
    """Plans take raw device pointers: a wrong dtype, a strided view, another device or a
    short buffer would be read or written out of bounds by the kernels. ``need`` is the
    minimum element count."""
    if not hasattr(t, "data_ptr") or not getattr(t, "is_cuda", False):
        raise ValueError(f"{name}: expected a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name}: dtype {t.dtype} does not match the plan ({dtype})")
    if not t.is_contiguous():
        raise ValueError(f"{name}: tensor must be contiguous")
    if t.device.index != device:
        raise ValueError(f"{name}: tensor is on cuda:{t.device.index}, the plan on cuda:{device}")
    if t.numel() < need:
        raise ValueError(f"{name}: {t.numel()} elements, the plan needs {need}")


def _check_host_buffer(a, itemsize: int, need: int, name: str) -> None:
    """Host buffers of the *_host entry points: numpy arrays or CPU tensors, C-contiguous,
    of the plan's element size and at least ``need`` elements."""
    if hasattr(a, "data_ptr"):
        if getattr(a, "is_cuda", False):
            raise ValueError(f"{name}: expected a host buffer, got a CUDA tensor")
        ok, size, n = a.is_contiguous(), a.element_size(), a.numel()
    else:
        ok, size, n = a.flags.c_contiguous, a.itemsize, a.size
    if not ok:
        raise ValueError(f"{name}: host buffer must be C-contiguous")
    if size != itemsize:
        raise ValueError(f"{name}: element size {size} does not match the plan ({itemsize})")
    if n < need:
        raise ValueError(f"{name}: {n} elements, the plan needs {need}")


class TransformPlan:
    """Device plan: ``batch`` signals of ``n`` samples -> transform output, all in HBM.
    x: [batch][ld_x] (float32 for Single, float64 for Double); out: [batch][ld_out]
    real, or [batch][ld_out][2] complex interleaved. ``out_range=(begin, count)``
    computes only outputs [begin, begin+count) (chunk sharding with halo)."""

    MODES = {"auto": 0, "seq": 1, "lookback": 2, "tc": 3}

    def __init__(self, spec: TransformSpec, n: int, batch: int = 1, boundary=BoundaryPolicy.Clamp,
                 out_range=None, mode: str = "auto"):
        h = C.c_void_p()
        begin, count = out_range if out_range is not None else (0, n)
        check(lib().sftgpu_transform_plan_create_ex(C.byref(spec._raw), n, batch, int(boundary), begin, count,
                                                    self.MODES[mode], C.byref(h)))
        self._h = h
        self._destroy = lib().sftgpu_plan_destroy
        self.n, self.batch, self.out_begin, self.count = n, batch, begin, count
        self.complex_out = bool(lib().sftgpu_plan_output_is_complex(h))
        conv = spec.kind in (TransformKind.TruncConvGauss, TransformKind.TruncConvMorlet)
        self.precision = Precision.Double if conv else spec.precision
        self.launches = lib().sftgpu_plan_launches_per_execute(h)
        self.device = _torch().cuda.current_device()
        self._cw = 2 if self.complex_out else 1

    def describe(self) -> dict:
        info = (C.c_int64 * 11)()
        check(lib().sftgpu_plan_describe(self._h, info, 11))
        keys = ("sequential", "direct_convolution", "positions_per_thread", "positions_per_tile", "warm_tiles",
                "chunks_per_signal", "ctas_per_launch", "launches", "orders", "group_mode", "tensor_cores")
        return dict(zip(keys, list(info)))

    @property
    def orders(self) -> int:
        """Basis orders the kernels evaluate (after dropping below-resolution terms)."""
        return self.describe()["orders"]

    def dtype(self):
        torch = _torch()
        return torch.float32 if self.precision == Precision.Single else torch.float64

    def empty_output(self):
        torch = _torch()
        shape = (self.batch, self.count, 2) if self.complex_out else (self.batch, self.count)
        return torch.empty(shape, dtype=self.dtype(), device="cuda")

    def execute(self, x, out, stream=None, ld_x=None, ld_out=None):
        """x: [batch][ld_x] and out: [batch][ld_out](x2 complex) contiguous CUDA tensors of
        the plan's dtype on the plan's device. One plan runs on one stream at a time;
        launches on a new stream are ordered after the plan's previous launch."""
        torch = _torch()
        lx, lo = ld_x or self.n, ld_out or self.count
        dt = self.dtype()
        _check_device_buffer(x, dt, (self.batch - 1) * lx + self.n, self.device, "x")
        _check_device_buffer(out, dt, ((self.batch - 1) * lo + self.count) * self._cw, self.device, "out")
        st = C.c_void_p(stream) if stream is not None else _stream_ptr(torch)
        check(lib().sftgpu_transform_execute(self._h, C.c_void_p(x.data_ptr()), lx,
                                             C.c_void_p(out.data_ptr()), lo, st))

    def _check_host(self, x_host, out_host):
        isz = 4 if self.precision == Precision.Single else 8
        _check_host_buffer(x_host, isz, self.batch * self.n, "x_host")
        _check_host_buffer(out_host, isz, self.batch * self.count * self._cw, "out_host")

    def execute_host(self, x_host: np.ndarray, out_host: np.ndarray, stream=None):
        torch = _torch()
        self._check_host(x_host, out_host)
        st = C.c_void_p(stream) if stream is not None else _stream_ptr(torch)
        check(lib().sftgpu_transform_execute_host(self._h, C.c_void_p(_host_ptr(x_host)),
                                                  C.c_void_p(_host_ptr(out_host)), st))

    def execute_host_async(self, x_host: np.ndarray, out_host: np.ndarray, stream=None):
        """Pipelined host-buffer execution (``sftgpu_transform_execute_host_async``): returns
        once queued; ``stream`` (default: torch's current) waits for the result copy."""
        self._check_host(x_host, out_host)
        st = C.c_void_p(stream) if stream is not None else _stream_ptr(_torch())
        check(lib().sftgpu_transform_execute_host_async(self._h, C.c_void_p(_host_ptr(x_host)),
                                                        C.c_void_p(_host_ptr(out_host)), st))

    def synchronize(self):
        check(lib().sftgpu_plan_synchronize(self._h))

    def __del__(self):
        # the destroy entry point is bound at creation: module globals may already be
        # torn down when this runs at interpreter exit
        if getattr(self, "_h", None) and getattr(self, "_destroy", None):
            self._destroy(self._h)
            self._h = None


class MultiScalePlan(TransformPlan):
    """All scales of a scalogram over ONE signal in one persistent tensor-core launch
    (``sftgpu_multiscale_plan_create``): x is the signal ([n] or [1][n], fp32), out is
    [len(specs)][count][2] (complex) or [len(specs)][count]. Every spec must be fp32,
    K4-eligible, with the same order count and output kind (ValueError otherwise);
    at most 128 specs."""

    def __init__(self, specs, n: int, boundary=BoundaryPolicy.Clamp, out_range=None):
        specs = list(specs)
        arr = (_abi.Spec * len(specs))(*[sp._raw for sp in specs])
        begin, count = out_range if out_range is not None else (0, n)
        h = C.c_void_p()
        check(lib().sftgpu_multiscale_plan_create(arr, len(specs), n, int(boundary), begin, count, C.byref(h)))
        self._h = h
        self._destroy = lib().sftgpu_plan_destroy
        self.n, self.batch, self.out_begin, self.count = n, len(specs), begin, count
        self.complex_out = bool(lib().sftgpu_plan_output_is_complex(h))
        self.precision = Precision.Single
        self.launches = lib().sftgpu_plan_launches_per_execute(h)
        self.device = _torch().cuda.current_device()
        self._cw = 2 if self.complex_out else 1

    def execute(self, x, out, stream=None, ld_x=None, ld_out=None):
        torch = _torch()
        lo = ld_out or self.count
        dt = self.dtype()
        _check_device_buffer(x, dt, self.n, self.device, "x")
        _check_device_buffer(out, dt, ((self.batch - 1) * lo + self.count) * self._cw, self.device, "out")
        st = C.c_void_p(stream) if stream is not None else _stream_ptr(torch)
        check(lib().sftgpu_transform_execute(self._h, C.c_void_p(x.data_ptr()), ld_x or self.n,
                                             C.c_void_p(out.data_ptr()), lo, st))

    def _check_host(self, x_host, out_host):
        _check_host_buffer(x_host, 4, self.n, "x_host")
        _check_host_buffer(out_host, 4, self.batch * self.count * self._cw, "out_host")


def _run(sig: Signal, spec: TransformSpec) -> TransformResult:
    """One reference-signature call (``sftgpu_transform_oneshot``): the library caches the
    plan, its device buffers and pinned staging per (spec, n, boundary, device)."""
    x = np.ascontiguousarray(sig.samples, dtype=np.float64)
    out = np.empty(2 * x.size, dtype=np.float64)
    cplx = C.c_int(0)
    check(lib().sftgpu_transform_oneshot(C.byref(spec._raw), x.size, int(sig.boundary), x.ctypes.data_as(C.c_void_p),
                                         out.ctypes.data_as(C.c_void_p), C.byref(cplx)))
    vals = out.view(np.complex128) if cplx.value else out[:x.size].astype(np.complex128)
    return TransformResult(vals, bool(cplx.value), spec.abbreviation, spec.strategy, spec.precision,
                           spec.kernel_rmse_percent)


def gauss_smooth(sig: Signal, spec: TransformSpec, workers: int = 1) -> TransformResult:
    """proj/src/transforms.cpp:279-335. ``workers`` is accepted for API parity."""
    if spec.kind not in (TransformKind.Gauss, TransformKind.GaussD, TransformKind.GaussDD):
        raise ValueError("gauss_smooth: spec kind mismatch")
    return _run(sig, spec)


def morlet_direct_transform(sig: Signal, spec: TransformSpec, workers: int = 1) -> TransformResult:
    """proj/src/transforms.cpp:337-371."""
    if spec.kind != TransformKind.MorletDirect:
        raise ValueError("morlet_direct_transform: spec mismatch")
    return _run(sig, spec)


def morlet_multiply_transform(sig: Signal, spec: TransformSpec, workers: int = 1) -> TransformResult:
    """proj/src/transforms.cpp:373-428."""
    if spec.kind != TransformKind.MorletMultiply:
        raise ValueError("morlet_multiply_transform: spec mismatch")
    return _run(sig, spec)


def truncated_reference(sig: Signal, spec: TransformSpec, workers: int = 1) -> TransformResult:
    """GCT3 / MCT3 (proj/src/transforms.cpp:430-442) on the GPU direct-convolution kernel."""
    if spec.kind not in (TransformKind.TruncConvGauss, TransformKind.TruncConvMorlet):
        raise ValueError("truncated_reference: spec mismatch")
    return _run(sig, spec)


def apply_transform(sig: Signal, spec: TransformSpec, workers: int = 1) -> TransformResult:
    """proj/src/transforms.cpp:444-459."""
    return _run(sig, spec)


def truncated_convolution(sig: Signal, kernel: KernelTaps, workers: int = 1) -> np.ndarray:
    """proj/src/kernels.cpp:35-51 on the GPU (fp64): out[n] = sum_k taps[k] x[n - (lo + k)]."""
    torch = _torch()
    if kernel.taps.size < 1:
        raise ValueError("truncated_convolution: empty kernel")
    x = torch.from_numpy(sig.samples).to("cuda")
    t = torch.from_numpy(np.ascontiguousarray(np.column_stack([kernel.taps.real, kernel.taps.imag]).ravel())).to("cuda")
    out = torch.empty(2 * sig.size(), dtype=torch.float64, device="cuda")
    check(lib().sftgpu_truncated_convolution(C.c_void_p(x.data_ptr()), sig.size(), int(sig.boundary),
                                             C.c_void_p(t.data_ptr()), kernel.taps.size, kernel.lo,
                                             C.c_void_p(out.data_ptr()), _stream_ptr(torch)))
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    return o[0::2] + 1j * o[1::2]
