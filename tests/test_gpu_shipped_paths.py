"""Parity of the shipped paths at the shapes they run in production (round-2 additions):

* the public one-call API (``morlet_direct_transform`` etc.) creates and destroys a
  look-back plan per call: stale look-back payloads of a freed plan must never be
  accepted by the next plan at the same address;
* BASELINE config 5 at full shape (N=2^24, sigma up to 16384, K4 with 147 chunk items
  per scale), both shardings, against the fp64 oracle over bounded windows;
* the sliding-sum route (proj/src/engine.cpp:323-337) against the oracle's sliding-sum
  route;
* "also checked against direct convolution" (north_star) for config 2 at sigma=8192 and
  config 3, through K3 (GPU fp64 direct convolution with the effective kernel);
* what "matches the reference" means at config 1: the exact transform (long-double
  direct convolution with the effective kernel) against the GPU and against the
  reference's default Recursive2 strategy.
"""
import numpy as np
import pytest

from conftest import rel_max
from test_gpu_transforms import oracle_transform

pytestmark = pytest.mark.gpu


def _vals(o):
    o = o.double().cpu().numpy()
    return o[..., 0] + 1j * o[..., 1] if o.shape[-1] == 2 and o.ndim >= 2 else o


# ------------------------------------------------------------------ cross-plan reuse
@pytest.mark.parametrize("prec", [0, 1])
def test_fresh_lookback_plans_never_accept_a_freed_plans_payloads(sft, O, prec):
    """60 create / execute-once / destroy cycles of same-shape look-back plans (the
    drop-in API's pattern), alternating two inputs: every plan's first launch carries the
    same launch tag as its freed predecessor's, so an uninitialised workspace would let a
    tile accept the previous signal's aggregates. Each result equals that input's first
    result bit for bit, and the first results match the fp64 oracle."""
    import torch

    spec = sft.make_transform_spec("MDS5P6", 8192.0, 10.0, sft.TransformOptions(precision=prec))
    n = 102400
    pr = sft.Precision.Double if prec else sft.Precision.Single
    xs = [sft.generate_signals(sft.TestSignalKind.SeededNoise, n, seed, 1, pr) for seed in (1234, 99)]
    refs = [None, None]
    for i in range(60):
        plan = sft.TransformPlan(spec, n, mode="lookback")
        assert plan.describe()["sequential"] == 0
        o = plan.empty_output()
        plan.execute(xs[i % 2], o)
        torch.cuda.synchronize()
        if refs[i % 2] is None:
            refs[i % 2] = o.clone()
        else:
            assert torch.equal(o, refs[i % 2]), i
        del plan
    for k in range(2):
        xh = xs[k].double().cpu().numpy()[0]
        assert rel_max(_vals(refs[k])[0], oracle_transform(O, xh, 1, spec)) < (1e-12 if prec else 1e-5)


def test_one_call_api_alternating_signals(sft, O):
    """The reference-signature entry point (one plan per call) on alternating signals:
    every call reproduces that signal's result exactly."""
    spec = sft.make_transform_spec("MDS5P6", 8192.0, 10.0, sft.TransformOptions(precision=0))
    sigs = [sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 102400, s).astype(np.float32)) for s in (5, 6)]
    first = [sft.morlet_direct_transform(s, spec).values for s in sigs]
    for i in range(30):
        assert np.array_equal(sft.morlet_direct_transform(sigs[i % 2], spec).values, first[i % 2]), i
    ref = oracle_transform(O, sigs[1].samples, 1, spec)
    assert rel_max(first[1], ref) < 1e-5


def test_plan_used_from_two_streams_is_ordered(sft, O):
    """One look-back plan executed alternately on two streams without host syncs: the
    plan orders each launch after its previous one (shared workspace and launch epochs),
    so every result is exact."""
    import torch

    spec = sft.make_transform_spec("MDS5P6", 4096.0, 10.0, sft.TransformOptions(precision=0))
    n = 102400
    xs = [sft.generate_signals(sft.TestSignalKind.SeededNoise, n, s, 1, sft.Precision.Single) for s in (1, 2)]
    plan = sft.TransformPlan(spec, n, mode="lookback")
    refs = []
    for x in xs:
        o = plan.empty_output()
        plan.execute(x, o)
        refs.append(o)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [plan.empty_output() for _ in range(20)]
    for i in range(20):
        s = streams[i % 2]
        with torch.cuda.stream(s):
            plan.execute(xs[i % 2], outs[i], stream=s.cuda_stream)
    torch.cuda.synchronize()
    for i in range(20):
        assert torch.equal(outs[i], refs[i % 2]), i


# ------------------------------------------------------------------ config 5 at full shape
def oracle_window(O, xh, spec, a, b, boundary=1):
    """fp64 oracle outputs [a, b) of a long signal, computed on the bounded input window
    those outputs read (x[o - n0 - K, o - n0 + K], transforms.cpp:287-288): the cut ends
    of the window are never read by these outputs, the true signal ends keep the
    boundary policy."""
    K, n0, n = spec.half_width, spec.n0, xh.size
    lo, hi = max(0, a - n0 - K - 2), min(n, b - n0 + K + 2)
    ref = oracle_transform(O, xh[lo:hi], boundary, spec)
    return ref[a - lo:b - lo]


def test_config5_full_shape_both_shardings(sft, O):
    """BASELINE config 5 shape: N=2^24, scales sigma in {16, ~1000, 8192, 16384}
    (K up to 49152), the production path (auto: K4 where eligible) for one rank, for
    two scale-sharded ranks and for two chunk-sharded (ranged) ranks. Windows at both
    signal ends, at the chunk-shard boundary and inside are checked against the fp64
    oracle (<= 1e-5, north_star); the sharded results equal the single-rank one (scale:
    bit for bit; chunk: each rank starts its own warm-up, <= 2e-6)."""
    import torch

    from paper_2110_11866_b200 import scalogram as SG

    sigmas = [16.0, 1000.0, 8192.0, 16384.0]
    specs = SG.build_specs(sigmas, xi=10.0, pd=6)
    n = 1 << 24
    x = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 1234, 1, sft.Precision.Single)[0]
    one = SG.Scalogram(n, specs)
    o1 = one.empty_output()
    one.run(x, o1)
    torch.cuda.synchronize()
    # scale sharding: ranks own alternate scales
    full_scale = torch.empty_like(o1)
    for r in range(2):
        sc = SG.Scalogram(n, specs, 2, r, "scale")
        o = sc.empty_output()
        sc.run(x, o)
        torch.cuda.synchronize()
        for j, i in enumerate(sc.rows):
            full_scale[i] = o[j]
    assert torch.equal(full_scale, o1)
    del full_scale
    # chunk sharding: ranged plans, each with its own halo
    full_chunk = torch.empty_like(o1)
    for r in range(2):
        sc = SG.Scalogram(n, specs, 2, r, "chunk")
        o = sc.empty_output()
        sc.run(x, o)
        torch.cuda.synchronize()
        full_chunk[:, sc.begin:sc.begin + sc.count] = o
    scale = o1.abs().amax(dim=(1, 2), keepdim=True)
    assert float(((full_chunk - o1).abs() / scale).max()) <= 2e-6
    xh = x.double().cpu().numpy()
    half = n // 2
    windows = [(0, 3000), (half - 2000, half + 2000), (9_876_543, 9_879_543), (n - 3000, n)]
    for i, spec in enumerate(specs):
        for a, b in windows:
            ref = oracle_window(O, xh, spec, a, b)
            for got in (o1, full_chunk):
                assert rel_max(_vals(got[i, a:b]), ref) < 1e-5, (sigmas[i], a)


# ------------------------------------------------------------------ sliding-sum route
@pytest.mark.parametrize("K,p,alpha,n", [(6, 2, 0.0, 500), (40, 3, 0.0, 3000), (40, 1, 0.01, 3000),
                                         (300, 5, 0.0, 20000)])
@pytest.mark.parametrize("boundary", [0, 1])
def test_sliding_sum_route_vs_oracle(sft, O, K, p, alpha, n, boundary):
    """sft_via_sliding_sum (proj/src/engine.cpp:323-337) against the oracle's restatement
    of the same route (phased sequence rebased, sliding_sum_flat, rescale): <= 1e-10
    relative (fp64; the routes differ only in rounding)."""
    beta = np.pi / K
    x = O.make_test_signal(O.SEEDED_NOISE, n, 31 + K)
    cfg = sft.SftConfig(K, beta, sft.OrderSpec.order(p), alpha, 0, sft.Strategy.KernelIntegral, sft.Precision.Double)
    got = sft.sft_via_sliding_sum(sft.Signal(x, boundary), cfg)
    oc = O.Cfg(K, beta, p, None, alpha, O.KERNEL_INTEGRAL, O.DOUBLE)
    rc, rs = O.sft_via_sliding_sum(x, boundary, oc)
    ref = rc - 1j * rs
    assert rel_max(got.c - 1j * got.s, ref) < 1e-10


# ------------------------------------------------------------------ direct convolution
def _k3(sft, x, spec):
    taps = sft.effective_kernel(spec)
    return sft.truncated_convolution(sft.Signal(x), taps)


def test_config2_sigma8192_vs_direct_convolution(sft, O):
    """Config 2 at sigma=8192 (K=24576): the fp32 ASFT transform against the GPU fp64
    direct convolution with the effective kernel (K3, itself <= 1e-13 of the oracle)."""
    spec = sft.make_gauss_spec(8192.0, 0, 6, 10, sft.TransformOptions(precision=0, strategy=0))
    for offset in (0.0, 1.0):
        x = (O.make_test_signal(O.SEEDED_NOISE, 102400, 1234) + offset).astype(np.float32).astype(np.float64)
        got = sft.gauss_smooth(sft.Signal(x), spec).values.real
        assert rel_max(got, _k3(sft, x, spec).real) < 1e-5


def test_config3_vs_direct_convolution(sft, O):
    """Config 3 (headline, MDS5P6 fp32 ASFT, sigma=8192) against K3's fp64 direct
    convolution with the effective kernel (49153 complex taps)."""
    spec = sft.make_transform_spec("MDS5P6", 8192.0, 10.0, sft.TransformOptions(precision=0, strategy=0))
    x = O.make_test_signal(O.SEEDED_NOISE, 102400, 1234).astype(np.float32).astype(np.float64)
    got = sft.morlet_direct_transform(sft.Signal(x), spec).values
    assert rel_max(got, _k3(sft, x, spec)) < 1e-5


def test_direct_convolution_kernel_vs_oracle_at_config3(sft, O):
    """K3 itself at the config-3 kernel, spot-checked against the oracle's fp64 direct
    convolution on a short signal."""
    spec = sft.make_transform_spec("MDS5P6", 8192.0, 10.0, sft.TransformOptions(precision=0, strategy=0))
    taps = sft.effective_kernel(spec)
    x = O.make_test_signal(O.SEEDED_NOISE, 6000, 4)
    got = sft.truncated_convolution(sft.Signal(x), taps)
    ref = O.truncated_convolution(x, 1, taps.taps, taps.lo, 8)
    assert rel_max(got, ref) < 1e-13


# ------------------------------------------------------------------ strategy deviations at config 1
def test_config1_exact_reference_and_strategy_deviations(sft, O):
    """Config 1 (GDP6 SFT fp64, N=102400, sigma=8192). The exact transform at spot
    outputs is a long-double direct convolution with the effective kernel. The GPU
    (kernel-integral semantics) is within 1e-12 of it; the reference's default strategy,
    Recursive2 (oracle restatement, proj/src/engine.cpp:53-120), drifts by ~5e-9
    (DESIGN.md §5 table), so "matches the reference within 1e-12" is defined against
    the reference's KernelIntegral strategy and the exact value, not Recursive2."""
    spec = sft.make_gauss_spec(8192.0, 0, 6, 0, sft.TransformOptions(strategy=0))
    n = 102400
    x = O.make_test_signal(O.SEEDED_NOISE, n, 1234)
    got = sft.gauss_smooth(sft.Signal(x), spec).values.real
    taps = sft.effective_kernel(spec)
    t = taps.taps.real.astype(np.longdouble)
    spots = np.array([0, 1, 777, 24575, 24576, 51200, 77823, 100000, n - 2, n - 1])
    xl = x.astype(np.longdouble)
    exact = []
    for o in spots:
        j = o - (taps.lo + np.arange(t.size))  # out[o] = sum_k taps[k] x[o - (lo + k)]
        exact.append(np.sum(t * xl[np.clip(j, 0, n - 1)]))  # clamp boundary
    exact = np.array(exact, dtype=np.longdouble)
    scale = float(np.max(np.abs(exact)))
    gpu_err = float(np.max(np.abs(got[spots].astype(np.longdouble) - exact))) / scale
    assert gpu_err < 1e-12
    b = spec.gauss_coeffs
    gamma = 1.0 / (2.0 * spec.sigma ** 2)
    ki = O.gauss_smooth(x, 1, 0, spec.half_width, spec.beta, 0, 0.0, gamma, O.KERNEL_INTEGRAL, O.DOUBLE,
                        b.a, b.b, b.d, 8).real
    r2 = O.gauss_smooth(x, 1, 0, spec.half_width, spec.beta, 0, 0.0, gamma, O.RECURSIVE2, O.DOUBLE,
                        b.a, b.b, b.d, 8).real
    ki_err = float(np.max(np.abs(ki[spots].astype(np.longdouble) - exact))) / scale
    r2_err = float(np.max(np.abs(r2[spots].astype(np.longdouble) - exact))) / scale
    assert ki_err < 1e-12
    assert 1e-11 < r2_err < 1e-7  # the default strategy's recursion drift (~5e-9)
    assert rel_max(got, ki) < 1e-12
