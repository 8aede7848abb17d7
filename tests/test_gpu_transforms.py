"""GPU parity for the fused transform path (K1: scan + coefficient combine), ported from
proj/tests/test_transforms.cpp plus full-size checks at BASELINE.json's configs.

Checkers: the reference's exactness identity (transform == truncated convolution with
the effective kernel, :14-19, < 1e-9 in fp64), the oracle's restatement of the
reference combine (oracle.gauss_smooth / morlet_direct / morlet_multiply), and the
fp64 oracle for the fp32 ASFT kernels (north_star: <= 1e-5 relative, fp64 SFT <= 1e-12).
"""
import math

import numpy as np
import pytest

from conftest import rel_max

pytestmark = pytest.mark.gpu


def oracle_transform(O, x, boundary, spec, workers=8, precision=None):
    """The reference combine restated in oracle/, on the same coefficients."""
    import paper_2110_11866_b200 as P

    prec = O.DOUBLE if precision is None else precision
    k = spec.kind
    if k in (P.TransformKind.Gauss, P.TransformKind.GaussD, P.TransformKind.GaussDD):
        b = spec.gauss_coeffs
        gamma = 1.0 / (2.0 * spec.sigma ** 2)
        return O.gauss_smooth(x, boundary, int(k), spec.half_width, spec.beta, spec.n0, spec.alpha, gamma,
                              O.KERNEL_INTEGRAL, prec, b.a, b.b, b.d, workers).astype(np.complex128)
    if k == P.TransformKind.MorletDirect:
        c = spec.morlet_coeffs
        gamma = 1.0 / (2.0 * spec.sigma ** 2)
        return O.morlet_direct(x, boundary, spec.half_width, spec.beta, spec.n0, spec.alpha, gamma,
                               O.KERNEL_INTEGRAL, prec, c.cos_orders, c.cos_coeffs, c.sin_orders, c.sin_coeffs,
                               workers)
    if k == P.TransformKind.MorletMultiply:
        e = spec.envelope_coeffs
        return O.morlet_multiply(x, boundary, spec.half_width, spec.beta, spec.n0, spec.alpha, spec.sigma, spec.xi,
                                 O.KERNEL_INTEGRAL, prec, e.cos_coeffs.real, workers)
    raise ValueError(k)


def exactness_error(sft, O, sig, spec):
    res = sft.apply_transform(sig, spec)
    taps = sft.effective_kernel(spec)
    ref = O.truncated_convolution(sig.samples, int(sig.boundary), taps.taps, taps.lo, 8)
    return rel_max(res.values, ref)


def test_every_transform_equals_convolution_with_fitted_kernel(sft, O):
    """proj/tests/test_transforms.cpp:23-40"""
    sig = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 96, 101))
    for strategy in (0, 1, 2):
        opts = sft.TransformOptions(strategy=strategy)
        for n0 in (0, 1):
            for kind in (0, 1, 2):
                assert exactness_error(sft, O, sig, sft.make_gauss_spec(6.0, kind, 4, n0, opts)) < 1e-9
            assert exactness_error(sft, O, sig, sft.make_morlet_direct_spec(8.0, 6.0, 5, n0, opts)) < 1e-9
            assert exactness_error(sft, O, sig, sft.make_morlet_multiply_spec(8.0, 6.0, 3, n0, opts)) < 1e-9


def test_tuned_beta_keeps_identity(sft, O):
    sig = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 120, 7))
    spec = sft.make_gauss_spec(8.0, 0, 4, 2, sft.TransformOptions(tune_beta=True))
    assert exactness_error(sft, O, sig, spec) < 1e-9


def test_constant_signal_responses(sft):
    ones = sft.Signal(np.ones(64))
    smooth = sft.make_gauss_spec(8.0, 0, 5, 0, sft.TransformOptions(tune_beta=True, half_width=32))
    r = sft.gauss_smooth(ones, smooth)
    mass = sft.effective_kernel(smooth).taps.real.sum()
    assert abs(mass - 1.0) < 1e-3
    assert np.allclose(r.values.real, mass, rtol=1e-10, atol=0)
    flat = sft.gauss_smooth(ones, sft.make_gauss_spec(8.0, 1, 4, 0))
    assert np.max(np.abs(flat.values)) < 1e-10
    d_asft = sft.make_gauss_spec(16.0, 1, 5, 1, sft.TransformOptions(tune_beta=True))
    assert np.max(np.abs(sft.gauss_smooth(ones, d_asft).values)) < 2e-4


def test_ramp_slope_response(sft, O):
    size = 200
    sig = sft.Signal(np.arange(size, dtype=float), sft.BoundaryPolicy.Clamp)
    spec = sft.make_gauss_spec(8.0, 1, 4, 0, sft.TransformOptions(tune_beta=True))
    r = sft.gauss_smooth(sig, spec)
    K = spec.half_width
    taps = np.array([O.gauss_d(8.0, i) for i in range(-K, K + 1)])
    oracle = O.truncated_convolution(sig.samples, 1, taps, -K)
    for n in range(K, size - K):
        assert abs(r.values[n].real - oracle[n].real) <= 0.01 * abs(oracle[n].real)
        assert abs(r.values[n].real - 1.0) <= 0.03


def test_zero_shift_reduces_to_plain(sft, O):
    sig = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 80, 3))
    s = sft.make_gauss_spec(8.0, 0, 4, 0)
    z = s.copy()
    z.n0 = 0
    z.alpha = 0.0
    assert np.array_equal(sft.gauss_smooth(sig, s).values, sft.gauss_smooth(sig, z).values)


def test_impulse_peaks_agree(sft):
    x = np.zeros(129)
    x[64] = 1.0
    sig = sft.Signal(x, sft.BoundaryPolicy.Zero)
    o = sft.TransformOptions(tune_beta=True)
    s0 = sft.make_gauss_spec(10.0, 0, 4, 0, o)
    s2 = sft.make_gauss_spec(10.0, 0, 4, 2, o)
    rs, ra = sft.gauss_smooth(sig, s0), sft.gauss_smooth(sig, s2)
    assert int(np.argmax(np.abs(rs.values))) == 64 and int(np.argmax(np.abs(ra.values))) == 64
    K = s0.half_width
    for n in range(64 - (K - 2), 64 + (K - 2) + 1):
        assert abs(ra.values[n].real - rs.values[n].real) <= 5e-3 * max(abs(rs.values[n].real), 0.01)


def test_pure_tone_morlet_flat_magnitude(sft):
    size, sigma, xi = 2048, 60.0, 10.0
    sig = sft.Signal(np.cos(xi * np.arange(size) / sigma))
    spec = sft.make_morlet_direct_spec(sigma, xi, 6, 0)
    r = sft.morlet_direct_transform(sig, spec)
    K = spec.half_width
    mag = np.abs(r.values[K:size - K])
    assert (mag.max() - mag.min()) / mag.max() < 0.02
    assert mag.max() > 0.1


def test_zero_signal_maps_to_zero(sft):
    sig = sft.Signal(np.zeros(64), sft.BoundaryPolicy.Zero)
    assert np.max(np.abs(sft.morlet_direct_transform(sig, sft.make_morlet_direct_spec(8.0, 6.0, 5, 0)).values)) == 0.0
    assert np.max(np.abs(sft.morlet_multiply_transform(sig, sft.make_morlet_multiply_spec(8.0, 6.0, 3, 0)).values)) == 0.0


def test_noise_accuracy_vs_true_kernel(sft, O):
    sig = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 256, 55))
    spec = sft.make_gauss_spec(16.0, 0, 4, 0, sft.TransformOptions(tune_beta=True))
    r = sft.gauss_smooth(sig, spec)
    K = spec.half_width
    ref = O.truncated_convolution(sig.samples, 1, np.array([O.gauss(16.0, i) for i in range(-K, K + 1)]), -K)
    err = math.sqrt(np.sum(np.abs(r.values - ref) ** 2) / max(1e-30, np.sum(np.abs(ref) ** 2)))
    assert err < 3.0 * spec.kernel_rmse_percent / 100.0 + 1e-6
    assert spec.kernel_rmse_percent < 0.6


def test_sft_asft_interior_agreement(sft, O):
    sig = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 512, 77))
    s0 = sft.make_morlet_direct_spec(12.0, 8.0, 6, 0)
    s3 = sft.make_morlet_direct_spec(12.0, 8.0, 6, 3)
    rs, ra = sft.morlet_direct_transform(sig, s0), sft.morlet_direct_transform(sig, s3)
    K = s0.half_width
    num = np.sum(np.abs(rs.values[3 * K:512 - 3 * K] - ra.values[3 * K:512 - 3 * K]) ** 2)
    den = np.sum(np.abs(rs.values[3 * K:512 - 3 * K]) ** 2)
    assert math.sqrt(num / den) < 5.0 * max(s0.kernel_rmse_percent, s3.kernel_rmse_percent) / 100.0


def test_abbreviation_factory_names(sft, O):
    x = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 64, 5))
    for name in ("GDP6", "MDP5", "MDP6", "MDP7", "MDP9", "MDP11", "MDS5P5", "MDS5P7", "MDS5P9", "MDS5P11",
                 "MMP2", "MMP3", "MMP4", "MMP5", "MMS5P2", "MMS5P3", "MMS5P4", "MMS5P5", "GCT3", "MCT3"):
        sigma = 16.0 if name[0] == "G" else 60.0
        r = sft.apply_transform(x, sft.make_transform_spec(name, sigma, 10.0))
        assert r.values.size == 64 and np.all(np.isfinite(r.values))


def test_reference_paths_truncated_true_kernels(sft):
    x = np.zeros(97)
    x[48] = 1.0
    sig = sft.Signal(x, sft.BoundaryPolicy.Zero)
    rg = sft.apply_transform(sig, sft.make_transform_spec("GCT3", 8.0, 0.0))
    g = lambda t: math.sqrt((1 / 128) / math.pi) * math.exp(-(1 / 128) * t * t)
    assert abs(rg.values[48].real - g(0)) <= 1e-14 * g(0)
    assert abs(rg.values[72].real - g(24)) <= 1e-12 * g(24)
    assert rg.values[73].real == 0.0
    rm = sft.apply_transform(sig, sft.make_transform_spec("MCT3", 8.0, 6.0))
    import oracle as O

    m0, m8 = O.morlet(8.0, 6.0, 0.0), O.morlet(8.0, 6.0, -8.0)
    assert abs(rm.values[48].real - m0.real) <= 1e-13 * abs(m0.real)
    assert abs(rm.values[40].imag - m8.imag) <= 1e-12 * max(abs(m8.imag), 1.0)
    assert rm.complex_valued


def test_single_tracks_double(sft, O):
    sig = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 256, 33))
    for strategy in (0, 1, 2):
        for n0 in (0, 2):
            spec = sft.make_gauss_spec(12.0, 0, 4, n0, sft.TransformOptions(strategy=strategy))
            ref = sft.gauss_smooth(sig, spec)
            spec.precision = sft.Precision.Single
            lo = sft.gauss_smooth(sig, spec)
            assert np.max(np.abs(lo.values - ref.values)) < 1e-3 * np.max(np.abs(ref.values))


def test_results_independent_of_workers_and_batch(sft, O):
    """Bit-identical regardless of worker count (test_transforms.cpp:267-277) and of the
    batch a signal is processed in (grid-independence of the look-back scan)."""
    import torch

    sig = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 200, 21))
    for spec in (sft.make_gauss_spec(8.0, 2, 4, 2), sft.make_morlet_direct_spec(8.0, 6.0, 5, 1),
                 sft.make_morlet_multiply_spec(8.0, 6.0, 3, 1)):
        one = sft.apply_transform(sig, spec, 1)
        four = sft.apply_transform(sig, spec, 4)
        assert np.array_equal(one.values, four.values)
        plan = sft.TransformPlan(spec, 200, 5, sig.boundary)
        xb = torch.from_numpy(np.tile(sig.samples, (5, 1))).cuda()
        out = plan.empty_output()
        plan.execute(xb, out)
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        vals = o[..., 0] + 1j * o[..., 1] if plan.complex_out else o
        for b in range(5):
            assert np.array_equal(vals[b], one.values if plan.complex_out else one.values.real)


def test_shift_validation(sft):
    with pytest.raises(ValueError):
        sft.make_gauss_spec(8.0, 0, 4, 3)
    with pytest.raises(ValueError):
        sft.make_morlet_direct_spec(8.0, 6.0, 5, 3)
    sft.make_gauss_spec(8.0, 0, 4, 2)


@pytest.mark.parametrize("abbrev,sigma,xi,n0kind", [("GDP6", 6.0, 0.0, 0), ("MDS2P5", 9.0, 7.0, 0),
                                                    ("MMS1P3", 5.0, 6.0, 0), ("MMP2", 4.0, 3.0, 0)])
@pytest.mark.parametrize("n", [1, 2, 7, 33, 1000, 4099])
@pytest.mark.parametrize("boundary", [0, 1])
def test_edge_sizes_vs_oracle(sft, O, abbrev, sigma, xi, n0kind, n, boundary):
    """Ragged sizes (N=1 .. non-multiples of the tile), both boundary policies, K > N."""
    spec = sft.make_transform_spec(abbrev, sigma, xi)
    x = O.make_test_signal(O.SEEDED_NOISE, n, 77 + n)
    got = sft.apply_transform(sft.Signal(x, boundary), spec).values
    ref = oracle_transform(O, x, boundary, spec)
    assert rel_max(got, ref) < 1e-12


def test_config1_gauss_sft_fp64_full_size(sft, O):
    """BASELINE config 1: GDP6 SFT fp64, N=102400, sigma=8192, K=24576: <= 1e-12."""
    spec = sft.make_gauss_spec(8192.0, 0, 6, 0, sft.TransformOptions(strategy=0))
    x = O.make_test_signal(O.SEEDED_NOISE, 102400, 1234)
    got = sft.gauss_smooth(sft.Signal(x), spec).values.real
    ref = oracle_transform(O, x, 1, spec).real
    assert rel_max(got, ref) < 1e-12


@pytest.mark.parametrize("sigma", [64.0, 512.0, 8192.0])
@pytest.mark.parametrize("offset", [0.0, 1.0])
def test_config2_gauss_asft_fp32(sft, O, sigma, offset):
    """BASELINE config 2: Gauss ASFT fp32 (P=6, n0=10), N=102400: <= 1e-5 vs the fp64
    oracle of the same spec; also vs direct convolution with the effective kernel."""
    spec = sft.make_gauss_spec(sigma, 0, 6, 10, sft.TransformOptions(precision=0, strategy=0))
    x = (O.make_test_signal(O.SEEDED_NOISE, 102400, 1234) + offset).astype(np.float32).astype(np.float64)
    got = sft.gauss_smooth(sft.Signal(x), spec).values.real
    ref = oracle_transform(O, x, 1, spec).real
    assert rel_max(got, ref) < 1e-5
    if sigma <= 512.0:
        taps = sft.effective_kernel(spec)
        conv = O.truncated_convolution(x, 1, taps.taps, taps.lo, 8).real
        assert rel_max(got, conv) < 1e-5


def test_config3_morlet_direct_fp32_headline(sft, O):
    """BASELINE config 3 (headline): MDS5P6 fp32 ASFT, N=102400, sigma=8192, xi=10."""
    spec = sft.make_transform_spec("MDS5P6", 8192.0, 10.0, sft.TransformOptions(precision=0, strategy=0))
    assert spec.ps == 7 and abs(spec.kernel_rmse_percent - 0.6127) < 1e-3
    x = O.make_test_signal(O.SEEDED_NOISE, 102400, 1234).astype(np.float32).astype(np.float64)
    got = sft.morlet_direct_transform(sft.Signal(x), spec).values
    ref = oracle_transform(O, x, 1, spec)
    assert rel_max(got, ref) < 1e-5


def test_config4_morlet_multiply_fp32_batch(sft, O):
    """BASELINE config 4 shape (MMS5P3 fp32, sigma=8192, xi=10) on a batch of signals:
    every row vs the fp64 oracle (a sample of rows at full length)."""
    import torch

    spec = sft.make_transform_spec("MMS5P3", 8192.0, 10.0, sft.TransformOptions(precision=0))
    B, n = 16, 102400
    xb = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 1234, B, sft.Precision.Single)
    plan = sft.TransformPlan(spec, n, B)
    out = plan.empty_output()
    plan.execute(xb, out)
    torch.cuda.synchronize()
    xh = xb.double().cpu().numpy()
    oh = out.cpu().numpy()
    for b in (0, 7, 15):
        ref = oracle_transform(O, xh[b], 1, spec)
        assert rel_max(oh[b, :, 0] + 1j * oh[b, :, 1], ref) < 1e-5


def test_device_generator_bit_exact(sft, O):
    import torch

    for kind in (0, 1, 3):
        g = sft.generate_signals(kind, 1000, 42, 3, sft.Precision.Double).cpu().numpy()
        for b in range(3):
            assert np.array_equal(g[b], O.make_test_signal(kind, 1000, 42 + b))
    ch = sft.generate_signals(2, 1000, 1, 1, sft.Precision.Double).cpu().numpy()[0]
    assert np.max(np.abs(ch - O.make_test_signal(2, 1000, 1))) < 1e-12


def test_gpu_truncated_convolution_matches_oracle(sft, O):
    x = O.make_test_signal(O.SEEDED_NOISE, 3000, 9)
    rng = np.random.default_rng(0)
    taps = rng.standard_normal(1500) + 1j * rng.standard_normal(1500)
    for boundary in (0, 1):
        got = sft.truncated_convolution(sft.Signal(x, boundary), sft.KernelTaps(taps, -700))
        ref = O.truncated_convolution(x, boundary, taps, -700, 8)
        assert rel_max(got, ref) < 1e-13


@pytest.mark.parametrize("abbrev,sigma,xi,prec,tol", [("MMS5P3", 64.0, 10.0, 0, 1e-5), ("GDP6", 100.0, 0.0, 1, 1e-12),
                                                      ("MDS3P6", 40.0, 8.0, 0, 1e-5), ("MMP2", 30.0, 4.0, 1, 1e-12)])
def test_batched_seq_mode_vs_oracle(sft, O, abbrev, sigma, xi, prec, tol):
    """Batches >= 256 signals run one CTA per signal (SEQ mode, no look-back): rows are
    checked against the oracle, and every row against the single-signal (LB) result."""
    import torch

    spec = sft.make_transform_spec(abbrev, sigma, xi, sft.TransformOptions(precision=prec))
    B, n = 300, 3001
    xb = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 99, B, sft.Precision(prec))
    plan = sft.TransformPlan(spec, n, B)
    out = plan.empty_output()
    plan.execute(xb, out)
    torch.cuda.synchronize()
    xh = xb.double().cpu().numpy()
    oh = out.double().cpu().numpy()
    vals = oh[..., 0] + 1j * oh[..., 1] if plan.complex_out else oh
    for b in (0, 137, 299):
        assert rel_max(vals[b], oracle_transform(O, xh[b], 1, spec)) < tol
    single = sft.TransformPlan(spec, n, 1)
    o1 = single.empty_output()
    for b in (5, 250):
        single.execute(xb[b:b + 1].contiguous(), o1)
        torch.cuda.synchronize()
        r = o1.double().cpu().numpy()[0]
        r = r[..., 0] + 1j * r[..., 1] if plan.complex_out else r
        assert rel_max(vals[b], r) < tol


@pytest.mark.parametrize("prec,tol", [(0, 2e-6), (1, 1e-12)])
def test_range_plans_match_full_transform(sft, O, prec, tol):
    """Chunk sharding: plans over an output range [b, b+c) read their halo from the full
    signal and reproduce the full transform's rows (boundary chunks included)."""
    import torch

    spec = sft.make_transform_spec("MDS3P6", 40.0, 8.0, sft.TransformOptions(precision=prec))
    n = 10007
    x = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 5, 1, sft.Precision(prec))
    full = sft.TransformPlan(spec, n)
    fo = full.empty_output()
    full.execute(x, fo)
    for b, c in ((0, 1), (0, 2500), (2500, 2500), (9000, 1007), (n - 1, 1), (123, 9000)):
        p = sft.TransformPlan(spec, n, 1, sft.BoundaryPolicy.Clamp, (b, c))
        po = p.empty_output()
        p.execute(x, po)
        torch.cuda.synchronize()
        a = po[0].double().cpu().numpy()
        r = fo[0, b:b + c].double().cpu().numpy()
        assert np.max(np.abs(a - r)) <= tol * np.max(np.abs(fo.double().cpu().numpy()))


def test_scalogram_single_gpu_vs_oracle(sft, O):
    """Config 5 shape on a reduced grid: every scale row vs the oracle, both shardings
    (world=1) agree."""
    import torch

    from paper_2110_11866_b200 import scalogram as SG

    sig = SG.scale_sigmas(6, 16.0, 256.0)
    specs = SG.build_specs(sig, xi=10.0, pd=6)
    n = 20000
    x = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 1234, 1, sft.Precision.Single)[0]
    sc = SG.Scalogram(n, specs)
    out = sc.empty_output()
    sc.run(x, out)
    torch.cuda.synchronize()
    xh = x.double().cpu().numpy()
    o = out.double().cpu().numpy()
    for r, i in enumerate(sc.rows):
        s = specs[i]
        c = s.morlet_coeffs
        ref = O.morlet_direct(xh, 1, s.half_width, s.beta, s.n0, s.alpha, 1.0 / (2 * s.sigma ** 2), O.KERNEL_INTEGRAL,
                              O.DOUBLE, c.cos_orders, c.cos_coeffs, c.sin_orders, c.sin_coeffs)
        assert rel_max(o[r, :, 0] + 1j * o[r, :, 1], ref) < 1e-5


@pytest.mark.parametrize("abbrev,sigma,xi,prec,tol", [("MDS3P6", 40.0, 8.0, 0, 2e-6), ("GDP6", 300.0, 0.0, 1, 1e-12),
                                                      ("MMS5P3", 100.0, 10.0, 0, 2e-6)])
def test_chunked_sequential_matches_lookback(sft, O, abbrev, sigma, xi, prec, tol):
    """A long single signal in sequential mode is split into chunks that each start from
    their own warm-up; it must agree with the look-back path and with the oracle."""
    import torch

    spec = sft.make_transform_spec(abbrev, sigma, xi, sft.TransformOptions(precision=prec))
    n = 300007
    x = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 11, 1, sft.Precision(prec))
    outs = {}
    for mode in ("seq", "lookback"):
        p = sft.TransformPlan(spec, n, 1, mode=mode)
        d = p.describe()
        assert d["sequential"] == (mode == "seq")
        if mode == "seq":
            assert d["chunks_per_signal"] > 1
        o = p.empty_output()
        p.execute(x, o)
        torch.cuda.synchronize()
        outs[mode] = o[0].double().cpu().numpy()
    scale = np.max(np.abs(outs["lookback"]))
    assert np.max(np.abs(outs["seq"] - outs["lookback"])) <= tol * scale
    xh = x[0].double().cpu().numpy()
    ref = oracle_transform(O, xh, 1, spec)
    got = outs["seq"][..., 0] + 1j * outs["seq"][..., 1] if outs["seq"].ndim == 2 else outs["seq"]
    assert rel_max(got, ref) < (1e-5 if prec == 0 else 1e-12)


@pytest.mark.parametrize("mode", ["lookback", "seq"])
@pytest.mark.parametrize("prec,tol", [(0, 1e-5), (1, 1e-12)])
@pytest.mark.parametrize("boundary", [0, 1])
def test_split_launches_modes_boundaries(sft, O, mode, prec, tol, boundary):
    """17 orders (MMS5P5: 11 real-frequency + 6 kappa orders; xi=6 keeps the kappa terms
    above fp64 resolution) run as two accumulating launches; both execution modes, both
    precisions and both boundary policies agree with the oracle."""
    import torch

    spec = sft.make_transform_spec("MMS5P5", 60.0, 6.0, sft.TransformOptions(precision=prec))
    n = 20011
    x = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 3, 2, sft.Precision(prec))
    plan = sft.TransformPlan(spec, n, 2, boundary, mode=mode)
    assert plan.launches == 2
    out = plan.empty_output()
    plan.execute(x, out)
    torch.cuda.synchronize()
    xh = x.double().cpu().numpy()
    oh = out.double().cpu().numpy()
    for b in range(2):
        ref = oracle_transform(O, xh[b], boundary, spec)
        assert rel_max(oh[b, :, 0] + 1j * oh[b, :, 1], ref) < tol


@pytest.mark.parametrize("prec,tol", [(0, 1e-5), (1, 1e-12)])
def test_sequential_ranged_plans(sft, O, prec, tol):
    """Ranged plans in sequential (chunked) mode: each output chunk starts its own warm-up
    inside the range and still matches the full-signal oracle."""
    import torch

    spec = sft.make_transform_spec("GDS3P6", 50.0, 0.0, sft.TransformOptions(precision=prec))
    n = 400009
    x = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 21, 1, sft.Precision(prec))
    ref = oracle_transform(O, x[0].double().cpu().numpy(), 1, spec).real
    for b, c in ((0, 150000), (150000, 250009), (333, 7)):
        p = sft.TransformPlan(spec, n, 1, sft.BoundaryPolicy.Clamp, (b, c), mode="seq")
        o = p.empty_output()
        p.execute(x, o)
        torch.cuda.synchronize()
        assert rel_max(o[0].double().cpu().numpy(), ref[b:b + c]) < tol


def test_plan_reuse_and_graph_capture(sft, O):
    """Plans carry no host-side per-launch state: repeated executes and CUDA-graph
    replays give identical results."""
    import torch

    spec = sft.make_transform_spec("MDS5P6", 512.0, 10.0, sft.TransformOptions(precision=0))
    n = 50000
    x = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 8, 1, sft.Precision.Single)
    plan = sft.TransformPlan(spec, n)
    o1, o2 = plan.empty_output(), plan.empty_output()
    plan.execute(x, o1)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        plan.execute(x, o2)  # warm on the capture stream
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        o2.zero_()
        with torch.cuda.graph(g, stream=s):
            for _ in range(3):
                plan.execute(x, o2)
        for _ in range(4):
            g.replay()
        s.synchronize()
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)


@pytest.mark.parametrize("prec", [0, 1])
def test_lookback_launch_tags_reject_stale_payloads(sft, O, prec):
    """The look-back payloads of fp32 plans carry a launch tag (epoch mod 15) instead of
    a flag, fp64 plans a flag with the full epoch: across 40 launches (the tag wraps
    twice) over alternating inputs, every result equals that input's first result bit
    for bit, so no tile ever consumed a predecessor's payload from an earlier launch."""
    import torch

    spec = sft.make_transform_spec("MDS5P6", 8192.0, 10.0, sft.TransformOptions(precision=prec))
    n = 102400
    pr = sft.Precision.Double if prec else sft.Precision.Single
    xs = [sft.generate_signals(sft.TestSignalKind.SeededNoise, n, seed, 1, pr) for seed in (3, 4)]
    plan = sft.TransformPlan(spec, n, mode="lookback")
    assert plan.describe()["sequential"] == 0
    refs = []
    for x in xs:
        o = plan.empty_output()
        plan.execute(x, o)
        refs.append(o)
    o = plan.empty_output()
    for i in range(40):
        plan.execute(xs[i % 2], o)
        torch.cuda.synchronize()
        assert torch.equal(o, refs[i % 2]), i
    xh = xs[1].double().cpu().numpy()[0]
    got = refs[1].double().cpu().numpy()
    got = got[..., 0] + 1j * got[..., 1]
    assert rel_max(got[0], oracle_transform(O, xh, 1, spec)) < (1e-12 if prec else 1e-5)


@pytest.mark.parametrize("mode", ["lookback", "seq"])
def test_pipelined_host_execution(sft, O, mode):
    """sftgpu_transform_execute_host_async: a stream of distinct pinned host buffers, all
    calls in flight before one sync, each result bit-identical to the synchronous call."""
    import torch

    spec = sft.make_transform_spec("MDS5P6", 512.0, 10.0, sft.TransformOptions(precision=0))
    n, batch, calls = 40000, 2, 7
    plan = sft.TransformPlan(spec, n, batch=batch, mode=mode)
    xs = [torch.from_numpy(np.stack([O.make_test_signal(O.SEEDED_NOISE, n, 100 + 3 * i + b) for b in range(batch)])
                           .astype(np.float32)).pin_memory() for i in range(calls)]
    outs = [torch.empty(tuple(plan.empty_output().shape), dtype=torch.float32).pin_memory() for _ in range(calls)]
    for i in range(calls):
        plan.execute_host_async(xs[i].numpy(), outs[i].numpy())
    torch.cuda.current_stream().synchronize()
    plan.synchronize()
    ref = np.empty(tuple(outs[0].shape), dtype=np.float32)
    for i in range(calls):
        plan.execute_host(xs[i].numpy(), ref)
        assert np.array_equal(outs[i].numpy(), ref)


@pytest.mark.parametrize("xi,nord", [(10.0, 7), (6.0, 11)])
def test_multiply_kappa_terms_below_resolution_are_skipped(sft, O, xi, nord):
    """The multiplication method's kappa correction (transforms.cpp:373-428) scales with
    e^{-xi^2/2}: at xi=10 it is ~2e-22 of the envelope weights, below fp64 resolution,
    and the plan drops those orders (one complex injection constant for the remaining
    2P+1); at xi=6 they stay. Either way the result matches the oracle, which sums all
    3P+2 orders."""
    import torch

    spec = sft.make_transform_spec("MMS5P3", 300.0, xi, sft.TransformOptions(precision=1))
    n = 9001
    plan = sft.TransformPlan(spec, n, 1, mode="lookback")
    x = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, 5, 1, sft.Precision.Double)
    out = plan.empty_output()
    plan.execute(x, out)
    torch.cuda.synchronize()
    assert plan.orders == nord
    ref = oracle_transform(O, x[0].cpu().numpy(), 1, spec)
    oh = out[0].cpu().numpy()
    assert rel_max(oh[:, 0] + 1j * oh[:, 1], ref) < 1e-12
