"""CPU: the product's host precompute (libsftgpu's fits and spec factories, no GPU
needed) against the reference's printed values and its fit tests
(proj/tests/test_fourier_fit.cpp, proj/test_output.txt)."""
import json
import math
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_values.json")))


def test_morlet_golden_fits(sft):
    """proj/test_output.txt:33-38: P_S selection and kernel RMSE to ~15 digits."""
    g = GOLD["morlet_fits"]
    s = sft.make_transform_spec("MDP6", 60.0, 8.0)
    assert s.ps == g["MDP6_sigma60_xi8"]["ps"]
    assert abs(s.kernel_rmse_percent - g["MDP6_sigma60_xi8"]["kernel_rmse_percent"]) < 1e-12
    assert abs(s.morlet_coeffs.fit_rmse_percent - g["MDP6_sigma60_xi8"]["fit_grid_residual_percent"]) < 1e-12
    s = sft.make_transform_spec("MDS5P7", 60.0, 10.0)
    assert abs(s.kernel_rmse_percent - g["MDS5P7_sigma60_xi10"]["kernel_rmse_percent"]) < 1e-12


def test_fit_recovers_target_in_span(sft):
    K = 32
    beta = math.pi / K
    t = np.cos(beta * 2 * np.arange(-K, K + 1))
    f = sft.fit_mmse(t, K, beta, [0, 1, 2, 3, 4], [])
    for p in range(5):
        assert abs(f.cos_coeffs[p].real - (1.0 if p == 2 else 0.0)) < 1e-10
        assert abs(f.cos_coeffs[p].imag) < 1e-14
    assert f.fit_rmse_percent < 1e-8


def test_fit_matches_independent_normal_equations(sft):
    """proj/tests/test_fourier_fit.cpp:49-77 with numpy's lstsq as the independent solver."""
    K = 12
    beta = math.pi / K
    q = np.arange(-K, K + 1, dtype=float)
    g = 1.0 / (2 * 16.0)
    target = math.sqrt(g / math.pi) * np.exp(-g * q * q)
    basis = np.stack([np.cos(beta * p * q) for p in range(4)], axis=1)
    ref, *_ = np.linalg.lstsq(basis, target, rcond=None)
    f = sft.fit_mmse(target, K, beta, [0, 1, 2, 3], [])
    ref_rmse = math.sqrt(np.sum((basis @ ref - target) ** 2) / np.sum(target ** 2)) * 100
    assert abs(f.fit_rmse_percent - ref_rmse) <= 1e-10 * ref_rmse
    assert np.allclose(f.cos_coeffs.real, ref, rtol=1e-9, atol=0)


def test_residual_orthogonal_and_monotone(sft):
    K = 64
    q = np.arange(-K, K + 1, dtype=float)
    g = 1.0 / (2 * 400.0)
    target = math.sqrt(g / math.pi) * np.exp(-g * q * q)
    f = sft.fit_mmse(target, K, math.pi / K, [0, 1, 2, 3], [])
    rec = sum(f.cos_coeffs[p].real * np.cos(math.pi / K * p * q) for p in range(4))
    for p in range(4):
        assert abs(np.sum((rec - target) * np.cos(math.pi / K * p * q))) < 1e-9 * math.sqrt(np.sum(target ** 2))
    prev = 1e9
    for order in range(1, 7):
        b = sft.fit_gaussian_bundle(30.0, 96, order, math.pi / 96)
        assert b.fit_rmse_g <= prev + 1e-12
        prev = b.fit_rmse_g


def test_degenerate_basis_rejected(sft):
    with pytest.raises(sft.FitDegenerateError):
        sft.fit_mmse(np.ones(25), 12, 1e-9, [0, 1, 2, 3, 4], [])


def test_beta_tuning_accuracy_scale(sft):
    """proj/tests/test_fourier_fit.cpp:119-130"""
    _, r3 = sft.tune_beta_gauss(256.0 / 3.5, 256, 3)
    assert r3 <= 0.20
    _, r6 = sft.tune_beta_gauss(256.0 / 4.6, 256, 6)
    assert r6 <= 0.003
    _, r5 = sft.tune_beta_gauss(256.0 / 3.5, 256, 5)
    assert r5 <= r3


def test_optimal_start_order(sft):
    """proj/tests/test_fourier_fit.cpp:153-176"""
    assert sft.select_optimal_ps(60.0, 1.0, 180, 6) == 0
    prev = 0
    for xi in (4.0, 10.0, 16.0):
        ps = sft.select_optimal_ps(60.0, xi, 180, 6)
        assert ps >= prev
        prev = ps
    p0 = round(12.0 * 180.0 / (math.pi * 60.0))
    assert abs(sft.select_optimal_ps(60.0, 12.0, 180, 6) - (p0 - 3)) <= 2
    best = sft.select_optimal_ps(60.0, 16.0, 180, 6)
    assert best > 0
    assert sft.morlet_direct_kernel_rmse(60.0, 16.0, 180, best, 6, 0) < sft.morlet_direct_kernel_rmse(60.0, 16.0, 180, 0, 6, 0)


def test_kappa_negligible_at_large_xi(sft):
    K = 180
    beta = math.pi / K
    wk = sft.fit_morlet_direct(60.0, 20.0, K, 10, 6, beta)
    q = np.arange(-K, K + 1, dtype=float)
    cxi = 1.0 / math.sqrt(1.0 + math.exp(-400.0) - 2.0 * math.exp(-0.75 * 400.0))
    env = cxi / (math.pi ** 0.25 * math.sqrt(60.0)) * np.exp(-q * q / (2 * 3600.0))
    cf = sft.fit_mmse(env * np.cos(20.0 * q / 60.0), K, beta, list(range(10, 16)), [])
    assert np.max(np.abs(wk.cos_coeffs.real - cf.cos_coeffs.real)) < 1e-8


def test_envelope_weights_fold_back(sft):
    env = sft.fit_morlet_envelope(60.0, 10.0, 180, 3, math.pi / 180)
    for n in (-50, -7, 0, 13, 101):
        es = sum((env.cos_coeffs[abs(p)].real * (1 if p == 0 else 0.5)) * np.exp(1j * env.beta * p * n) for p in range(-3, 4))
        cs = sum(env.cos_coeffs[p].real * math.cos(env.beta * p * n) for p in range(4))
        assert abs(es.real - cs) <= 1e-12 * abs(cs) and abs(es.imag) < 1e-14


def test_truncation_baseline(O):
    """proj/test_output.txt:22 (0.4613%): 3-sigma truncated Gaussian vs full over [-3K,3K]."""
    K = 256
    sigma = K / 3.0
    tr = math.floor(3.0 * sigma + 1e-9)
    n = np.arange(-3 * K, 3 * K + 1)
    truth = np.array([O.gauss(sigma, float(v)) for v in n])
    approx = np.where(np.abs(n) <= tr, truth, 0.0)
    r = math.sqrt(np.sum((approx - truth) ** 2) / np.sum(truth ** 2)) * 100
    assert f"{r:.4f}" == f"{GOLD['truncation_baseline_percent']['value']:.4f}"


def golden_min(f, lo, hi, prescan, tol):
    at = lambda i: lo + (hi - lo) * i / (prescan - 1)
    vals = [f(at(i)) for i in range(prescan)]
    bi = int(np.argmin(vals))
    a, b = at(max(0, bi - 1)), at(min(prescan - 1, bi + 1))
    ip = (math.sqrt(5.0) - 1.0) / 2.0
    c, d = b - ip * (b - a), a + ip * (b - a)
    fc, fd = f(c), f(d)
    while b - a > tol * b:
        if fc < fd:
            b, d, fd = d, c, fc
            c = b - ip * (b - a)
            fc = f(c)
        else:
            a, c, fc = c, d, fd
            d = a + ip * (b - a)
            fd = f(d)
    return 0.5 * (a + b)


@pytest.mark.parametrize("variant,P", [("SFT", 4), ("ASFT", 3), ("SFT", 6)])
def test_table1_cells(sft, variant, P):
    """proj/test_output.txt:8-17: the reference's Table-1 reproduction (eval.cpp:98-133
    restated in the test), joint (sigma, beta) tuning at K=256 -> the printed cells."""
    K, n0 = 256, (0 if variant == "SFT" else 10)
    sig_star = golden_min(lambda s: sft.tune_beta_gauss(s, K, P, n0)[1], K / 5.0, K / 2.8, 17, 1e-5)
    beta, _ = sft.tune_beta_gauss(sig_star, K, P, n0)
    spec = sft.make_gauss_spec(sig_star, sft.GaussKind.Value, P, n0, sft.TransformOptions(half_width=K, beta=beta))
    want = GOLD["table1"][variant][str(P)]
    assert f"{sig_star:.2f}" == f"{want[0]:.2f}"
    for kind, w in zip((0, 1, 2), want[1:]):
        got = sft.gauss_kernel_rmse(spec, kind, n0)
        assert f"{got:.4g}" == f"{w:.4g}", (kind, got, w)


def test_abbreviation_codec(sft):
    """proj/tests/test_transforms.cpp:200-233"""
    d = sft.parse_abbreviation("MDS5P7")
    assert d.kind == sft.TransformKind.MorletDirect and d.n0 == 5 and d.order == 7
    m = sft.parse_abbreviation("MMP3")
    assert m.kind == sft.TransformKind.MorletMultiply and m.n0 == 0 and m.order == 3
    assert sft.parse_abbreviation("GDP6").kind == sft.TransformKind.Gauss
    for bad in ("XP3", "GMP3", "MD", "MDSP3", "MDP0"):
        with pytest.raises(ValueError):
            sft.parse_abbreviation(bad)
    assert sft.encode_abbreviation(sft.TransformKind.GaussD, 2, 4) == "GDS2P4:d1"
    assert sft.encode_abbreviation(sft.TransformKind.MorletMultiply, 0, 3) == "MMP3"


def test_shift_and_param_validation(sft):
    with pytest.raises(ValueError):
        sft.make_gauss_spec(8.0, 0, 4, 3)
    with pytest.raises(ValueError):
        sft.make_morlet_direct_spec(8.0, 6.0, 5, 3)
    with pytest.raises(ValueError):
        sft.make_morlet_direct_spec(8.0, 0.0, 5, 0)
    with pytest.raises(ValueError):
        sft.make_gauss_spec(0.0, 0, 4, 0)
    sft.make_gauss_spec(8.0, 0, 4, 2)


def test_effective_kernel_shapes(sft):
    s = sft.make_gauss_spec(8.0, 0, 4, 2)
    t = sft.effective_kernel(s)
    assert t.lo == -24 + 2 and t.taps.size == 49
    g = sft.make_transform_spec("GCT3", 8.0, 0.0)
    assert g.half_width == 24 and sft.effective_kernel(g).lo == -24


def test_config3_spec_matches_survey_probe(sft):
    """MDS5P6 at sigma=8192, xi=10 -> P_S = 7, kernel RMSE 0.6127%."""
    s = sft.make_transform_spec("MDS5P6", 8192.0, 10.0, sft.TransformOptions(precision=sft.Precision.Single))
    assert s.ps == 7 and s.half_width == 24576 and f"{s.kernel_rmse_percent:.4f}" == "0.6127"


def test_coefficient_file_round_trip(sft, tmp_path):
    """proj/tests/test_fourier_fit.cpp:210-241: sets survive the "sft-coefficients v1"
    text format bit-for-bit (%.17g); a bad header is rejected."""
    direct = sft.make_morlet_direct_spec(60.0, 10.0, 6, 5, sft.TransformOptions(half_width=120))
    path = str(tmp_path / "c.coef")
    sft.write_coefficient_sets(path, [direct])
    text = open(path).read()
    assert text.startswith("sft-coefficients v1\nset kind=MorletDirect K=120 ")
    loaded = sft.read_coefficient_sets(path)
    assert len(loaded) == 1 and loaded[0].half_width == 120 and loaded[0].n0 == 5
    raw = direct._raw.morlet
    assert list(loaded[0].cos_coeffs[:2 * raw.n_cos]) == list(raw.cos_coeffs[:2 * raw.n_cos])
    assert list(loaded[0].sin_coeffs[:2 * raw.n_sin]) == list(raw.sin_coeffs[:2 * raw.n_sin])
    again = sft.morlet_direct_spec_from_coeffs(loaded[0], sft.Precision.Double, sft.Strategy.Recursive2, True)
    assert again.ps == direct.ps and again.pd == 6 and again.n0 == 5 and again.alpha == direct.alpha
    assert abs(again.kernel_rmse_percent - direct.kernel_rmse_percent) < 1e-12
    bad = tmp_path / "bad.coef"
    bad.write_text("not a header\n")
    with pytest.raises(ValueError):
        sft.read_coefficient_sets(str(bad))


def test_scalogram_coefficient_cache_matches_fresh_fits(sft):
    """The committed 128-scale coefficient cache equals fresh fits (spot check)."""
    import os

    from paper_2110_11866_b200 import scalogram as SG

    cache = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2110_11866_b200",
                         "data", "scalogram128_xi10_pd6.coef")
    sets = sft.read_coefficient_sets(cache)
    sig = SG.scale_sigmas()
    assert len(sets) == 128
    for i in (0, 40, 90):
        fresh = sft.make_morlet_direct_spec(sig[i], 10.0, 6, SG.default_n0(sig[i]),
                                            sft.TransformOptions(precision=sft.Precision.Single))
        raw = fresh._raw.morlet
        assert sets[i].n_cos == raw.n_cos and list(sets[i].cos_orders[:raw.n_cos]) == list(raw.cos_orders[:raw.n_cos])
        assert max(abs(a - b) for a, b in zip(sets[i].cos_coeffs[:2 * raw.n_cos], raw.cos_coeffs[:2 * raw.n_cos])) < 1e-15
