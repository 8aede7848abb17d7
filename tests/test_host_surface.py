"""CPU: host-side parts of the drop-in surface that need no GPU (proj/src/fourier_fit.cpp
reconstruct / tune_beta, proj/src/sliding_sum.cpp cost models), checked against the
reference's definitions and printed values."""
import math

import numpy as np


def test_tune_beta_generic_profile(sft):
    K = 40
    b, r = sft.tune_beta(lambda x: (x - 0.9 * math.pi / K) ** 2 + 1.0, K)
    assert abs(b - 0.9 * math.pi / K) < 1e-3 * math.pi / K
    assert abs(r - 1.0) < 1e-12
    # a profile minimised at the edge of [0.5, 1.5] pi/K stays inside the bracket
    b2, _ = sft.tune_beta(lambda x: x, K)
    assert 0.5 * math.pi / K <= b2 < 0.52 * math.pi / K


def test_reconstruct_matches_series(sft):
    K = 18
    q = np.arange(-K, K + 1)
    target = np.exp(-q ** 2 / 72.0)
    cs = sft.fit_mmse(target, K, math.pi / K, list(range(7)), [])
    pts = np.array([-4.5, 0.0, 3.0, 11.25])
    got = sft.reconstruct(cs, pts)
    want = sum(cs.cos_coeffs[i] * np.cos(math.pi / K * p * pts) for i, p in enumerate(cs.cos_orders))
    assert np.allclose(got, want, rtol=0, atol=1e-14)
    assert abs(got[2].real - math.exp(-9 / 72.0)) < 2e-3


def test_cost_models(sft):
    cr = sft.cost_model(500, 37, blocked=True)
    assert (cr.parallel_steps, cr.outer_iterations, cr.total_adds, cr.total_mults) == (6, 2, 7744, 0)  # test_output.txt:41
    flat = sft.cost_model(5, 3)
    assert flat.parallel_steps == 2 and flat.total_adds == 5 * 2 + 5 * 2
    assert sft.cost_model(100, 10, core_budget=100).predicted_regime.startswith("O(log2 L)")
    sc = sft.sft_method_counts(1000, 7, 24, 1)
    assert (sc.mults, sc.adds) == (49000, 343000)
    cc = sft.conv_method_counts(1000, 8.0, 10 ** 9)
    assert cc.adds == 1000 * 49 and cc.regime.startswith("O(log2 sigma)")
