"""GPU parity for the component engine (K1 in components mode), ported from the
reference's hot-path pin proj/tests/test_engine.cpp. Every case runs the product
kernel through the C ABI and checks it against the reference's own oracle for the
case (brute-force defining sums, :14-31) or against the CPU restatement in oracle/.
"""
import math

import numpy as np
import pytest

from conftest import rel_max

pytestmark = pytest.mark.gpu


def ext(x, j, boundary):
    n = len(x)
    if 0 <= j < n:
        return x[j]
    if boundary == 0:
        return 0.0
    return x[0] if j < 0 else x[-1]


def brute(x, K, omega, alpha, boundary=1, lo=0, hi=None):
    """c[n] = sum_k x[n-k] e^{-alpha k} cos(omega k), s likewise with sin
    (proj/tests/test_engine.cpp:14-31)."""
    n = len(x)
    hi = n - 1 if hi is None else hi
    idx = np.arange(lo, hi + 1)
    xe = lambda j: np.array([ext(x, int(v), boundary) for v in j])
    c = np.zeros(idx.size)
    s = np.zeros(idx.size)
    for lag in range(-K, K + 1):
        w = math.exp(-alpha * lag) * xe(idx - lag)
        c += w * math.cos(omega * lag)
        s += w * math.sin(omega * lag)
    return c, s


def cfg(sft, K, beta, p, alpha=0.0, strategy=None, precision=None):
    return sft.SftConfig(K, beta, sft.OrderSpec.order(p), alpha, 0,
                         strategy if strategy is not None else sft.Strategy.Recursive2,
                         precision if precision is not None else sft.Precision.Double)


def maxdiff(a, b):
    return max(np.max(np.abs(a.c - b[0])), np.max(np.abs(a.s - b[1])))


STRATS = (0, 1, 2)


def test_constant_order_zero_sums_window(sft):
    K = 8
    ones = sft.Signal(np.ones(40))
    for st in STRATS:
        comp = sft.sft_components(ones, cfg(sft, K, math.pi / K, 0, strategy=st))
        assert np.allclose(comp.c, 2 * K + 1, rtol=1e-12, atol=0)
        assert np.max(np.abs(comp.s)) < 1e-10


def test_constant_higher_orders_match_window_sum(sft):
    K = 8
    beta = math.pi / K
    ones = sft.Signal(np.ones(40))
    for p in (1, 2, 3):
        ws = sum(math.cos(beta * p * lag) for lag in range(-K, K + 1))
        comp = sft.sft_components(ones, cfg(sft, K, beta, p))
        assert np.max(np.abs(comp.c - ws)) < 1e-9
        assert np.max(np.abs(comp.s)) < 1e-10


def test_all_strategies_agree_with_brute_force(sft, O):
    K = 8
    x = O.make_test_signal(O.SEEDED_NOISE, 64, 7)
    for beta in (math.pi / K, 1.07 * math.pi / K):
        ref = brute(x, K, beta * 3, 0.0)
        for st in STRATS:
            comp = sft.sft_components(sft.Signal(x), cfg(sft, K, beta, 3, strategy=st))
            assert maxdiff(comp, ref) < 1e-10


def test_single_precision_coarse_tolerance(sft, O):
    K = 12
    x = O.make_test_signal(O.SEEDED_NOISE, 200, 11)
    ref = brute(x, K, math.pi / K * 3, 0.0)
    bound = 1e-4 * (2 * K + 1) * np.max(np.abs(x))
    for st in STRATS:
        comp = sft.sft_components(sft.Signal(x), cfg(sft, K, math.pi / K, 3, strategy=st, precision=0))
        assert maxdiff(comp, ref) < bound


def test_attenuated_matches_brute_force(sft, O):
    K, alpha = 8, 0.05
    x = O.make_test_signal(O.SEEDED_NOISE, 64, 19)
    ref = brute(x, K, math.pi / K * 2, alpha)
    for st in STRATS:
        comp = sft.asft_components(sft.Signal(x), cfg(sft, K, math.pi / K, 2, alpha, st))
        assert maxdiff(comp, ref) < 1e-9


def test_attenuated_impulse_closed_form(sft):
    K, alpha, center, p = 10, 0.08, 25, 2
    beta = math.pi / K
    x = np.zeros(51)
    x[25] = 1.0
    comp = sft.asft_components(sft.Signal(x, sft.BoundaryPolicy.Zero), cfg(sft, K, beta, p, alpha, 1))
    for n in range(51):
        lag = n - center
        if abs(lag) <= K:
            assert abs(comp.c[n] - math.exp(-alpha * lag) * math.cos(beta * p * lag)) < 1e-9
            assert abs(comp.s[n] - math.exp(-alpha * lag) * math.sin(beta * p * lag)) < 1e-9
        else:
            assert abs(comp.c[n]) < 1e-10 and abs(comp.s[n]) < 1e-10


def test_tiny_attenuation_approaches_plain(sft, O):
    K = 8
    x = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 64, 23))
    plain = sft.sft_components(x, cfg(sft, K, math.pi / K, 2, 0.0, 1))
    tiny = sft.asft_components(x, cfg(sft, K, math.pi / K, 2, 1e-8, 1))
    assert maxdiff(plain, (tiny.c, tiny.s)) < 1e-5 * np.max(np.abs(plain.c))


def test_linearity(sft, O):
    K = 7
    c = cfg(sft, K, math.pi / K, 2)
    x = O.make_test_signal(O.SEEDED_NOISE, 80, 5)
    y = O.make_test_signal(O.SEEDED_NOISE, 80, 6)
    cx = sft.sft_components(sft.Signal(x), c)
    cy = sft.sft_components(sft.Signal(y), c)
    cm = sft.sft_components(sft.Signal(2.5 * x - 1.25 * y), c)
    assert np.max(np.abs(cm.c - (2.5 * cx.c - 1.25 * cy.c))) < 1e-10
    assert np.max(np.abs(cm.s - (2.5 * cx.s - 1.25 * cy.s))) < 1e-10


def test_shift_covariance(sft, O):
    K = 6
    c = cfg(sft, K, math.pi / K, 2, 0.0, 1)
    x = O.make_test_signal(O.SEEDED_NOISE, 96, 9)
    sh = np.zeros(96)
    sh[1:] = x[:95]
    cx = sft.sft_components(sft.Signal(x, 0), c)
    cs = sft.sft_components(sft.Signal(sh, 0), c)
    for n in range(K + 2, 96 - K - 2):
        assert abs(cs.c[n] - cx.c[n - 1]) < 1e-10 and abs(cs.s[n] - cx.s[n - 1]) < 1e-10


def test_real_frequency_equals_integer_order_exactly(sft, O):
    K = 9
    beta = math.pi / K
    x = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 70, 13))
    ci = cfg(sft, K, beta, 3, strategy=0)
    cr = cfg(sft, K, beta, 3, strategy=0)
    cr.order = sft.OrderSpec.frequency(beta * 3)
    a = sft.sft_components(x, ci)
    b = sft.sft_components(x, cr)
    assert np.array_equal(a.c, b.c) and np.array_equal(a.s, b.s)


def test_real_frequency_requires_kernel_integral(sft, O):
    c = cfg(sft, 8, math.pi / 8, 1, strategy=1)
    c.order = sft.OrderSpec.frequency(0.3)
    with pytest.raises(ValueError):
        sft.sft_components(sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 32, 1)), c)


def test_negative_real_frequency(sft, O):
    K, omega = 8, -0.21
    x = O.make_test_signal(O.SEEDED_NOISE, 64, 29)
    c = cfg(sft, K, math.pi / K, 0, strategy=0)
    c.order = sft.OrderSpec.frequency(omega)
    comp = sft.sft_components(sft.Signal(x), c)
    assert maxdiff(comp, brute(x, K, omega, 0.0)) < 1e-10


def test_2k1_variant_matches_default(sft, O):
    K = 8
    x = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 64, 37))
    for alpha in (0.0, 0.03):
        a = cfg(sft, K, math.pi / K, 2, alpha, 1)
        b = cfg(sft, K, math.pi / K, 2, alpha, 1)
        b.window_2k1 = True
        ca = sft.components_over(x, a, 0, 63)
        cb = sft.components_over(x, b, 0, 63)
        assert maxdiff(ca, (cb.c, cb.s)) < 1e-10


def test_extended_range_sees_boundary(sft, O):
    K = 5
    x = O.make_test_signal(O.SEEDED_NOISE, 40, 41)
    ext_ = sft.components_over(sft.Signal(x), cfg(sft, K, math.pi / K, 1), -3, 36)
    ref = brute(x, K, math.pi / K, 0.0)
    for n in range(3, 40):
        assert abs(ext_.c[n] - ref[0][n - 3]) < 1e-10
    # and the whole signed range against brute force with boundary reads
    rb = brute(x, K, math.pi / K, 0.0, 1, -3, 36)
    assert maxdiff(ext_, rb) < 1e-10


def test_sliding_sum_route_equals_kernel_integral(sft, O):
    K = 16
    x = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 256, 17))
    for p in range(7):
        c = cfg(sft, K, math.pi / K, p, strategy=0)
        d = sft.sft_components(x, c)
        t = sft.sft_via_sliding_sum(x, c)
        assert maxdiff(d, (t.c, t.s)) < 1e-10 * max(1.0, np.max(np.abs(d.c)))
    c = cfg(sft, K, math.pi / K, 2, 0.01, 0)
    t = sft.sft_via_sliding_sum(x, c)
    assert maxdiff(sft.asft_components(x, c), (t.c, t.s)) < 1e-9
    z = sft.sft_via_sliding_sum(sft.Signal(np.ones(64)), cfg(sft, 8, math.pi / 8, 0, strategy=0))
    assert np.allclose(z.c, 17.0, rtol=1e-12, atol=0)


def test_sliding_route_rejects_overflow(sft, O):
    x = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 20000, 1))
    with pytest.raises(ValueError):
        sft.sft_via_sliding_sum(x, cfg(sft, 16, math.pi / 16, 1, 0.1, 0))


def test_engine_validation(sft, O):
    x = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 16, 1))
    with pytest.raises(ValueError):
        sft.asft_components(x, cfg(sft, 4, math.pi / 4, 1, 0.0, 1))
    with pytest.raises(ValueError):
        sft.sft_components(x, cfg(sft, 4, math.pi / 4, 1, 0.5, 1))
    with pytest.raises(ValueError):
        sft.sft_components(x, cfg(sft, 0, 1.0, 0, 0.0, 1))
    with pytest.raises(ValueError):
        sft.components_over(x, cfg(sft, 4, math.pi / 4, 1), 5, 4)


@pytest.mark.parametrize("K,n,alpha,boundary", [(3, 1, 0.0, 1), (8, 5, 0.0, 0), (40, 100, 0.0, 1),
                                                 (300, 2000, 0.0, 1), (300, 5000, 1e-3, 0),
                                                 (1000, 700, 2e-4, 1), (2500, 20000, 0.0, 1)])
def test_components_match_oracle_fp64(sft, O, K, n, alpha, boundary):
    """fp64 components vs the oracle's kernel-integral restatement, ranges shifted
    like the ASFT reconstructions (lo = -n0); tolerance 1e-12 relative."""
    x = O.make_test_signal(O.SEEDED_NOISE, n, 1000 + K)
    lo, hi = -2, n - 3
    for p in (0, 1, 5):
        c = cfg(sft, K, math.pi / K, p, alpha, 0)
        got = sft.components_over(sft.Signal(x, boundary), c, lo, hi)
        rc, rs = O.components_over(x, boundary, O.Cfg(K, math.pi / K, p, alpha=alpha, strategy=0), lo, hi)
        scale = max(np.max(np.abs(rc)), np.max(np.abs(rs)))
        assert max(np.max(np.abs(got.c - rc)), np.max(np.abs(got.s - rs))) / scale < 1e-12


@pytest.mark.parametrize("offset", [0.0, 1.0])
def test_components_fp32_vs_fp64_oracle(sft, O, offset):
    """fp32 state with fp64 carries: <= 1e-5 relative to the fp64 oracle, including the
    DC-offset case that breaks a global fp32 prefix (SURVEY.md §7 hard parts)."""
    K, n = 24576, 102400
    x = (O.make_test_signal(O.SEEDED_NOISE, n, 1234) + offset).astype(np.float32).astype(np.float64)
    for p in (0, 6, 12):
        c = cfg(sft, K, math.pi / K, p, 7.45e-8, 0, 0)
        got = sft.components_over(sft.Signal(x), c, -5, n - 6)
        rc, rs = O.components_over(x, 1, O.Cfg(K, math.pi / K, p, alpha=7.45e-8, strategy=0), -5, n - 6)
        scale = max(np.max(np.abs(rc)), np.max(np.abs(rs)))
        err = max(np.max(np.abs(got.c - rc)), np.max(np.abs(got.s - rs))) / scale
        assert err < 1e-5, (p, err)


def test_window_state_two_routes_and_stability_probe(sft, O):
    """sliding_window_state (proj/src/engine.cpp:270-300): the sliding-sum route (K5) and
    the window-recurrence scan (K1) give the same u[n+K] (the reference's equivalence test,
    proj/tests/test_engine.cpp); stability_probe (engine.cpp:302-320) reports the fp32 scan
    against fp64: with the bounded 2K-window state the error does not grow with n."""
    x = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 3000, 21))
    st = sft.sliding_window_state(x, cfg(sft, 40, math.pi / 40, 3, strategy=0))
    assert np.max(np.abs(st.via_prefix - st.via_recurrence)) < 1e-10 * np.max(np.abs(st.via_recurrence))
    # brute force u[n] = sum_{j=n-K}^{n+K} x[j] e^{i omega j}
    xs, K, w = x.samples, 40, 3 * math.pi / 40
    for n in (0, 1234, 2999):
        j = np.clip(np.arange(n - K, n + K + 1), 0, 2999)
        u = np.sum(xs[j] * np.exp(1j * w * np.arange(n - K, n + K + 1)))
        assert abs(st.via_recurrence[n] - u) < 1e-10 * abs(u) + 1e-12
    with pytest.raises(ValueError):
        sft.sliding_window_state(x, cfg(sft, 40, math.pi / 40, 3, 0.01, strategy=0))
    y = sft.Signal(O.make_test_signal(O.SEEDED_NOISE, 100000, 3) + 1.0)
    rep = sft.stability_probe(y, cfg(sft, 256, math.pi / 256, 2, strategy=0))
    assert rep.max_component_error < 1e-5
    head, tail = rep.abs_error[:10000].max(), rep.abs_error[-10000:].max()
    assert tail < 4 * head + 1e-12 * rep.reference_scale
