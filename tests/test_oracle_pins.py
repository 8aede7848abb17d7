"""CPU: pin the oracle (oracle/, the restatement of the reference) against every
known-answer check the reference's own tests hold for the path, and against the
numbers its captured run printed (tests/golden/reference_values.json)."""
import json
import math
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_values.json")))


def brute(x, K, omega, alpha, boundary=1):
    n = len(x)
    def ext(j):
        if 0 <= j < n:
            return x[j]
        return 0.0 if boundary == 0 else (x[0] if j < 0 else x[-1])
    c, s = np.zeros(n), np.zeros(n)
    for i in range(n):
        for lag in range(-K, K + 1):
            w = math.exp(-alpha * lag) * ext(i - lag)
            c[i] += w * math.cos(omega * lag)
            s[i] += w * math.sin(omega * lag)
    return c, s


def md(a, b):
    return max(np.max(np.abs(a[0] - b[0])), np.max(np.abs(a[1] - b[1])))


def test_signal_generators(O):
    """proj/tests/test_signal.cpp:28-52"""
    assert np.all(O.make_test_signal(O.CONSTANT, 4, 0) == 1.0)
    imp = O.make_test_signal(O.IMPULSE, 5, 0)
    assert list(imp) == [0, 0, 1, 0, 0]
    a, b, c = (O.make_test_signal(O.SEEDED_NOISE, 3, s) for s in (42, 42, 43))
    assert np.array_equal(a, b) and np.all(np.abs(a) <= 1.0) and a[0] != c[0]
    assert np.array_equal(O.make_test_signal(O.CHIRP, 64, 1), O.make_test_signal(O.CHIRP, 64, 2))
    with pytest.raises(O.OracleInvalidArgument):
        O.make_test_signal(O.CONSTANT, 0, 0)


def test_splitmix_independent_restatement(O):
    """splitmix64 + uniform_pm1 (proj/src/signal.cpp:9-20) recomputed in Python."""
    st = 1234
    M = (1 << 64) - 1
    vals = []
    for _ in range(50):
        st = (st + 0x9E3779B97F4A7C15) & M
        z = st
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        z ^= z >> 31
        vals.append(2.0 * ((z >> 11) * 2.0 ** -53) - 1.0)
    assert np.array_equal(np.array(vals), O.make_test_signal(O.SEEDED_NOISE, 50, 1234))


@pytest.mark.parametrize("strategy", [0, 1, 2])
def test_strategies_vs_brute_force(O, strategy):
    """proj/tests/test_engine.cpp:80-91 and :106-116"""
    K = 8
    x = O.make_test_signal(O.SEEDED_NOISE, 64, 7)
    for beta in (math.pi / K, 1.07 * math.pi / K):
        ref = brute(x, K, beta * 3, 0.0)
        got = O.sft_components(x, O.CLAMP, O.Cfg(K, beta, 3, strategy=strategy))
        assert md(got, ref) < 1e-10
    x = O.make_test_signal(O.SEEDED_NOISE, 64, 19)
    ref = brute(x, K, math.pi / K * 2, 0.05)
    got = O.asft_components(x, O.CLAMP, O.Cfg(K, math.pi / K, 2, alpha=0.05, strategy=strategy))
    assert md(got, ref) < 1e-9


def test_single_precision_tolerance(O):
    """proj/tests/test_engine.cpp:93-104"""
    K = 12
    x = O.make_test_signal(O.SEEDED_NOISE, 200, 11)
    ref = brute(x, K, math.pi / K * 3, 0.0)
    bound = 1e-4 * (2 * K + 1) * np.max(np.abs(x))
    for st in (0, 1, 2):
        got = O.sft_components(x, O.CLAMP, O.Cfg(K, math.pi / K, 3, strategy=st, precision=O.SINGLE))
        assert md(got, ref) < bound


def test_constant_and_impulse_closed_forms(O):
    """proj/tests/test_engine.cpp:51-62, :118-141"""
    ones = np.ones(40)
    for st in (0, 1, 2):
        c, s = O.sft_components(ones, O.CLAMP, O.Cfg(8, math.pi / 8, 0, strategy=st))
        assert np.allclose(c, 17.0, rtol=1e-12, atol=0) and np.max(np.abs(s)) < 1e-10
    K, alpha, p = 10, 0.08, 2
    x = np.zeros(51)
    x[25] = 1.0
    c, s = O.asft_components(x, O.ZERO, O.Cfg(K, math.pi / K, p, alpha=alpha, strategy=O.RECURSIVE1))
    for n in range(51):
        lag = n - 25
        if abs(lag) <= K:
            assert abs(c[n] - math.exp(-alpha * lag) * math.cos(math.pi / K * p * lag)) < 1e-9
            assert abs(s[n] - math.exp(-alpha * lag) * math.sin(math.pi / K * p * lag)) < 1e-9
        else:
            assert abs(c[n]) < 1e-10 and abs(s[n]) < 1e-10


def test_window_state_two_routes(O):
    """proj/tests/test_engine.cpp:153-165"""
    x = O.make_test_signal(O.SEEDED_NOISE, 128, 3)
    a, b = O.sliding_window_state(x, O.CLAMP, 9, math.pi / 9, 2)
    assert np.max(np.abs(a - b)) < 1e-10
    a, b = O.sliding_window_state(np.zeros(64), O.ZERO, 6, math.pi / 6, 1)
    assert np.max(np.abs(a)) == 0.0 and np.max(np.abs(b)) == 0.0


def test_real_frequency_and_validation(O):
    """proj/tests/test_engine.cpp:227-258, :328-336"""
    K, beta = 9, math.pi / 9
    x = O.make_test_signal(O.SEEDED_NOISE, 70, 13)
    a = O.sft_components(x, O.CLAMP, O.Cfg(K, beta, 3, strategy=0))
    b = O.sft_components(x, O.CLAMP, O.Cfg(K, beta, omega=beta * 3, strategy=0))
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    with pytest.raises(O.OracleInvalidArgument):
        O.sft_components(x, O.CLAMP, O.Cfg(8, math.pi / 8, omega=0.3, strategy=1))
    x = O.make_test_signal(O.SEEDED_NOISE, 64, 29)
    got = O.sft_components(x, O.CLAMP, O.Cfg(8, math.pi / 8, omega=-0.21, strategy=0))
    assert md(got, brute(x, 8, -0.21, 0.0)) < 1e-10
    x = O.make_test_signal(O.SEEDED_NOISE, 16, 1)
    with pytest.raises(O.OracleInvalidArgument):
        O.asft_components(x, O.CLAMP, O.Cfg(4, math.pi / 4, 1, strategy=1))
    with pytest.raises(O.OracleInvalidArgument):
        O.sft_components(x, O.CLAMP, O.Cfg(4, math.pi / 4, 1, alpha=0.5, strategy=1))
    with pytest.raises(O.OracleInvalidArgument):
        O.sft_components(x, O.CLAMP, O.Cfg(0, 1.0, 0, strategy=1))


def test_sliding_route_equals_kernel_integral(O):
    """proj/tests/test_engine.cpp:284-305, :321-326"""
    K = 16
    x = O.make_test_signal(O.SEEDED_NOISE, 256, 17)
    for p in range(7):
        d = O.sft_components(x, O.CLAMP, O.Cfg(K, math.pi / K, p, strategy=0))
        t = O.sft_via_sliding_sum(x, O.CLAMP, O.Cfg(K, math.pi / K, p, strategy=0))
        assert md(d, t) < 1e-10 * max(1.0, np.max(np.abs(d[0])))
    cfg = O.Cfg(K, math.pi / K, 2, alpha=0.01, strategy=0)
    assert md(O.asft_components(x, O.CLAMP, cfg), O.sft_via_sliding_sum(x, O.CLAMP, cfg)) < 1e-9
    with pytest.raises(O.OracleInvalidArgument):
        O.sft_via_sliding_sum(O.make_test_signal(O.SEEDED_NOISE, 20000, 1), O.CLAMP,
                              O.Cfg(16, math.pi / 16, 1, alpha=0.1, strategy=0))


def test_stability_probe_reproduces_reference_run(O):
    """The reference's fp32 numerics printed in proj/test_output.txt:25 (criterion 5):
    reproduced to the printed 4 digits by the restated Recursive strategies."""
    g = GOLD["stability_probe"]
    sigma = g["sigma"]
    K = math.ceil(3 * sigma)
    alpha = 2.0 * (1.0 / (2 * sigma * sigma)) * g["n0"]
    x = O.make_test_signal(O.SEEDED_NOISE, g["N"], g["seed"])
    plain = O.stability_probe(x, O.CLAMP, K, math.pi / K, 2, 0.0, O.RECURSIVE2)
    asft = O.stability_probe(x, O.CLAMP, K, math.pi / K, 2, alpha, O.RECURSIVE2)
    state = O.stability_probe(x, O.CLAMP, K, math.pi / K, 2, alpha, O.RECURSIVE1)
    assert f"{plain['max_component_error']:.3e}" == f"{g['plain_recursive2_max_component_error']:.3e}"
    assert f"{asft['max_component_error']:.3e}" == f"{g['asft_recursive2_max_component_error']:.3e}"
    assert f"{state['max_state_magnitude']:.4g}" == f"{g['asft_recursive1_max_state']:.4g}"
    bound = np.max(np.abs(x)) / (1.0 - math.exp(-alpha))
    assert f"{bound:.4g}" == str(g["state_bound"])


def test_sliding_sum_known_answers(O):
    """proj/tests/test_sliding_sum.cpp:44-131 and proj/test_output.txt:41"""
    f = np.array(GOLD["flat_basic"]["f"], dtype=np.int64)
    assert list(O.sliding_sum(f, 3)) == GOLD["flat_basic"]["h"]
    for n, L, blocked, key, val in GOLD["plan_padding"]["cases"]:
        assert O.sliding_plan(n, L, blocked)[key] == val
    g = GOLD["blocked8_trace"]
    ints = (O.make_test_signal(O.SEEDED_NOISE, g["N"], 3) * 1000).astype(np.int64)
    out, tr = O.sliding_sum(ints, g["L"], blocked=True, trace=True)
    assert len(tr) == g["rounds"] and int(tr[:, 5].sum()) == g["total_adds"]
    plan = O.sliding_plan(g["N"], g["L"], True)
    assert plan["parallel_steps"] == g["rounds"] and plan["total_adds"] == g["total_adds"]
    for n, L in ((517, 100), (64, 8), (100, 1), (100, 100), (4096, 513), (9, 9), (1, 1), (2000, 77)):
        d = (O.make_test_signal(O.SEEDED_NOISE, n, 1000 + n) * 1000).astype(np.int64)
        brute_h = np.array([d[i:i + L].sum() for i in range(n - L + 1)])
        assert np.array_equal(O.sliding_sum(d, L), brute_h)
        assert np.array_equal(O.sliding_sum(d, L, blocked=True), brute_h)
    d = (O.make_test_signal(O.SEEDED_NOISE, 1500, 7) * 1000).astype(np.int64)
    for w in (2, 8):
        assert np.array_equal(O.sliding_sum(d, 200, workers=w), O.sliding_sum(d, 200))
        assert np.array_equal(O.sliding_sum(d, 200, blocked=True, workers=w), O.sliding_sum(d, 200, blocked=True))


def test_kernel_golden_values(O):
    """proj/tests/test_kernels.cpp:14-55 (arbitrary-precision reference values)"""
    k = GOLD["kernels"]
    assert abs(O.gauss(1.0, 0.0) - k["gauss_sigma1_t0"]) <= 1e-14 * k["gauss_sigma1_t0"]
    assert abs(O.gauss(2.0, 3.0) - k["gauss_sigma2_t3"]) <= 1e-14 * k["gauss_sigma2_t3"]
    assert abs(O.gauss_dd(1.0, 0.0) - k["gauss_dd_sigma1_t0"]) <= 1e-14 * abs(k["gauss_dd_sigma1_t0"])
    assert abs(O.gauss_dd(2.0, 5.0) - k["gauss_dd_sigma2_t5"]) <= 1e-13 * k["gauss_dd_sigma2_t5"]
    m = O.morlet(60.0, 6.0, 30.0)
    assert abs(m.real - k["morlet_sigma60_xi6_t30"][0]) <= 1e-13 * abs(m.real)
    assert abs(m.imag - k["morlet_sigma60_xi6_t30"][1]) <= 1e-13 * abs(m.imag)


def test_truncated_convolution_identities(O):
    """proj/tests/test_kernels.cpp:73-95"""
    taps = np.array([O.gauss(8.0, i) for i in range(-24, 25)])
    mass = taps.sum()
    sm = O.truncated_convolution(np.ones(64), O.CLAMP, taps, -24).real
    assert np.allclose(sm[24:40], mass, rtol=1e-12, atol=0)
    imp = np.zeros(61)
    imp[30] = 1.0
    td = np.array([O.gauss_d(8.0, i) for i in range(-24, 25)])
    r = O.truncated_convolution(imp, O.ZERO, td, -24).real
    for k in range(-24, 25):
        assert abs(r[30 + k] - O.gauss_d(8.0, k)) <= 1e-14 * max(abs(O.gauss_d(8.0, k)), 1e-300)
    x = O.make_test_signal(O.SEEDED_NOISE, 100, 3)
    assert np.array_equal(O.truncated_convolution(x, 1, taps, -24, 1), O.truncated_convolution(x, 1, taps, -24, 8))
