"""K7: the reference's recursive strategies (proj/src/engine.cpp:53-120) replayed on the GPU
with the reference's rounding. The bar is bit-identity: against the CPU restatement in
oracle/ (same operation order, no FMA contraction) and, where it is shipped, against the
reference itself compiled from its own sources (oracle/_ref). Cases follow the reference's
engine tests (proj/tests/test_engine.cpp): both recursions, both window forms, plain and
attenuated, Zero / Clamp boundaries, signed output ranges past both ends, fp32 and fp64,
tuned (non-pi/K) beta, and config 1's full shape (N=102400, K=24576, orders 0..6)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cfg(sft, K, beta, p, alpha, st, prec, w2k1=False):
    return sft.SftConfig(K, beta, sft.OrderSpec.order(p), alpha, 0, st, prec, w2k1)


def _same(got, ref):
    assert got.shape == ref.shape
    assert np.array_equal(got.view(np.int64), ref.view(np.int64)), \
        f"not bit-identical: max |d| = {np.max(np.abs(got - ref)):.3e}"


CASES = [
    # K, beta factor, p, alpha, strategy, precision, 2K+1 window, boundary, lo, hi
    (8, 1.0, 3, 0.0, 1, 1, False, 1, 0, 63),
    (8, 1.0, 3, 0.0, 2, 1, False, 1, 0, 63),
    (8, 1.07, 3, 0.0, 2, 1, True, 0, -20, 90),
    (8, 1.0, 2, 0.05, 1, 1, False, 0, 0, 63),
    (8, 1.0, 2, 0.05, 2, 1, True, 1, -5, 70),
    (12, 1.0, 3, 0.0, 1, 0, False, 1, 0, 199),
    (12, 1.0, 3, 0.0, 2, 0, False, 0, 0, 199),
    (40, 1.0, 0, 0.0, 2, 1, False, 1, 0, 999),
    (300, 1.0, 5, 1e-4, 2, 0, False, 1, -17, 4000),
    (300, 1.0, 5, 1e-4, 1, 1, True, 1, 0, 4095),
]


@pytest.mark.parametrize("K,bf,p,alpha,st,prec,w2k1,boundary,lo,hi", CASES)
def test_replay_bit_identical_to_oracle(sft, O, K, bf, p, alpha, st, prec, w2k1, boundary, lo, hi):
    x = O.make_test_signal(O.SEEDED_NOISE, 4096 if K == 300 else 64 if K == 8 else 200 if K == 12 else 1000, 7)
    sig = sft.Signal(x, sft.BoundaryPolicy(boundary))
    beta = bf * math.pi / K
    got = sft.components_over(sig, _cfg(sft, K, beta, p, alpha, st, prec, w2k1), lo, hi)
    rc, rs = O.components_over(x, boundary, O.Cfg(K, beta, p, alpha=alpha, strategy=st, precision=prec,
                                                  window_2k1=w2k1), lo, hi)
    _same(got.c, rc)
    _same(got.s, rs)


def test_replay_several_orders_one_call(sft, O):
    K = 64
    x = O.make_test_signal(O.SEEDED_NOISE, 2000, 3)
    cfgs = [_cfg(sft, K, math.pi / K, p, 0.0, 1 + (p & 1), p & 1) for p in range(7)]
    c, s = sft.components_replay(sft.Signal(x), cfgs, -K, 2000 + K)
    for p, cf in enumerate(cfgs):
        rc, rs = O.components_over(x, 1, O.Cfg(K, math.pi / K, p, strategy=int(cf.strategy),
                                               precision=int(cf.precision)), -K, 2000 + K)
        _same(c[p], rc)
        _same(s[p], rs)


def test_replay_config1_full_shape(sft, O):
    """BASELINE config 1 (GDP6, N=102400, K=24576) with the reference's default strategy:
    all seven orders bit-identical to the reference's Recursive2 arithmetic."""
    K, n = 24576, 102400
    x = O.make_test_signal(O.SEEDED_NOISE, n, 1234)
    cfgs = [_cfg(sft, K, math.pi / K, p, 0.0, 2, 1) for p in range(7)]
    c, s = sft.components_replay(sft.Signal(x), cfgs, 0, n - 1)
    for p in (0, 3, 6):
        rc, rs = O.components_over(x, 1, O.Cfg(K, math.pi / K, p), 0, n - 1)
        _same(c[p], rc)
        _same(s[p], rs)


def test_replay_vs_compiled_reference(sft, O):
    R = pytest.importorskip("oracle.ref")
    if not R.available():
        pytest.skip("compiled reference (oracle/_ref) not shipped")
    R.lib()
    x = O.make_test_signal(O.SEEDED_NOISE, 3000, 11)
    for (K, p, alpha, st, prec, w2k1, boundary, lo, hi) in [
        (50, 3, 0.0, 2, 1, False, 1, 0, 2999),
        (50, 3, 0.0, 1, 1, True, 0, -30, 3100),
        (50, 2, 0.01, 2, 0, False, 1, 0, 2999),
        (200, 4, 0.0, 2, 0, False, 1, -7, 2992),
    ]:
        beta = math.pi / K
        got = sft.components_over(sft.Signal(x, sft.BoundaryPolicy(boundary)),
                                  _cfg(sft, K, beta, p, alpha, st, prec, w2k1), lo, hi)
        rc, rs = R.components(x, boundary, K, beta, p=p, alpha=alpha, strategy=st, precision=prec,
                              window_2k1=w2k1, lo=lo, hi=hi)
        _same(got.c, rc)
        _same(got.s, rs)


def test_replay_fast_path_is_the_window_recurrence(sft, O):
    """exact=False runs the same config on K1: within the reference's own double-precision
    tolerance of the replay (proj/tests/test_engine.cpp:80-116)."""
    K = 32
    x = O.make_test_signal(O.SEEDED_NOISE, 500, 5)
    cf = _cfg(sft, K, math.pi / K, 2, 0.0, 2, 1)
    a = sft.sft_components(sft.Signal(x), cf)
    b = sft.sft_components(sft.Signal(x), cf, exact=False)
    assert np.max(np.abs(a.c - b.c)) < 1e-10 and np.max(np.abs(a.s - b.s)) < 1e-10


def test_replay_errors(sft):
    x = sft.Signal(np.ones(32))
    with pytest.raises(ValueError, match="alpha must be 0"):
        sft.sft_components(x, _cfg(sft, 4, math.pi / 4, 1, 0.1, 2, 1))
    with pytest.raises(ValueError, match="alpha must be > 0"):
        sft.asft_components(x, _cfg(sft, 4, math.pi / 4, 1, 0.0, 1, 1))
    with pytest.raises(ValueError, match="empty range"):
        sft.components_over(x, _cfg(sft, 4, math.pi / 4, 1, 0.0, 2, 1), 5, 4)
    with pytest.raises(ValueError, match="recursive strategies"):
        sft.components_replay(x, [_cfg(sft, 4, math.pi / 4, 1, 0.0, 0, 1)], 0, 31)
    with pytest.raises(ValueError, match="K must be >= 1"):
        sft.components_replay(x, [_cfg(sft, 0, math.pi / 4, 1, 0.0, 2, 1)], 0, 31)


def test_replay_peak_state_and_stability_probe(sft, O):
    """stability_probe on a recursive strategy reports the reference's max_state (the peak
    |filter state| of the fp32 recurrence, engine.cpp:101) and honours the bound of
    proj/tests/test_engine.cpp:305-317."""
    sigma = 32.0
    alpha = 2.0 * (1.0 / (2.0 * sigma * sigma)) * 4.0
    K = int(3 * sigma)
    x = O.make_test_signal(O.SEEDED_NOISE, 4000, 3)
    cf = _cfg(sft, K, math.pi / K, 2, alpha, 1, 0)
    rep = sft.stability_probe(sft.Signal(x), cf)
    bound = np.max(np.abs(x)) / (1.0 - math.exp(-alpha))
    assert rep.max_state_magnitude <= bound
    assert rep.max_component_error < 1e-2
    _, _, ms = O.components_over(x, 1, O.Cfg(K, math.pi / K, 2, alpha=alpha, strategy=1, precision=0), 0, 3999,
                                 want_state=True)
    assert abs(rep.max_state_magnitude - ms) <= 1e-6 * ms
