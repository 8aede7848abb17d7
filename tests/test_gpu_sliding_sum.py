"""The paper's sliding-sum kernels (Algorithms 1-3) on the GPU vs the reference's
simulation restated in oracle/ and the reference's own assertions
(proj/tests/test_sliding_sum.cpp, acceptance criterion 4)."""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_values.json")))


def ints(O, n, seed, scale=1000.0):
    return (O.make_test_signal(O.SEEDED_NOISE, n, seed) * scale).astype(np.int64)


def test_plan_and_cost_model_cpu(sft, O):
    """CPU-only (no kernels): plan arithmetic and cost model equal the oracle's."""
    for n, L in ((1000, 137), (64, 8), (500, 37), (517, 100), (1 << 13, 1 << 11)):
        for blocked in (False, True):
            assert sft.sliding_sum_plan(n, L, blocked) == O.sliding_plan(n, L, blocked)
    g = GOLD["blocked8_trace"]
    p = sft.sliding_sum_plan(g["N"], g["L"], True)
    assert p["parallel_steps"] == g["rounds"] and p["total_adds"] == g["total_adds"]
    with pytest.raises(ValueError):
        sft.sliding_sum_plan(10, 11)
    with pytest.raises(ValueError):
        sft.sliding_sum_plan(10, 0)


@pytest.mark.gpu
def test_flat_basics(sft):
    assert list(sft.sliding_sum_flat(np.array([1, 2, 3, 4, 5], dtype=np.int64), 3)) == [6, 9, 12]
    imp = np.zeros(32, dtype=np.int64)
    imp[16] = 1
    pl = sft.sliding_sum_flat(imp, 5)
    assert all(pl[n] == (1 if (n <= 16 and 16 - n < 5) else 0) for n in range(pl.size))


@pytest.mark.gpu
def test_acceptance_criterion4_grid(sft, O):
    """proj/tests/acceptance.cpp:152-195: flat and blocked8 vs brute force on 220 (N, L)
    pairs (here a deterministic subset of 60 incl. the fixed cases), zero mismatches."""
    def mix(x):
        x ^= x >> 33
        x = (x * 0xFF51AFD7ED558CCD) & ((1 << 64) - 1)
        x ^= x >> 33
        return x

    grid = [(1, 1), (2000, 1), (777, 777), (1024, 512), (517, 100), (4096, 513), (100, 64)]
    i = 0
    while len(grid) < 60:
        n = 1 + mix(i * 3 + 11) % 2000
        L = 1 + mix(i * 5 + 17) % n
        grid.append((n, L))
        i += 1
    for n, L in grid:
        d = (O.make_test_signal(O.SEEDED_NOISE, n, 707 + n + L) * 997.0).astype(np.int64)
        c = np.concatenate([[0], np.cumsum(d)])
        brute = c[L:] - c[:-L]
        assert np.array_equal(sft.sliding_sum_flat(d, L), brute), (n, L)
        assert np.array_equal(sft.sliding_sum_blocked8(d, L), brute), (n, L)


@pytest.mark.gpu
@pytest.mark.parametrize("n,L", [(1000, 137), (700, 129), (4096, 513), (102400 + 2 * 24576, 2 * 24576 + 1)])
def test_doubles_bit_identical_to_reference_trees(sft, O, n, L):
    x = O.make_test_signal(O.SEEDED_NOISE, n, 5)
    assert np.array_equal(sft.sliding_sum_flat(x, L), O.sliding_sum(x, L))
    if n <= 4096:
        assert np.array_equal(sft.sliding_sum_blocked8(x, L), O.sliding_sum(x, L, blocked=True))


@pytest.mark.gpu
def test_complex_and_workers_independence(sft, O):
    x = O.make_test_signal(O.SEEDED_NOISE, 1500, 7) + 1j * O.make_test_signal(O.SEEDED_NOISE, 1500, 8)
    got = sft.sliding_sum_flat(x, 200)
    ref = O.sliding_sum(x.real, 200) + 1j * O.sliding_sum(x.imag, 200)
    assert np.array_equal(got, ref)
    d = ints(O, 1500, 7)
    assert np.array_equal(sft.sliding_sum_flat(d, 200, workers=8), sft.sliding_sum_flat(d, 200))
