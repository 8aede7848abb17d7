"""The reference itself, compiled here from its own sources (oracle/ref.mk, mini-Eigen
and mini-doctest shims in oracle/ref_shim), and the restated oracle
pinned to it.

* the reference's own doctest suites (proj/tests/test_*.cpp minus test_cli.cpp) pass
  against the shim-built library;
* its acceptance suite reproduces the reference run's printed numbers
  (proj/test_output.txt) digit for digit for every library criterion (1-6);
* the restated oracle (oracle/sft_oracle.cpp, the CPU checker of every GPU test) agrees
  with the compiled reference on BASELINE configs 1-3 for every strategy and precision.
"""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
from conftest import rel_max

R = pytest.importorskip("oracle.ref")

pytestmark = pytest.mark.skipif(not R.available(), reason="reference sources and prebuilt oracle/_ref both absent")

REF_OUTPUT = "/root/reference/proj/test_output.txt"


@pytest.fixture(scope="module")
def ref():
    R.build()
    R.lib()
    return R


def test_reference_doctest_suites_pass(ref):
    res = subprocess.run([R.TESTS_BIN], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:]
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", res.stdout)
    assert m and int(m.group(1)) >= 78 and m.group(3) == "0", res.stdout[-500:]


@pytest.mark.skipif(not os.path.exists(REF_OUTPUT), reason="reference run log absent")
def test_acceptance_reproduces_reference_run_digits(ref, tmp_path):
    """Criteria 1-6 print fitted-kernel RMSEs (Table 1), the truncation baseline, the
    fitted-kernel exactness over 1500 runs, the sliding-sum trees, the fp32 numerics and
    the Morlet method comparison; every line must equal the reference run's line."""
    res = subprocess.run([R.ACCEPTANCE_BIN], capture_output=True, text=True, timeout=900, cwd=str(tmp_path))
    ours = res.stdout.splitlines()
    with open(REF_OUTPUT) as f:
        theirs = f.read().splitlines()

    def lines(src):
        keep = []
        for ln in src:
            s = ln.strip()
            if re.match(r"(SFT|ASFT) +P=", s) or re.match(r"(PASS|FAIL) +criterion [1-6]:", s):
                keep.append(re.sub(r"; [0-9.]+ s;", ";", s))  # criterion 1 prints its own wall time
        return keep

    a, b = lines(ours), lines(theirs)
    assert len(b) == 16 and a == b


def _x(n, seed=1234, f32=False):
    x = R.make_test_signal(3, n, seed)
    assert np.array_equal(x, O.make_test_signal(O.SEEDED_NOISE, n, seed))
    return x.astype(np.float32).astype(np.float64) if f32 else x


def _oracle_of(spec, x, strategy, precision):
    """The restated oracle on the reference spec's own coefficients."""
    gamma = 1.0 / (2.0 * spec.sigma ** 2)
    if spec.kind <= 2:
        a, b, d = spec.gauss_coeffs()
        return O.gauss_smooth(x, 1, spec.kind, spec.half_width, spec.beta, spec.n0, spec.alpha, gamma, strategy,
                              precision, a, b, d, 8).astype(np.complex128)
    if spec.kind == 3:
        co, cc, so, sc = spec.morlet_coeffs()
        return O.morlet_direct(x, 1, spec.half_width, spec.beta, spec.n0, spec.alpha, gamma, strategy, precision,
                               co, cc, so, sc, 8)
    co, cc, _, _ = spec.morlet_coeffs(envelope=True)
    return O.morlet_multiply(x, 1, spec.half_width, spec.beta, spec.n0, spec.alpha, spec.sigma, spec.xi, strategy,
                             precision, cc.real, 8)


@pytest.mark.parametrize("abbrev,sigma,xi,f32", [("GDP6", 8192.0, 0.0, False),    # config 1
                                                 ("GDS10P6", 512.0, 0.0, True),   # config 2
                                                 ("MDS5P6", 8192.0, 10.0, True),  # config 3
                                                 ("MMS5P3", 300.0, 10.0, True)])  # config 4 spec, shorter sigma
@pytest.mark.parametrize("strategy", [0, 2])
@pytest.mark.parametrize("precision", [0, 1])
def test_oracle_restatement_matches_compiled_reference(ref, abbrev, sigma, xi, f32, strategy, precision):
    """Same input, same spec (the reference's own coefficients): fp64 agrees to rounding
    (<= 1e-13), fp32 bit for bit up to the reference's own reduction order (<= 1e-6:
    both run the reference's fp32 loops, which random-walk at this size)."""
    spec = R.Spec(abbrev, sigma, xi, strategy=strategy, precision=precision)
    x = _x(102400, f32=f32)
    got = R.apply_transform(spec, x, 1, 8)
    ora = _oracle_of(spec, x, strategy, precision)
    tol = 1e-13 if precision == 1 else 1e-6
    assert rel_max(ora, got) <= tol


def test_reference_spec_matches_product_host_fit(ref):
    """The product's host precompute (csrc/host_fit.cpp) and the compiled reference build
    the same spec for the headline config: P_S, K, beta, n0 and coefficients."""
    import paper_2110_11866_b200 as P

    ours = P.make_transform_spec("MDS5P6", 8192.0, 10.0, P.TransformOptions(precision=0))
    theirs = R.Spec("MDS5P6", 8192.0, 10.0, precision=0)
    assert (ours.ps, ours.half_width, ours.n0) == (theirs.ps, theirs.half_width, theirs.n0)
    assert ours.beta == theirs.beta and ours.alpha == theirs.alpha
    co, cc, so, sc = theirs.morlet_coeffs()
    mc = ours.morlet_coeffs
    assert list(mc.cos_orders) == co and list(mc.sin_orders) == so
    assert rel_max(mc.cos_coeffs, cc) < 1e-9 and rel_max(mc.sin_coeffs, sc) < 1e-9
    assert abs(ours.kernel_rmse_percent - theirs.kernel_rmse_percent) < 1e-9 * theirs.kernel_rmse_percent


def test_sliding_sum_route_oracle_vs_reference(ref):
    x = _x(3000, 5)
    K, beta = 40, np.pi / 40
    c, s = R.components(x, 1, K, beta, p=3, strategy=0, sliding_route=True)
    oc, os_ = O.sft_via_sliding_sum(x, 1, O.Cfg(K, beta, 3, None, 0.0, O.KERNEL_INTEGRAL, O.DOUBLE))
    assert rel_max(oc - 1j * os_, c - 1j * s) < 1e-13
