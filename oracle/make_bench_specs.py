"""TEST INFRASTRUCTURE ONLY: writes oracle/bench_specs.json, the coefficients of every
bench.py workload's spec as built by the compiled reference's own factory
(oracle/_ref, make_transform_spec). bench.py's reference arm falls back to this fixture
plus the restated port only where oracle/_ref is absent; it never loads the product.

    python oracle/make_bench_specs.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import oracle.ref as R  # noqa: E402

WORKLOADS = [("MDS5P6", 8192.0, 10.0), ("GDP6", 8192.0, 0.0), ("GDS10P6", 8192.0, 0.0), ("MMS5P3", 8192.0, 10.0)]


def main():
    out = {}
    for abbrev, sigma, xi in WORKLOADS:
        s = R.Spec(abbrev, sigma, xi)
        d = {"kind": s.kind, "K": s.half_width, "beta": s.beta, "n0": s.n0, "alpha": s.alpha, "sigma": s.sigma,
             "xi": s.xi, "ps": s.ps, "pd": s.pd, "max_order": s.max_order}
        if s.kind <= 2:
            a, b, dd = s.gauss_coeffs()
            d.update(a=a.tolist(), b=b.tolist(), d=dd.tolist())
        else:
            co, cc, so, sc = s.morlet_coeffs(envelope=s.kind == 4)
            d.update(cos_orders=co, cos_coeffs=[cc.real.tolist(), cc.imag.tolist()], sin_orders=so,
                     sin_coeffs=[sc.real.tolist(), sc.imag.tolist()])
        out[f"{abbrev}@{sigma:g}"] = d
    with open(os.path.join(HERE, "bench_specs.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
