"""GPU: the reference-signature entry points (gauss_smooth / morlet_direct_transform /
morlet_multiply_transform / apply_transform, proj/include/sft/transforms.hpp:86-102) go
through sftgpu_transform_oneshot, whose plans are cached inside the library: repeated
calls reuse one plan and give the plan path's result bit for bit; concurrent callers are
serialised per cached plan."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _plan_path(sft, sig, spec):
    import torch

    plan = sft.TransformPlan(spec, sig.size(), 1, sig.boundary)
    x = torch.from_numpy(sig.samples).to(device="cuda", dtype=plan.dtype())
    out = plan.empty_output()
    plan.execute(x, out)
    torch.cuda.synchronize()
    o = out[0].double().cpu().numpy()
    return (o[:, 0] + 1j * o[:, 1]) if plan.complex_out else o.astype(np.complex128)


@pytest.mark.parametrize("abbrev,sigma,xi,prec", [("MDS5P6", 300.0, 10.0, 0), ("GDS4P6", 200.0, 0.0, 0),
                                                  ("GDP6", 150.0, 0.0, 1), ("MMS5P3", 400.0, 10.0, 0)])
def test_oneshot_matches_plan_path_and_reuses(sft, abbrev, sigma, xi, prec):
    spec = sft.make_transform_spec(abbrev, sigma, xi, sft.TransformOptions(precision=prec))
    sig = sft.make_test_signal(sft.TestSignalKind.SeededNoise, 30001, 17)
    ref = _plan_path(sft, sig, spec)
    for _ in range(3):  # cached plan reused: identical results every time
        got = sft.apply_transform(sig, spec).values
        assert np.array_equal(got, ref)


def test_oneshot_concurrent_callers(sft):
    specs = [sft.make_transform_spec("MDS3P6", 64.0 * (i + 1), 8.0, sft.TransformOptions(precision=0))
             for i in range(3)]
    sigs = [sft.make_test_signal(sft.TestSignalKind.SeededNoise, 20000 + 7 * i, 100 + i) for i in range(3)]
    refs = [sft.morlet_direct_transform(s, sp).values for s, sp in zip(sigs, specs)]
    errors = []

    def worker(k):
        try:
            for _ in range(10):
                i = k % 3
                v = sft.morlet_direct_transform(sigs[i], specs[i]).values
                if not np.array_equal(v, refs[i]):
                    errors.append(k)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors
