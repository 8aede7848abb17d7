"""K4 vs K1 over specs whose lead / trail stream offsets (lo + K) mod 4, (lo - K) mod 4
cover every value, real and complex outputs (TMA loader staging)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_11866_b200 as P
cases = [a.split(":") for a in sys.argv[1:]] or [
    ("GDS10P6", "8192", "0"), ("GDS9P6", "8192", "0"), ("GDS11P6", "8192", "0"), ("GDS8P6", "8192", "0"),
    ("MDS5P6", "8192", "10"), ("MDS6P6", "8192", "10"), ("MDS4P6", "8192", "10"), ("MDS7P6", "8192", "10"),
    ("GDS5P6", "3001", "0"), ("MDS5P6", "3001", "10")]
for ab, sg, xi in cases:
    spec = P.make_transform_spec(ab, float(sg), float(xi), P.TransformOptions(precision=0))
    n, b = 102400, 2
    xb = P.generate_signals(P.TestSignalKind.SeededNoise, n, 7, b, P.Precision.Single)
    outs = []
    for mode in ("tc", "seq"):
        plan = P.TransformPlan(spec, n, b, mode=mode)
        o = plan.empty_output()
        plan.execute(xb, o)
        torch.cuda.synchronize()
        outs.append(o.double())
    err = float((outs[0] - outs[1]).abs().max() / outs[1].abs().max())
    print(ab, sg, xi, f"rel {err:.2e}", flush=True)
