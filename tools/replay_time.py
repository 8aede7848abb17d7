"""K7 timing: the reference's Recursive2 fp64 replayed on the GPU at BASELINE config 1's
shape (N=102400, K=24576, orders 0..6, one call, host buffers in and out), beside the
compiled reference's components_over for one order when it is shipped (oracle/_ref)."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2110_11866_b200 as P

K, n = 24576, 102400
x = P.make_test_signal(P.TestSignalKind.SeededNoise, n, 1234).samples
cfgs = [P.SftConfig(K, math.pi / K, P.OrderSpec.order(p), 0.0, 0, P.Strategy.Recursive2, P.Precision.Double)
        for p in range(7)]
sig = P.Signal(x)
P.components_replay(sig, cfgs, 0, n - 1)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    P.components_replay(sig, cfgs, 0, n - 1)
    ts.append(time.perf_counter() - t0)
res = {"what": "components_replay Recursive2 fp64, 7 orders, N=102400, K=24576 (host in/out)",
       "gpu_ms_median": sorted(ts)[2] * 1e3}
try:
    import oracle.ref as R
    if R.available():
        R.lib()
        t0 = time.perf_counter()
        R.components(x, 1, K, math.pi / K, p=3)
        res["compiled_reference_ms_one_order"] = (time.perf_counter() - t0) * 1e3
except Exception as e:  # noqa: BLE001
    res["reference"] = str(e)
print(json.dumps(res))
