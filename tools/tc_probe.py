"""A/B of K4 (tensor cores) vs K1 (CUDA cores) on the config-4 shape: errors vs the fp64
oracle on sample rows, and kernel time with CUDA events (L2-cold: 5 GB working set)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_11866_b200 as P
import oracle as O
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_transforms import oracle_transform

def rel(a, b): return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
cases = [("MMS5P3", 8192.0, 10.0, 4096), ("MDS5P6", 8192.0, 10.0, 4096), ("GDS10P6", 8192.0, 0.0, 4096)]
if len(sys.argv) > 1: cases = cases[:int(sys.argv[1])]
for ab, sg, xi, B in cases:
    spec = P.make_transform_spec(ab, sg, xi, P.TransformOptions(precision=0))
    n = 102400
    xb = P.generate_signals(P.TestSignalKind.SeededNoise, n, 1234, B, P.Precision.Single)
    res = {}
    for mode in ("tc", "seq"):
        plan = P.TransformPlan(spec, n, B, mode=mode)
        out = plan.empty_output()
        for _ in range(3): plan.execute(xb, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): plan.execute(xb, out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        oh = out[:4].double().cpu().numpy()
        vals = oh[..., 0] + 1j * oh[..., 1] if plan.complex_out else oh
        res[mode] = (ms, vals)
    xh = xb[:4].double().cpu().numpy()
    errs = [rel(res["tc"][1][b], oracle_transform(O, xh[b], 1, spec)) for b in (0, 3)]
    bytes_ = B * n * (12 if res["tc"][1].dtype == np.complex128 else 8)
    print(f"{ab} B={B}: tc {res['tc'][0]:.3f} ms ({bytes_/res['tc'][0]/1e6:.0f} GB/s)  seq {res['seq'][0]:.3f} ms  "
          f"tc-vs-oracle {max(errs):.2e}  tc-vs-seq {rel(res['tc'][1], res['seq'][1]):.2e}", flush=True)
