"""Per-scale timing of the scalogram plans (single stream), to see how K1's
sequential mode behaves across sigma (warm-up overhead, chunk count)."""
import sys

sys.path.insert(0, ".")
import torch

import paper_2110_11866_b200 as P
from paper_2110_11866_b200 import scalogram as SG

n = 1 << 24
x = P.generate_signals(P.TestSignalKind.SeededNoise, n, 1234, 1, P.Precision.Single)[0]
for mode in ("seq", "lookback"):
    for sg in (16.0, 128.0, 1024.0, 4096.0, 16384.0):
        spec = SG.build_specs([sg])[0]
        p = P.TransformPlan(spec, n, 1, mode=mode)
        out = p.empty_output()
        for _ in range(3):
            p.execute(x, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            p.execute(x, out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        d = p.describe()
        print(f"{mode:8s} sigma={sg:7.0f} K={spec.half_width:6d} ms={ms:7.3f} GB/s={n*12/ms/1e6:7.1f} "
              f"chunks={d['chunks_per_signal']} ctas={d['ctas_per_launch']} warm={d['warm_tiles']}")
