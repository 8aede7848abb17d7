import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_11866_b200 as P
ab = sys.argv[1] if len(sys.argv) > 1 else "GDS10P6"
sg = float(sys.argv[2]) if len(sys.argv) > 2 else 8192.0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 102400
spec = P.make_transform_spec(ab, sg, 10.0 if ab.startswith("M") else 0.0, P.TransformOptions(precision=0))
xb = P.generate_signals(P.TestSignalKind.SeededNoise, n, 77, 2, P.Precision.Single)
plan = P.TransformPlan(spec, n, 2, mode="tc")
out = plan.empty_output()
plan.execute(xb, out)
torch.cuda.synchronize()
print("ok", ab, out.abs().max().item())
