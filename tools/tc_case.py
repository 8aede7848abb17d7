"""Run one K4 case (argv: abbrev sigma xi n batch) and print its error vs the CUDA-core path."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_11866_b200 as P
ab, sg, xi, n, b = sys.argv[1], float(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
spec = P.make_transform_spec(ab, sg, xi, P.TransformOptions(precision=0))
xb = P.generate_signals(P.TestSignalKind.SeededNoise, n, 77, b, P.Precision.Single)
outs = []
for mode in ("tc", "seq"):
    plan = P.TransformPlan(spec, n, b, mode=mode)
    o = plan.empty_output()
    plan.execute(xb, o)
    torch.cuda.synchronize()
    outs.append(o)
d = (outs[0] - outs[1]).abs().max().item() / outs[1].abs().max().item()
print(ab, sg, n, b, "rel", d, flush=True)
