"""One K4 launch (plus a warm-up) on the config-4 spec for ncu: python tools/tc_one.py [batch] [mode]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_11866_b200 as P
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
mode = sys.argv[2] if len(sys.argv) > 2 else "tc"
spec = P.make_transform_spec("MMS5P3", 8192.0, 10.0, P.TransformOptions(precision=0))
xb = P.generate_signals(P.TestSignalKind.SeededNoise, 102400, 1234, B, P.Precision.Single)
plan = P.TransformPlan(spec, 102400, B, mode=mode)
out = plan.empty_output()
for _ in range(2):
    plan.execute(xb, out)
torch.cuda.synchronize()
print("ok", plan.describe())
