"""One multi-scale K4 launch of BASELINE config 5 (128 scales, N=2^24) for ncu / traces:
python tools/sg_one.py [n_scales] [log2 n]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_11866_b200 as P
from paper_2110_11866_b200 import scalogram as SG
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 128
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 24)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
specs = SG.build_specs(SG.scale_sigmas(ns), 10.0, 6, cache=os.path.join(root, "paper_2110_11866_b200", "data",
                                                                        f"scalogram{ns}_xi10_pd6.coef"))
x = P.generate_signals(P.TestSignalKind.SeededNoise, n, 1234, 1, P.Precision.Single)[0]
sc = SG.Scalogram(n, specs)
out = sc.empty_output()
for _ in range(2):
    sc.run(x, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(3):
    sc.run(x, out)
e1.record()
torch.cuda.synchronize()
print("ok", len(sc.multi), "multi-scale launches;", e0.elapsed_time(e1) / 3, "ms")
