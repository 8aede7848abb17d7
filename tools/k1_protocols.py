"""Headline (config 3) step time in a CUDA graph of K back-to-back steps after a 2x-L2 flush,
isolating what makes cold steps slower than warm ones:
 fresh   : disjoint buffer pairs, outputs never touched (bench.py's protocol)
 touched : disjoint pairs, outputs zero-filled before the flush (pages touched, L2 still cold)
 noflush : as fresh but without the flush
 same    : one pair for every step (only the first step is cold)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_11866_b200 as P

spec = P.make_transform_spec("MDS5P6", 8192.0, 10.0, P.TransformOptions(precision=0))
n, K = 102400, 200
plan = P.TransformPlan(spec, n, 1)
flush = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
base = P.generate_signals(P.TestSignalKind.SeededNoise, n, 1234, 1, P.Precision.Single)


def run(kind):
    xs = [base.clone() for _ in range(K)] if kind != "same" else [base] * K
    outs = [plan.empty_output() for _ in range(K)] if kind != "same" else [plan.empty_output()] * K
    if kind == "touched":
        for o in outs:
            o.zero_()
    wx, wo = base.clone(), plan.empty_output()
    with torch.cuda.stream(s):
        for _ in range(5):
            plan.execute(wx, wo)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for k in range(K):
                plan.execute(xs[k], outs[k])
        res = []
        for rep in range(3):
            if kind != "noflush":
                flush.fill_(rep + 1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) * 1e3 / K)
            if kind == "fresh":  # later replays are no longer first-touch: rebuild
                break
    print(f"{kind:8s} per step: " + " ".join(f"{v:.2f}" for v in res) + " us")


for kind in ("fresh", "touched", "noflush", "same"):
    run(kind)
