"""Headline (config 3) K1 step time under three L2/TLB protocols, device-timed:
(a) disjoint never-touched buffer pairs per step, one flush before a graph of K steps (bench.py);
(b) one buffer pair, 2x L2 flushed before every step, events around each step only;
(c) one buffer pair, back-to-back (L2-warm; not a valid bench number, for reference)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_11866_b200 as P

spec = P.make_transform_spec("MDS5P6", 8192.0, 10.0, P.TransformOptions(precision=0))
n = 102400
plan = P.TransformPlan(spec, n, 1)
L2 = 126 * 2**20
flush = torch.empty(2 * L2 // 4, dtype=torch.int32, device="cuda")
K = 200
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    x = P.generate_signals(P.TestSignalKind.SeededNoise, n, 1234, 1, P.Precision.Single)
    o = plan.empty_output()
    for _ in range(20): plan.execute(x, o)
    # (b)
    ts = []
    for k in range(K):
        flush.fill_(k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); plan.execute(x, o); e1.record(s)
        ts.append((e0, e1))
    s.synchronize()
    b = sorted(a.elapsed_time(c) * 1e3 for a, c in ts)
    # (b') same with a graph of one step per replay
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.execute(x, o)
    g.replay(); s.synchronize()
    ts = []
    for k in range(K):
        flush.fill_(k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); g.replay(); e1.record(s)
        ts.append((e0, e1))
    s.synchronize()
    bg = sorted(a.elapsed_time(c) * 1e3 for a, c in ts)
    # (c) warm back-to-back graph of K
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=s):
        for _ in range(K): plan.execute(x, o)
    g2.replay(); s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); g2.replay(); e1.record(s); s.synchronize()
    c = e0.elapsed_time(e1) * 1e3 / K
    # (d) flush-kernel between steps inside one graph: time(graph with flushes) - time(flushes only)
    small = torch.empty(2 * L2 // 4, dtype=torch.int32, device="cuda")
    g3, g4 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    KK = 50
    with torch.cuda.graph(g3, stream=s):
        for k in range(KK): small.fill_(k); plan.execute(x, o)
    with torch.cuda.graph(g4, stream=s):
        for k in range(KK): small.fill_(k)
    for gg in (g3, g4): gg.replay()
    s.synchronize()
    r = []
    for gg in (g3, g4, g3, g4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); gg.replay(); e1.record(s); s.synchronize(); r.append(e0.elapsed_time(e1) * 1e3 / KK)
print(f"(b) per-step flush, eager launch: median {b[K//2]:.2f} us  p10 {b[K//10]:.2f}  p90 {b[9*K//10]:.2f}")
print(f"(b') per-step flush, 1-step graph: median {bg[K//2]:.2f} us  p10 {bg[K//10]:.2f}  p90 {bg[9*K//10]:.2f}")
print(f"(c) warm back-to-back graph: {c:.2f} us")
print(f"(d) graph flush+step minus flush-only: {(r[0]-r[1]):.2f} / {(r[2]-r[3]):.2f} us")
