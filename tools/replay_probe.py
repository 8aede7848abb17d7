"""K7 cost split: one call with 1 or 7 orders (the serial chains run in parallel threads),
fp64 / fp32, config 1's shape and a short signal (fixed overheads)."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_11866_b200 as P

def t(n, K, no, prec, st=P.Strategy.Recursive2):
    x = P.make_test_signal(P.TestSignalKind.SeededNoise, n, 1234).samples
    cf = [P.SftConfig(K, math.pi / K, P.OrderSpec.order(p), 0.0, 0, st, prec) for p in range(no)]
    sig = P.Signal(x)
    P.components_replay(sig, cf, 0, n - 1)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); P.components_replay(sig, cf, 0, n - 1); ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3

for (n, K) in ((102400, 24576), (1000, 8)):
    for no in (1, 7):
        for prec in (P.Precision.Double, P.Precision.Single):
            print(f"n={n} K={K} orders={no} {prec.name}: {t(n, K, no, prec):.2f} ms")
print(f"Recursive1 fp64 n=102400 1 order: {t(102400, 24576, 1, P.Precision.Double, P.Strategy.Recursive1):.2f} ms")
