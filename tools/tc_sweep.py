"""Randomised K4-vs-K1 agreement sweep over specs and geometries (kinds, sigma, xi, n0,
orders, n, batch, boundary, output ranges): prints the worst relative difference per case
and fails if any exceeds 1e-5."""
import sys, os, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_11866_b200 as sft

def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(1e-30, np.max(np.abs(b))))

rng = random.Random(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
cases = int(sys.argv[2]) if len(sys.argv) > 2 else 40
worst = 0.0
for c in range(cases):
    fam = rng.choice(["GD", "MD", "MM", "GD"])
    asft = rng.random() < 0.6
    kind = fam + ("S" if asft else "P")
    sigma = rng.choice([20.0, 50.0, 200.0, 700.0, 1500.0, 4000.0, 8192.0])
    n0 = min(rng.choice([0, 1, 3, 5, 10]), int(sigma // 4))
    xi = rng.choice([6.0, 8.0, 10.0, 12.0])
    order = rng.choice([3, 4, 5, 6]) if kind.startswith("G") else rng.choice([3, 5, 6])
    if kind.startswith("MM"):
        order = rng.choice([2, 3])
    ab = f"{fam}S{n0}P{order}" if asft else f"{fam}P{order}"
    try:
        spec = sft.make_transform_spec(ab, sigma, xi if kind.startswith("M") else 0.0,
                                       sft.TransformOptions(precision=0))
    except ValueError as e:
        continue
    n = rng.choice([5000, 12345, 40000, 102400, 300001])
    batch = rng.choice([1, 2, 3, 7])
    bnd = rng.choice([0, 1])
    rngd = None
    if rng.random() < 0.3:
        b0 = rng.randrange(0, n // 2)
        rngd = (b0, rng.randrange(1, n - b0))
    xb = sft.generate_signals(sft.TestSignalKind.SeededNoise, n, rng.randrange(1000), batch, sft.Precision.Single)
    if rng.random() < 0.3:
        xb = xb + 1.0
    outs = {}
    for mode in ("tc", "seq"):
        try:
            plan = sft.TransformPlan(spec, n, batch, bnd, rngd, mode=mode)
        except ValueError as e:
            outs = None
            break
        o = plan.empty_output()
        plan.execute(xb, o)
        torch.cuda.synchronize()
        oh = o.double().cpu().numpy()
        outs[mode] = oh[..., 0] + 1j * oh[..., 1] if plan.complex_out else oh
    if outs is None:
        print(f"{ab:10s} sigma={sigma:6.0f} skipped (not K4-eligible)")
        continue
    e = rel(outs["tc"], outs["seq"])
    worst = max(worst, e)
    print(f"{ab:10s} sigma={sigma:6.0f} xi={xi:4.0f} n={n:6d} B={batch} bnd={bnd} range={rngd} tc-vs-k1 {e:.2e}", flush=True)
print("worst", worst)
sys.exit(0 if worst < 1e-5 else 1)
