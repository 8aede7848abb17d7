"""Per-tile phase timeline of K1 LB (the headline path: one signal, one tile per CTA);
needs a library built with the trace hooks, e.g. into a side copy used via SFTGPU_LIB:
SFTGPU_EXTRA_NVCC_FLAGS="-DSFTK_TRACE=1" python paper_2110_11866_b200/build.py
Phases (globaltimer ns, relative to the earliest CTA entry): entry, ticket, staged,
published, carry (window carry ready), done. Prints per-phase min / median / max over
tiles and the per-tile rows."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_11866_b200 as P
from paper_2110_11866_b200 import _abi

abbrev = sys.argv[1] if len(sys.argv) > 1 else "MDS5P6"
sigma = float(sys.argv[2]) if len(sys.argv) > 2 else 8192.0
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # 0 fp32, 1 fp64
spec = P.make_transform_spec(abbrev, sigma, 10.0 if abbrev[0] == "M" else 0.0, P.TransformOptions(precision=prec))
xb = P.generate_signals(P.TestSignalKind.SeededNoise, 102400, 1234, 1, P.Precision.Double if prec else P.Precision.Single)
plan = P.TransformPlan(spec, 102400, 1)
out = plan.empty_output()
tiles = plan.describe()["ctas_per_launch"]
tr = torch.zeros(tiles * 8, dtype=torch.int64, device="cuda")
lib = _abi.lib()
lib.sftgpu_debug_set_scan_trace.argtypes = [C.c_void_p]
for _ in range(20):
    plan.execute(xb, out)
cold = "cold" in sys.argv  # fresh input/output buffers and 2x L2 written before the traced run
if cold:
    xb = xb.clone()
    out = plan.empty_output()
    torch.empty(2 * 126 * 2**20 // 4, dtype=torch.int32, device="cuda").fill_(1)
lib.sftgpu_debug_set_scan_trace(C.c_void_p(tr.data_ptr()))
plan.execute(xb, out)
torch.cuda.synchronize()
lib.sftgpu_debug_set_scan_trace(None)
t = tr.cpu().numpy().reshape(tiles, 8).astype(np.int64)
used = t[:, 0] > 0
t = t[used]
t0 = t[:, 0].min()
r = np.where(t > 0, t - t0, -1)
names = ["entry", "ticket", "staged", "publish", "carry", "done", "lead_sum", "carry_go"]
print(f"{abbrev} sigma={sigma}: {len(t)} tiles, span {r.max() / 1000:.2f} us")
for k, n in enumerate(names):
    v = r[:, k][r[:, k] >= 0]
    if len(v):
        print(f"  {n:8s} min {v.min() / 1000:6.2f}  med {np.median(v) / 1000:6.2f}  max {v.max() / 1000:6.2f} us")
print("tile " + " ".join(f"{n:>8s}" for n in names))
for g in range(len(r)):
    print(f"{g:4d} " + " ".join(f"{v / 1000:8.2f}" if v >= 0 else "       -" for v in r[g]))
