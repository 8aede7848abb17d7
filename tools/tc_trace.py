"""Per-tile pipeline trace of K4 (CTA 0); needs a library built with the trace hooks:
SFTGPU_EXTRA_NVCC_FLAGS="-DTCK_TRACE=1" python paper_2110_11866_b200/build.py
(then rebuild without it). Columns: clocks: clocks of loader issue / xfull, GEMM1 issue,
scan start / SS ready, GEMM2 issue, epilogue start / end, relative to the first event."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_11866_b200 as P
from paper_2110_11866_b200 import _abi
B = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1] != "sg" else 1184
if len(sys.argv) > 1 and sys.argv[1] == "sg":  # BASELINE config 5: multi-scale plan, 128 scales, N=2^24
    from paper_2110_11866_b200 import scalogram as SG
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    specs = SG.build_specs(SG.scale_sigmas(128), 10.0, 6,
                           cache=os.path.join(root, "paper_2110_11866_b200", "data", "scalogram128_xi10_pd6.coef"))
    xb = P.generate_signals(P.TestSignalKind.SeededNoise, 1 << 24, 1234, 1, P.Precision.Single)[0]
    plan = P.MultiScalePlan(specs, 1 << 24)
else:
    spec = P.make_transform_spec("MMS5P3", 8192.0, 10.0, P.TransformOptions(precision=0))
    xb = P.generate_signals(P.TestSignalKind.SeededNoise, 102400, 1234, B, P.Precision.Single)
    plan = P.TransformPlan(spec, 102400, B, mode="tc")
out = plan.empty_output()
plan.execute(xb, out)
tr = torch.zeros(64 * 16, dtype=torch.int64, device="cuda")
lib = _abi.lib()
lib.sftgpu_debug_set_tc_trace.argtypes = [C.c_void_p]
lib.sftgpu_debug_set_tc_trace(C.c_void_p(tr.data_ptr()))
plan.execute(xb, out)
torch.cuda.synchronize()
lib.sftgpu_debug_set_tc_trace(None)
t = tr.cpu().numpy().reshape(64, 16).astype(np.int64)
t0 = t[t > 0].min()
names = ["ld_go", "mma_go", "g1_iss", "scan_g1", "st_tmem", "g2_iss", "epi_g2", "epi_end", "ph1", "ph2", "ld_full", "trail_iss", "trail_done", "tma_iss", "e_rel", "trail_full"]
print("tile " + " ".join(f"{n:>8s}" for n in names))
for g in range(64):
    print(f"{g:4d} " + " ".join(f"{(v - t0) if v > 0 else -1:8d}" for v in t[g]))
