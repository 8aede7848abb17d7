import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2110_11866_b200 as sft, oracle as O
from test_gpu_transforms import oracle_transform
from conftest import rel_max
spec = sft.make_transform_spec("MMS5P3", 8192.0, 10.0, sft.TransformOptions(precision=0))
n = 102400
for off in (0.0, 1.0, 3.0):
    x = O.make_test_signal(O.SEEDED_NOISE, n, 11) + off
    xb = torch.tensor(np.stack([x, 0.5 * x]), dtype=torch.float32, device="cuda")
    xh = xb.double().cpu().numpy()
    for bnd in (0, 1):
        ref = oracle_transform(O, xh[0], bnd, spec)
        errs = []
        for mode in ("tc", "seq", "lookback"):
            plan = sft.TransformPlan(spec, n, 2, bnd, mode=mode)
            out = plan.empty_output(); plan.execute(xb, out); torch.cuda.synchronize()
            o = out.double().cpu().numpy(); v = o[..., 0] + 1j * o[..., 1]
            errs.append(rel_max(v[0], ref))
        print(f"offset {off} boundary {bnd}: tc {errs[0]:.2e} seq {errs[1]:.2e} lb {errs[2]:.2e}", flush=True)
