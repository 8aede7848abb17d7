"""K4 config-4 time vs the signal / output row padding (tests whether the 409.6 KB
lockstep stride between the CTAs' signals maps unevenly onto HBM channels)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_11866_b200 as P
B, n = 4096, 102400
spec = P.make_transform_spec("MMS5P3", 8192.0, 10.0, P.TransformOptions(precision=0))
plan = P.TransformPlan(spec, n, B, mode="tc")
for pad in [int(a) for a in sys.argv[1:]] or [0, 32, 96, 256, 1056, 4128, 12320]:
    lx = n + pad
    x = torch.randn(B * lx, device="cuda")
    out = torch.empty(B * lx * 2, device="cuda")
    for _ in range(2):
        plan.execute(x, out, ld_x=lx, ld_out=lx)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        plan.execute(x, out, ld_x=lx, ld_out=lx)
    e1.record()
    torch.cuda.synchronize()
    print(f"pad {pad:6d}: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
    del x, out
