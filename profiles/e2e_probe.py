import time, ctypes as C, torch, numpy as np
import paper_2110_11866_b200 as sft
from paper_2110_11866_b200._abi import lib
spec = sft.make_transform_spec("MDS5P6", 8192.0, 10.0, sft.TransformOptions(precision=0))
n = 102400
plan = sft.TransformPlan(spec, n)
xs = [torch.randn(1, n).pin_memory() for _ in range(3)]
os_ = [torch.empty(1, n, 2).pin_memory() for _ in range(3)]
st = torch.cuda.Stream()
L = lib()
def run(kind, steps=300):
    xp = [C.c_void_p(x.data_ptr()) for x in xs]; op = [C.c_void_p(o.data_ptr()) for o in os_]
    s = C.c_void_p(st.cuda_stream)
    for rep in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        for i in range(steps):
            if kind == "async_np": plan.execute_host_async(xs[i%3].numpy(), os_[i%3].numpy(), st.cuda_stream)
            elif kind == "async_raw": L.sftgpu_transform_execute_host_async(plan._h, xp[i%3], op[i%3], s)
            elif kind == "sync_raw": L.sftgpu_transform_execute_host(plan._h, xp[i%3], op[i%3], s)
            elif kind == "ctypes_only": L.sftgpu_plan_output_is_complex(plan._h)
            elif kind == "copies_only":
                with torch.cuda.stream(st):
                    d = torch.empty(1, n, device="cuda") if i == 0 else d
                    do = torch.empty(1, n, 2, device="cuda") if i == 0 else do
                    d.copy_(xs[i%3], non_blocking=True); os_[i%3].copy_(do, non_blocking=True)
        st.synchronize(); dt = (time.perf_counter() - t) / steps
    print(f"{kind:12s} {dt*1e6:8.2f} us/step")
for k in ("ctypes_only", "copies_only", "sync_raw", "async_raw", "async_np"): run(k)
