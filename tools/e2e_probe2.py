"""Host-path probe for the headline e2e: per-step time of (a) serial H2D+D2H copies,
(b) H2D / D2H on two streams (overlap), (c) CPU submission cost of the pipelined C-ABI
call (no sync), (d) the pipelined call end to end."""
import sys, os, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_11866_b200 as sft
from paper_2110_11866_b200._abi import lib
spec = sft.make_transform_spec("MDS5P6", 8192.0, 10.0, sft.TransformOptions(precision=0))
n = 102400
plan = sft.TransformPlan(spec, n)
xs = [torch.randn(1, n).pin_memory() for _ in range(3)]
os_ = [torch.empty(1, n, 2).pin_memory() for _ in range(3)]
d, do = torch.empty(1, n, device="cuda"), torch.empty(1, n, 2, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
L = lib()
xp = [C.c_void_p(x.data_ptr()) for x in xs]; op = [C.c_void_p(o.data_ptr()) for o in os_]
S = 300
def timeit(f):
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter(); f(); torch.cuda.synchronize()
    return (time.perf_counter() - t) / S * 1e6
def serial():
    with torch.cuda.stream(s1):
        for i in range(S):
            d.copy_(xs[i % 3], non_blocking=True); os_[i % 3].copy_(do, non_blocking=True)
def two_streams():
    for i in range(S):
        with torch.cuda.stream(s1): d.copy_(xs[i % 3], non_blocking=True)
        with torch.cuda.stream(s2): os_[i % 3].copy_(do, non_blocking=True)
def h2d_only():
    with torch.cuda.stream(s1):
        for i in range(S): d.copy_(xs[i % 3], non_blocking=True)
def d2h_only():
    with torch.cuda.stream(s1):
        for i in range(S): os_[i % 3].copy_(do, non_blocking=True)
def submit_only():
    s = C.c_void_p(s1.cuda_stream)
    t = time.perf_counter()
    for i in range(S): L.sftgpu_transform_execute_host_async(plan._h, xp[i % 3], op[i % 3], s)
    submit_only.t = (time.perf_counter() - t) / S * 1e6
def pipelined():
    s = C.c_void_p(s1.cuda_stream)
    for i in range(S): L.sftgpu_transform_execute_host_async(plan._h, xp[i % 3], op[i % 3], s)
    s1.synchronize()
def wrapper():
    with torch.cuda.stream(s1):
        for i in range(S): plan.execute_host_async(xs[i % 3].numpy(), os_[i % 3].numpy(), s1.cuda_stream)
    s1.synchronize()
for name, f in (("wrapper", wrapper), ("h2d_only", h2d_only), ("d2h_only", d2h_only), ("serial", serial), ("two_streams", two_streams),
                ("pipelined", pipelined)):
    print(f"{name:12s} {timeit(f):8.2f} us/step", flush=True)
timeit(submit_only)
print(f"submit cost  {submit_only.t:8.2f} us/step (CPU, pipelined C-ABI call)")
