"""Headline e2e path: host time per sftgpu_transform_execute_host_async call (enqueue only)
against the wall time per transform with the final synchronize, 3 pinned buffer pairs."""
import os, sys, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_11866_b200 as P
from paper_2110_11866_b200 import _abi

spec = P.make_transform_spec("MDS5P6", 8192.0, 10.0, P.TransformOptions(precision=0))
n = 102400
plan = P.TransformPlan(spec, n, 1)
xs = [torch.randn(1, n).pin_memory() for _ in range(3)]
os_ = [torch.empty(1, n, 2).pin_memory() for _ in range(3)]
lib = _abi.lib()
def call(i):
    r = lib.sftgpu_transform_execute_host_async(plan._h, C.c_void_p(xs[i % 3].data_ptr()), C.c_void_p(os_[i % 3].data_ptr()), None)
    assert r == 0
for i in range(50): call(i)
lib.sftgpu_plan_synchronize(plan._h)
for steps in (300, 1000):
    t0 = time.perf_counter()
    for i in range(steps): call(i)
    t1 = time.perf_counter()
    lib.sftgpu_plan_synchronize(plan._h)
    t2 = time.perf_counter()
    print(f"{steps} calls: enqueue {1e6*(t1-t0)/steps:.1f} us/call, wall {1e6*(t2-t0)/steps:.1f} us/transform")
