# Round-2 pass 2: GPU tests vs the compiled reference, smoke, bench both arms (cold-L2 timing).
timeout 900 python -m pytest tests/test_gpu_vs_reference.py tests/test_gpu_shipped_paths.py -q 2>&1 | tail -15 > gpurun_out/pytest_ref.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_md.json 2> gpurun_out/bench_md.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python bench.py --workload gauss_sft_fp64 --no-cpu > gpurun_out/bench_g64.json 2> gpurun_out/bench_g64.err
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
python - <<'PY' > gpurun_out/refport.txt 2>&1
import time, numpy as np, oracle as O, oracle.ref as R, os
spec = R.Spec("MDS5P6", 8192.0, 10.0, strategy=2, precision=1)
x = O.make_test_signal(3, 102400, 1234)
co, cc, so, sc = spec.morlet_coeffs(); g = 1/(2*8192.0**2); w = os.cpu_count()
def t(f, n=9):
    f(); ts=[]
    for _ in range(n):
        a=time.perf_counter(); f(); ts.append(time.perf_counter()-a)
    return sorted(ts)[n//2]*1e3
for _ in range(2):
    print("ref", t(lambda: R.apply_transform(spec, x, 1, w)), "port", t(lambda: O.morlet_direct(x, 1, spec.half_width, spec.beta, spec.n0, spec.alpha, g, 2, 1, co, cc, so, sc, w)))
PY
cat gpurun_out/pytest_ref.log gpurun_out/smoke.log gpurun_out/refport.txt; cut -c1-600 gpurun_out/bench_md.json; cut -c1-300 gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_md.err
