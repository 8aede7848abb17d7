# Round-2 re-entry check of HEAD: GPU tests, smoke, bench lines for the K4 workloads and the headline.
mkdir -p gpurun_out/r2d
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2d/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r2d/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d/smoke.log 2>&1
for w in morlet_direct morlet_multiply_batch scalogram; do
  timeout 600 python bench.py --workload $w > gpurun_out/r2d/bench_$w.json 2> gpurun_out/r2d/bench_$w.err
done
cat gpurun_out/r2d/pytest_gpu.log gpurun_out/r2d/smoke.log; for f in gpurun_out/r2d/bench_*.json; do echo $f; cut -c1-400 $f; done
