set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for w in morlet_direct gauss_sft_fp64 gauss_asft_fp32 morlet_multiply_batch scalogram; do
  timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 300 python bench.py --impl reference > gpurun_out/bench_reference.json 2>gpurun_out/bench_reference.err
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; tail -n1 gpurun_out/bench_*.json | cut -c1-400
