# Round-2 re-entry pass: full GPU suite, smoke, bench both arms + kernel-only lines per workload.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_md.json 2> gpurun_out/bench_md.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash profiles/bench_all.sh > gpurun_out/bench_all.txt 2>&1
nproc > gpurun_out/nproc.txt
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench_all.txt; cut -c1-700 gpurun_out/bench_md.json; cut -c1-400 gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_md.err gpurun_out/bench_ref.err
