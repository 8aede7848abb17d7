# Round-2 closing evidence at HEAD (K4 issue order, K7 speedups): GPU tests, smoke, bench lines for every
# headline), ncu launch lists and full captures of the dominant kernels, C++ drop-in e2e.
mkdir -p gpurun_out/ev5
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/ev5/smi.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ev5/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev5/smoke.log 2>&1
for w in morlet_direct gauss_sft_fp64 gauss_asft_fp32 morlet_multiply_batch scalogram; do
  timeout 600 python bench.py --workload $w > gpurun_out/ev5/bench_$w.json 2> gpurun_out/ev5/bench_$w.err
done
timeout 600 python bench.py --impl reference > gpurun_out/ev5/bench_reference.json 2> gpurun_out/ev5/bench_reference.err
./tools/cpp_e2e 300 > gpurun_out/ev5/cpp_e2e.json 2>&1
timeout 300 python tools/replay_time.py > gpurun_out/ev5/replay_time.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev5/launches_morlet_direct.csv python bench.py --steps 20 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/ev5/launches_batch.csv python bench.py --workload morlet_multiply_batch --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/ev5/launches_scalogram.csv python bench.py --workload scalogram --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sft_scan -s 5 -c 1 -o gpurun_out/ev5/prof_morlet_direct -f python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sft_tc -s 1 -c 1 -o gpurun_out/ev5/prof_batch -f python tools/tc_one.py 4096 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sft_tc -s 2 -c 1 -o gpurun_out/ev5/prof_scalogram -f python tools/sg_one.py > /dev/null 2>&1
cat gpurun_out/ev5/pytest_gpu.log gpurun_out/ev5/smoke.log; for f in gpurun_out/ev5/bench_*.json; do echo $f; cut -c1-300 $f; done; cat gpurun_out/ev5/cpp_e2e.json gpurun_out/ev5/replay_time.json; ls -la gpurun_out/ev5 | head -40
