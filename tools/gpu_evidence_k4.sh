# K4 evidence refresh: GPU tests, config 4/5 bench lines, launch lists, ncu full captures.
mkdir -p gpurun_out/ev4
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ev4/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev4/smoke.log 2>&1
for w in morlet_multiply_batch scalogram; do
  timeout 600 python bench.py --workload $w > gpurun_out/ev4/bench_$w.json 2> gpurun_out/ev4/bench_$w.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/ev4/launches_batch.csv python bench.py --workload morlet_multiply_batch --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/ev4/launches_scalogram.csv python bench.py --workload scalogram --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sft_tc -s 1 -c 1 -o gpurun_out/ev4/prof_batch -f python tools/tc_one.py 4096 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sft_tc -s 2 -c 1 -o gpurun_out/ev4/prof_scalogram -f python tools/sg_one.py > /dev/null 2>&1
cat gpurun_out/ev4/pytest_gpu.log gpurun_out/ev4/smoke.log; for f in gpurun_out/ev4/bench_*.json; do echo $f; cut -c1-200 $f; done; ls gpurun_out/ev4
