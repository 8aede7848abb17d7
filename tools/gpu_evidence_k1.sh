# Evidence refresh after a K1 change: GPU tests, smoke, bench lines for every workload,
# the reference arm, and the headline's ncu launch list + one full capture of K1.
mkdir -p gpurun_out/ev
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ev/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1
for w in morlet_direct gauss_sft_fp64 gauss_asft_fp32 morlet_multiply_batch scalogram; do
  timeout 600 python bench.py --workload $w > gpurun_out/ev/bench_$w.json 2> gpurun_out/ev/bench_$w.err
done
timeout 300 python bench.py --impl reference > gpurun_out/ev/bench_reference.json 2> gpurun_out/ev/bench_reference.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches_morlet_direct.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sft_scan -s 3 -c 1 -o gpurun_out/ev/prof_morlet_direct -f python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
[ -f .ab_libs/trace.so ] && SFTGPU_LIB=.ab_libs/trace.so timeout 200 python tools/scan_trace.py MDS5P6 8192 > gpurun_out/ev/scan_trace_md.txt 2>&1
cat gpurun_out/ev/pytest_gpu.log gpurun_out/ev/smoke.log; ls -la gpurun_out/ev | head -30
