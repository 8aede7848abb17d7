# K4 iteration: tensor-core parity tests, config-4/5 kernel-only bench lines, pipeline trace.
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_shipped_paths.py -q -x 2>&1 | tail -15 > gpurun_out/k4_pytest.log
bash profiles/bench_all.sh morlet_multiply_batch scalogram > gpurun_out/k4_bench.txt 2>&1
SFTGPU_LIB=tools/libsftgpu_trace.so timeout 120 python tools/tc_trace.py 4096 > gpurun_out/k4_trace.txt 2>&1
cat gpurun_out/k4_pytest.log gpurun_out/k4_bench.txt; head -45 gpurun_out/k4_trace.txt
