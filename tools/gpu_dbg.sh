timeout 300 python tools/tc_rcase.py 2>&1 | tail -10
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -2
bash profiles/bench_all.sh morlet_multiply_batch scalogram 2>&1
SFTGPU_LIB=tools/libsftgpu_trace.so timeout 120 python tools/tc_trace.py 4096 > gpurun_out/k4_trace.txt 2>&1
