timeout 300 python tools/tc_rcase.py 2>&1 | tail -10
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_shipped_paths.py tests/test_gpu_transforms.py -q -x 2>&1 | tail -2
bash profiles/bench_all.sh morlet_multiply_batch scalogram 2>&1
