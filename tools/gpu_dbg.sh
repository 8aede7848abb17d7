timeout 300 python tools/tc_rcase.py GDS10P6:8192:0 MDS5P6:8192:10 MMS5P3:8192:10 GDS5P6:3001:0 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -2
bash profiles/bench_all.sh morlet_multiply_batch scalogram 2>&1
