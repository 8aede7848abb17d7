timeout 120 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -1
timeout 300 python tools/tc_probe.py 2>&1 | tail -3
timeout 120 python tools/tc_trace.py 2>&1 | sed -n '1,1p;18,22p'
