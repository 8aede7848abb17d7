timeout 300 python tools/tc_trace.py 2>&1 | sed -n '1,3p;14,26p'
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -3
timeout 300 python tools/tc_probe.py 1 2>&1 | tail -5
