timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu --workload morlet_multiply_batch --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e'])"
