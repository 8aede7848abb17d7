timeout 300 python tools/e2e_probe2.py 2>&1 | grep -E "wrapper|pipelined"
for i in 1 2; do timeout 300 python bench.py --no-cpu --steps 50 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['e2e']['value'], 1e6*102400/d['e2e']['value']/1e6)"; done
