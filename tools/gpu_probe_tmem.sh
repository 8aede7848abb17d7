mkdir -p gpurun_out/pr
for d in 0 24 64 128 192 216 32 248; do
  for w in morlet_multiply_batch; do
  SFTGPU_TC_DBG=$d SFTGPU_LIB=.ab_libs/probe.so timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu 2>/dev/null | tail -1 > gpurun_out/pr/${w}_$d.json
  python -c "import json; d=json.loads(open('gpurun_out/pr/${w}_$d.json').read()); print('$w dbg=$d', round(d['ms_per_step']*1000,1), 'us', d['clocks']['sm_mhz'])"
  done
done
