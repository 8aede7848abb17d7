# A/B/C timing of K4 variant libraries on one box: base, then each VARIANTS entry
# "name:ENV=val" (library .ab_libs/<name>.so), alternated twice, for the W workloads.
W=${W:-morlet_multiply_batch scalogram}
mkdir -p gpurun_out/ab3
for w in $W; do
  for r in 1 2; do
    for v in base $VARIANTS; do
      name=${v%%:*}; envs=""; [ "$v" != "$name" ] && envs=${v#*:}
      env $envs SFTGPU_LIB=.ab_libs/$name.so timeout 300 python bench.py --workload $w --no-cpu 2>/dev/null | tail -1 > gpurun_out/ab3/${w}_${name}_$r.json
    done
  done
done
for f in gpurun_out/ab3/*.json; do
  python -c "import json; d=json.loads(open('$f').read()); print('$f', round(d['ms_per_step'] * 1000, 1), 'us', d['clocks']['sm_mhz'])" 2>/dev/null || echo "$f: no result"
done
