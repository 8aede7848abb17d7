# A/B timing on one GPU box: a reference build of the library (.ab_libs/base.so, e.g. built
# from a git worktree of the previous commit) against the working tree, alternated twice.
#   W="<bench workloads>" TESTS=<pytest paths> bash tools/gpu_ab.sh   (under gpurun)
W=${W:-morlet_multiply_batch}
run() { env "$@" timeout 300 python bench.py --workload $w 2>/dev/null | tail -1; }
[ -n "$TESTS" ] && timeout 900 python -m pytest $TESTS -x -q 2>&1 | tail -3 > gpurun_out/ab_tests.log
for w in $W; do
  for r in 1 2; do
    run SFTGPU_LIB=.ab_libs/base.so > gpurun_out/ab_${w}_base_$r.json
    run X=1 > gpurun_out/ab_${w}_new_$r.json
  done
done
cat gpurun_out/ab_tests.log 2>/dev/null
for f in gpurun_out/ab_*.json; do
  python -c "import json; d=json.loads(open('$f').read()); print('$f', round(d['ms_per_step'] * 1000, 3), 'us', d['clocks']['sm_mhz'])" 2>/dev/null || echo "$f: no result"
done
