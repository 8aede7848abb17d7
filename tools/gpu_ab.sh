# A/B timing on one GPU box: a reference build of the library (.ab_libs/base.so, e.g. built
# from a git worktree of the previous commit) against the working tree, alternated twice.
#   W=<bench workload> TESTS=<pytest paths> bash tools/gpu_ab.sh   (under gpurun)
W=${W:-morlet_multiply_batch}
run() { env "$@" timeout 300 python bench.py --workload $W 2>/dev/null | tail -1; }
[ -n "$TESTS" ] && timeout 600 python -m pytest $TESTS -x -q 2>&1 | tail -3
for r in 1 2; do
  run SFTGPU_LIB=.ab_libs/base.so > gpurun_out/ab_base_$r.json
  run X=1 > gpurun_out/ab_new_$r.json
done
for f in gpurun_out/ab_*.json; do
  python -c "import json; d=json.loads(open('$f').read()); print('$f', round(d['ms_per_step'], 4), d['clocks']['sm_mhz'])"
done
