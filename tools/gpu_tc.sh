timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for w in morlet_multiply_batch scalogram; do timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -c 600 gpurun_out/bench_$w.json; echo; done
