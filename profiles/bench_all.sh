#!/bin/bash
# One line per workload: ms/step, roofline fraction, e2e (kernel-only numbers under -no-cpu).
for w in ${@:-morlet_direct gauss_sft_fp64 gauss_asft_fp32 morlet_multiply_batch scalogram}; do
  python bench.py --workload $w --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(f\"{d['config']['workload']:24s} {d['ms_per_step']*1e3:10.2f} us  frac {d['roofline']['frac']:.4f}  e2e {d['e2e']['value']:.1f}\")"
done
