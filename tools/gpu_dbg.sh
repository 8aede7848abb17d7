for d in 0 32 24 56 0 32; do echo "== dbg $d"; SFTGPU_TC_DBG=$d bash profiles/bench_all.sh morlet_multiply_batch scalogram 2>&1; done
