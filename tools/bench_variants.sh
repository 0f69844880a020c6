#!/bin/bash
# usage: tools/bench_variants.sh lib1.so lib2.so ...   (on the GPU box)
for L in "$@"; do
  PSSGP_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['roofline']['per_kernel_ms_per_step'].items()})"
done
