#!/bin/bash
# usage: tools/bench_variants_cfg.sh "bench args" lib1.so lib2.so ...   (on the GPU box)
ARGS=$1; shift
for L in "$@"; do
  PSSGP_LIB=$(realpath $L) timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline $ARGS > /tmp/bv.log 2>&1
  tail -1 /tmp/bv.log | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['roofline']['per_kernel_ms_per_step'].items()})
except Exception as e:
    print('$L FAILED'); print(open('/tmp/bv.log').read()[-1500:])
"
done
