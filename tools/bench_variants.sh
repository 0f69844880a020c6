#!/bin/bash
# usage: tools/bench_variants.sh lib1.so lib2.so ...   (on the GPU box; paths relative to repo root)
for L in "$@"; do
  PSSGP_LIB=$(realpath $L) timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /tmp/bv.log 2>&1
  tail -1 /tmp/bv.log | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],4), d['config']['ctas'], {k: round(v,4) for k,v in d['roofline']['per_kernel_ms_per_step'].items()})
except Exception as e:
    print('$L FAILED'); print(open('/tmp/bv.log').read()[-2000:])
"
done
