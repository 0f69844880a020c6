#!/bin/bash
set -u
OUT=gpurun_out/${1:-w16}
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "wide or pade or irregular or kw_ or co2 or odd or sharded or general or config4 or config3" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"
tail -15 $OUT/pytest.log
for CFG in "c4" "c3"; do
  timeout 900 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$CFG.json 2> $OUT/bench_$CFG.err; echo "bench $CFG rc=$?"
  python -c "import json; d=json.load(open('$OUT/bench_$CFG.json')); print(d['ms_per_step'], json.dumps({k: round(v,3) for k,v in d['roofline']['per_kernel_ms_per_step'].items()}))"
done
