#!/bin/bash
set -u
OUT=gpurun_out/${1:-c3i}
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "pade or irregular or kw_ or odd" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
timeout 900 python tools/config_parity.py c3i > $OUT/parity_c3i.txt 2>&1; cat $OUT/parity_c3i.txt
for CFG in "c3 --irregular" "c4 --irregular --N 4194304"; do
  timeout 900 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench $CFG rc=$?"
  python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['ms_per_step'], json.dumps({k: round(v,3) for k,v in d['roofline']['per_kernel_ms_per_step'].items()}))"
done
