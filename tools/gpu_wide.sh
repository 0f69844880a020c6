#!/bin/bash
# GPU box: wide-path tests + C3 full-size parity + C3 / C3-irregular bench lines.
set -u
TAG=${1:-r2w}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -k "wide or pade or irregular or kw_ or sharded or nll_only or handle or config3" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -15 $OUT/pytest.log
for CFG in "c3" "c3 --irregular"; do
  timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_${CFG// /_}.json 2> $OUT/bench_${CFG// /_}.err; echo "bench $CFG rc=$?"
  python -c "import json,sys; d=json.load(open('$OUT/bench_${CFG// /_}.json')); print(d['ms_per_step'], json.dumps(d['roofline']['per_kernel_ms_per_step']))"
done
