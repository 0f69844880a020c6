#!/bin/bash
# GPU box: wide-path parity subset, then C4 / C3 bench lines (PSSGP_WIDE_DEBUG prints the plan occupancy)
set -u
OUT=gpurun_out/${1:-bw}
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "${2:-wide or pade or co2 or odd or general or config4}" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
for CFG in "c4" "c3"; do
  PSSGP_WIDE_DEBUG=1 timeout 900 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$CFG.json 2> $OUT/bench_$CFG.err; echo "bench $CFG rc=$?"; grep "wide plan" $OUT/bench_$CFG.err | head -2
  python -c "import json; d=json.load(open('$OUT/bench_$CFG.json')); print(d['ms_per_step'], d['config']['chain_len'], json.dumps({k: round(v,3) for k,v in d['roofline']['per_kernel_ms_per_step'].items()}))"
done
