#!/bin/bash
# GPU box: single-pass K1+K3 (PSSGP_FUSED=1) parity subset + interleaved bench A/B against the two-launch path.
set -u
OUT=gpurun_out/${1:-ab_fused}
mkdir -p $OUT
PSSGP_FUSED=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider \
  -k "random_sizes or config or small_chains or missing or metric_full or deterministic or graph or virtual or host" > $OUT/pytest_fused.log 2>&1
echo "fused pytest rc=$?"; tail -3 $OUT/pytest_fused.log
for i in 1 2 3; do
  for F in 0 1; do
    PSSGP_FUSED=$F timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_f${F}_$i.json 2>/dev/null
    python -c "import json; d=json.load(open('$OUT/bench_f${F}_$i.json')); print('fused=$F', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['roofline']['per_kernel_ms_per_step'].items()})"
  done
done
