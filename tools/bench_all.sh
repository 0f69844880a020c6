#!/bin/bash
# GPU box: one bench line per configuration (the headline, every BASELINE config and every NEXT row),
# collected in gpurun_out/TAG/rows.jsonl.  usage: tools/bench_all.sh TAG
set -u
TAG=${1:-rows}
OUT=gpurun_out/$TAG
mkdir -p $OUT
: > $OUT/rows.jsonl
run() {
  local name=$1; shift
  if timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > $OUT/$name.json 2> $OUT/$name.err; then
    python -c "import json,sys; d=json.load(open('$OUT/$name.json')); d['row']='$name'; print(json.dumps(d))" >> $OUT/rows.jsonl
    python -c "import json; d=json.load(open('$OUT/$name.json')); r=d['roofline']; print('$name', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,1), 'M steps/s', r['bound'], r['kernel'], round(r['frac'],3))"
  else
    echo "$name failed"; tail -3 $OUT/$name.err
  fi
}
run metric
run metric_uniform --uniform
run c2 --config c2
run c3 --config c3
run c3i --config c3 --irregular
run c4 --config c4
run c4i --config c4 --irregular --N 4194304
run c5 --config c5
run f32 --config f32
run batched --config batched
run grad --config grad
run gradb --config gradb
run gradco2 --config gradco2
run gradbt --config gradbt
run batchedbt --config batchedbt
run co2post --config co2post
