#!/bin/bash
# GPU box: for each configuration, the bench line, the ncu launch list of the same command and one
# `ncu --set full` capture per hot kernel exported to CSV (raw + SASS source).
# usage: tools/profile_configs.sh TAG "cfgkey|bench args|kernel regexes" ...
set -u
TAG=$1; shift
for SPEC in "$@"; do
  KEY=${SPEC%%|*}; REST=${SPEC#*|}; ARGS=${REST%%|*}; KERNELS=${REST#*|}
  OUT=gpurun_out/${TAG}_${KEY}
  mkdir -p $OUT
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline $ARGS"
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $ARGS > $OUT/bench.json 2> $OUT/bench.err || { echo "bench $KEY failed"; tail -5 $OUT/bench.err; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
  for K in $KERNELS; do
    timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:^${K}" -s 1 -c 1 -o /tmp/p_$K $CMD > $OUT/ncu_full_$K.log 2>&1
    ncu -i /tmp/p_$K.ncu-rep --page raw --csv > $OUT/raw_$K.csv 2>/dev/null
    ncu -i /tmp/p_$K.ncu-rep --page source --csv --print-source sass > $OUT/src_$K.csv 2>/dev/null
    rm -f /tmp/p_$K.ncu-rep
  done
  echo "profile $KEY done: $(python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['ms_per_step'])")"
done
