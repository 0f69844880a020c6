#!/bin/bash
# Run on the GPU box (via gpurun): plain bench, launch list, one full ncu capture per hot kernel.
# usage: tools/gpu_profile.sh <tag> [kernel-regex]
set -u
TAG=${1:-r1}
KRE=${2:-k_filter_apply|k_smoother_apply|k_filter_reduce}
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > $OUT/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -20 $OUT/plain_$TAG.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s 3 -c 3 \
    -o $OUT/prof_$TAG $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "profile done rc=$?"
