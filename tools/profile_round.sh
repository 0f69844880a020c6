#!/bin/bash
# Run on the GPU box (via gpurun): the bench line, the ncu launch list of the same command, and one
# `--set full` capture of each hot kernel exported to CSV (raw metrics + SASS source page).
# usage: tools/profile_round.sh TAG [bench args...]
set -u
TAG=$1; shift
ARGS=${*:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline $ARGS"
python bench.py --steps 10 --warmup 3 $ARGS > $OUT/bench.json 2> $OUT/bench.err || { echo "bench failed"; tail $OUT/bench.err; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv $CMD \
    > $OUT/ncu_launch.log 2>&1
for K in ${KERNELS:-k_filter_reduce k_filter_apply k_smoother_apply} ${EXTRA_KERNELS:-}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^${K}" -s 2 -c 1 -o /tmp/p_$K $CMD \
      > $OUT/ncu_full_$K.log 2>&1
  ncu -i /tmp/p_$K.ncu-rep --page raw --csv > $OUT/raw_$K.csv 2>/dev/null
  ncu -i /tmp/p_$K.ncu-rep --page source --csv --print-source sass > $OUT/src_$K.csv 2>/dev/null
  rm -f /tmp/p_$K.ncu-rep
done
echo "profile $TAG done"
