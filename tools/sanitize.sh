#!/bin/bash
# GPU box: one compute-sanitizer tool over tools/sanitize_case.py (after a plain run that must exit 0),
# plus three headline bench lines.  usage: tools/sanitize.sh TOOL
set -u
TOOL=${1:-memcheck}
OUT=gpurun_out/sanitizer
mkdir -p $OUT
timeout 600 python tools/sanitize_case.py > $OUT/plain_$TOOL.log 2>&1 || { echo "plain run failed"; tail $OUT/plain_$TOOL.log; exit 1; }
for i in 1 2 3; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_$i.json 2>/dev/null; python -c "import json; d=json.load(open('$OUT/bench_$i.json')); print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['roofline']['per_kernel_ms_per_step'].items()})"; done
EXTRA=""
[ "$TOOL" = "memcheck" ] && EXTRA="--leak-check full"
timeout 2400 compute-sanitizer --tool $TOOL $EXTRA --print-limit 50 --log-file $OUT/$TOOL.log python tools/sanitize_case.py > $OUT/${TOOL}_stdout.log 2>&1
echo "sanitizer rc=$?"
tail -5 $OUT/$TOOL.log
