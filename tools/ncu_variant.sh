#!/bin/bash
# usage (GPU box): tools/ncu_variant.sh TAG LIB KERNEL_REGEX [keep]
#   one full ncu capture of one launch -> gpurun_out/src_TAG.csv (SASS source page) +
#   gpurun_out/raw_TAG.csv (raw metrics); the .ncu-rep is deleted unless "keep" (64 MiB return cap)
set -u
TAG=$1; LIB=$2; KRE=$3; KEEP=${4:-}
mkdir -p gpurun_out
PSSGP_LIB=$(realpath $LIB) timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s 1 -c 1 \
    -o /tmp/prof_$TAG python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
echo "$TAG rc=$?"
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$TAG.csv 2>/dev/null
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>/dev/null
[ -n "$KEEP" ] && cp /tmp/prof_$TAG.ncu-rep gpurun_out/
rm -f /tmp/prof_$TAG.ncu-rep
