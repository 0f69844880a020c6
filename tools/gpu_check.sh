#!/bin/bash
# GPU box: the GPU test suite (incl. full-size parity), smoke, and the headline bench line.
# usage: tools/gpu_check.sh TAG [pytest -k expr]
set -u
TAG=${1:-r2}
K=${2:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -q -m gpu -k "$K" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
else
  timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
fi
tail -40 $OUT/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
tail -3 $OUT/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
cat $OUT/bench.json | head -c 3000
