mkdir -p gpurun_out
for M in 31 63; do
  PSSGP_WIDE_LPR=$M timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "wide or irregular or pade" > gpurun_out/par_$M.log 2>&1; echo "M=$M pytest exit $?" >> gpurun_out/par_$M.log
done
for M in 27 31 63; do
  PSSGP_WIDE_LPR=$M timeout 150 python bench.py --config c3 --irregular --no-cpu-baseline --steps 5 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c3irr', $M, j['ms_per_step'], j['config']['chain_len'], j['roofline'].get('per_kernel_ms_per_step'))" >> gpurun_out/sweep3.log 2>&1
done
PSSGP_WIDE_LPR=27 timeout 150 python bench.py --config c3 --no-cpu-baseline --steps 5 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c3', 27, j['ms_per_step'])" >> gpurun_out/sweep3.log 2>&1
tail -1 gpurun_out/par_31.log gpurun_out/par_63.log; cat gpurun_out/sweep3.log
