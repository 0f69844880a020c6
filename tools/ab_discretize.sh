# A/B of the lane-per-row discretisation (bit 6 of PSSGP_WIDE_LPR): parity of the per-step (F, Q) tests, C3 irregular bench
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "wide or irregular or pade" > gpurun_out/par_127.log 2>&1; echo "pytest exit $?" >> gpurun_out/par_127.log
for M in 63 127; do
  PSSGP_WIDE_LPR=$M timeout 150 python bench.py --config c3 --irregular --no-cpu-baseline --steps 5 --warmup 3 2>&1 | tail -n 1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c3irr', $M, j['ms_per_step'], j['roofline'].get('per_kernel_ms_per_step'))" >> gpurun_out/sweep4.log 2>&1
done
tail -n 2 gpurun_out/par_127.log; cat gpurun_out/sweep4.log
