# staged (F, Q) in the lane-per-row fold: C3 irregular / C3 bench, full GPU suite, full-size C3-irregular parity
mkdir -p gpurun_out
for C in "--config c3 --irregular" "--config c3"; do
  timeout 150 python bench.py $C --no-cpu-baseline --steps 5 --warmup 3 2>&1 | tail -n 1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$C', j['ms_per_step'], j['roofline'].get('per_kernel_ms_per_step'))" >> gpurun_out/sweep5.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputests.log
timeout 300 python tools/config_parity.py c3i > gpurun_out/c3i_parity.txt 2>&1
cat gpurun_out/sweep5.log; tail -n 2 gpurun_out/gputests.log; cat gpurun_out/c3i_parity.txt
