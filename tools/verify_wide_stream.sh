# full GPU suite at the new default, full-size C3 irregular parity, C3 irregular / C3 / metric bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputests.log
timeout 300 python tools/config_parity.py c3i > gpurun_out/c3i_parity.txt 2>&1
timeout 150 python bench.py --config c3 --irregular --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_c3i.log 2>&1
timeout 150 python bench.py --config c3 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1
timeout 300 python bench.py > gpurun_out/bench.log 2>&1
tail -n 2 gpurun_out/gputests.log; cat gpurun_out/c3i_parity.txt
