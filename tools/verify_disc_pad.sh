# kw_discretize_lpr writing whole records (padding column): C3 irregular bench, wide/pade parity, ncu of the kernel
mkdir -p gpurun_out
timeout 150 python bench.py --config c3 --irregular --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_c3i.log 2>&1
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "wide or irregular or pade" > gpurun_out/par_pad.log 2>&1; echo "pytest exit $?" >> gpurun_out/par_pad.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kw_discretize_lpr -c 1 -o gpurun_out/c3i_disc python bench.py --config c3 --irregular --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_disc.log 2>&1
tail -n 1 gpurun_out/bench_c3i.log | cut -c1-200; tail -n 2 gpurun_out/par_pad.log
