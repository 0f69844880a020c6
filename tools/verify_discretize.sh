# launch-bounds variants of kw_discretize_lpr on C3 irregular, then the full GPU suite and full-size C3-irregular parity (default build)
mkdir -p gpurun_out
bash tools/bench_variants_cfg.sh "--config c3 --irregular" variants/libpssgp_d1.so variants/libpssgp_d4.so variants/libpssgp_d5.so > gpurun_out/variants.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputests.log
timeout 300 python tools/config_parity.py c3i > gpurun_out/c3i_parity.txt 2>&1
cat gpurun_out/variants.log; tail -n 2 gpurun_out/gputests.log; cat gpurun_out/c3i_parity.txt
