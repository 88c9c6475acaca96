nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 250 > gpurun_out/clk_exp4.csv &
SMI=$!
TNC_CHUNK_KB=4 python tools/gemm_bench.py 8192 8192 8192 100
kill $SMI
python tools/gemm_bench.py 8192 8192 8192 1 && ncu --set full --clock-control none -k regex:tc_cgemm -c 1 -o gpurun_out/tc_f16 python tools/gemm_bench.py 8192 8192 8192 1 > gpurun_out/ncu_f16.log 2>&1; tail -2 gpurun_out/ncu_f16.log
