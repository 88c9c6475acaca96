nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clk_exp1.csv &
SMI=$!
python tools/gemm_bench.py 8192 8192 8192 100
python tools/gemm_bench.py 16384 16384 16384 4
for g in 4 16 64; do TNC_GROUP_M=$g python tools/gemm_bench.py 32768 16384 32768 1; done
TNC_TC_CFG=1 python tools/gemm_bench.py 32768 16384 32768 1
TNC_CHUNK_KB=8 python tools/gemm_bench.py 32768 16384 32768 1
kill $SMI
awk -F, 'NR>1{print $1,$2}' gpurun_out/clk_exp1.csv | sort | uniq -c | sort -rn | head -8
