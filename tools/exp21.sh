S="32768 16384 32768 1"
TNC_TC_CFG=2 TNC_CHUNK_KB=4 python tools/gemm_bench.py $S
TNC_TC_CFG=2 TNC_CHUNK_KB=4 ncu --set full --clock-control none --import-source on -k regex:tc_cgemm_2sm -c 1 -o gpurun_out/tc2sm python tools/gemm_bench.py $S > gpurun_out/ncu_tc2sm.log 2>&1
echo "ncu rc=$?"
