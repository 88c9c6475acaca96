for c in 1 2 4; do echo "f16 chunk_kb=$c"; TNC_CHUNK_KB=$c python tools/gemm_bench.py 8192 8192 8192 20; TNC_CHUNK_KB=$c python tools/diag_precision.py one 256 256 16384; done
echo "f16 sw64 4 stages"; TNC_TC_CFG=1 python tools/gemm_bench.py 8192 8192 8192 20
TNC_TC_CFG=1 TNC_CHUNK_KB=4 python tools/gemm_bench.py 8192 8192 8192 20
python tools/gemm_bench.py 32768 16384 32768 1
python tools/gemm_bench.py 8192 8192 8192 1 && ncu --set full --clock-control none -k regex:tc_cgemm -c 1 -o gpurun_out/tc_f16 python tools/gemm_bench.py 8192 8192 8192 1 > gpurun_out/ncu_f16.log 2>&1; tail -1 gpurun_out/ncu_f16.log
