S="32768 16384 32768 1"
echo "1sm default"; python tools/gemm_bench.py $S
echo "1sm chunk2"; TNC_CHUNK_KB=2 python tools/gemm_bench.py $S
echo "1sm sw64 4st"; TNC_TC_CFG=1 python tools/gemm_bench.py $S
echo "2sm chunk2"; TNC_TC_CFG=2 python tools/gemm_bench.py $S
echo "2sm chunk4"; TNC_TC_CFG=2 TNC_CHUNK_KB=4 python tools/gemm_bench.py $S
echo "2sm chunk2 g16"; TNC_TC_CFG=2 TNC_GROUP_M=16 python tools/gemm_bench.py $S
echo "2sm chunk2 g4"; TNC_TC_CFG=2 TNC_GROUP_M=4 python tools/gemm_bench.py $S
