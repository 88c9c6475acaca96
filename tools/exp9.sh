# elected MMA issue: parity first, then GEMM configs on the dominant C3 shape
python -m pytest tests/test_gpu_parity.py -x -q -k "tc or contract" 2>&1 | tail -2
S="32768 16384 32768 1"
echo "1sm default"; python tools/gemm_bench.py $S
echo "1sm chunk2"; TNC_CHUNK_KB=2 python tools/gemm_bench.py $S
echo "2sm chunk2"; TNC_TC_CFG=2 python tools/gemm_bench.py $S
echo "2sm chunk4"; TNC_TC_CFG=2 TNC_CHUNK_KB=4 python tools/gemm_bench.py $S
echo "tf32 1sm"; TNC_VARIANT=2 python tools/gemm_bench.py $S
TNC_TC_CFG=2 python -m pytest tests/test_gpu_parity.py -x -q -k "tc" 2>&1 | tail -2
