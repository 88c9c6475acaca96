export TNC_TC_CFG=2
timeout 60 python tools/diag_precision.py one 512 512 4096
timeout 60 python tools/diag_precision.py one 300 200 1000
timeout 120 python tools/gemm_bench.py 8192 8192 8192 20
timeout 300 python tools/gemm_bench.py 32768 16384 32768 1
unset TNC_TC_CFG
timeout 120 python tools/gemm_bench.py 8192 8192 8192 20
