set -x
python tools/diag_precision.py one 256 256 4096
python tools/diag_precision.py one 256 256 65536
python tools/diag_precision.py pos 256 256 4096
python tools/gemm_bench.py 8192 8192 8192 20
TNC_TC_CFG=1 python tools/gemm_bench.py 8192 8192 8192 20
python tools/gemm_bench.py 32768 16384 32768 1
TNC_TC_TF32=1 python tools/gemm_bench.py 8192 8192 8192 20
python tools/perm_bench.py
