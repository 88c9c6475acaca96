for c in 1 2 4 8; do echo "f16 chunk_kb=$c"; TNC_CHUNK_KB=$c python tools/gemm_bench.py 8192 8192 8192 20; TNC_CHUNK_KB=$c python tools/diag_precision.py one 256 256 16384; done
for c in 4 8 16; do echo "tf32 chunk_kb=$c"; TNC_TC_TF32=1 TNC_CHUNK_KB=$c python tools/gemm_bench.py 8192 8192 8192 20; done
