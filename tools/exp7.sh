export TNC_TC_CFG=2
for c in 2 4; do for g in 4 8 16; do echo "2sm chunk=$c group=$g"; TNC_CHUNK_KB=$c TNC_GROUP_M=$g timeout 120 python tools/gemm_bench.py 8192 8192 8192 20; done; done
unset TNC_TC_CFG
for c in 2 4; do echo "1sm chunk=$c"; TNC_CHUNK_KB=$c timeout 120 python tools/gemm_bench.py 8192 8192 8192 20; done
