S="32768 16384 32768 1"
for g in 8 16 32 64; do echo "2sm chunk4 g=$g"; TNC_TC_CFG=2 TNC_CHUNK_KB=4 TNC_GROUP_M=$g python tools/gemm_bench.py $S; done
for g in 32 64; do TNC_TC_CFG=2 TNC_CHUNK_KB=4 TNC_GROUP_M=$g ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:tc_cgemm -c 1 python tools/gemm_bench.py $S 2>&1 | grep -E "dram__bytes|duration|per_second" | sed "s/^/g=$g /"; done
