S="32768 16384 32768 1"
for g in 16 4 8 32 64; do echo "group_m=$g"; TNC_GROUP_M=$g python tools/gemm_bench.py $S; done
for g in 16 4 64; do TNC_GROUP_M=$g ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:tc_cgemm -c 1 python tools/gemm_bench.py $S 2>&1 | grep -E "dram__bytes|duration|per_second" | sed "s/^/g=$g /"; done
