S="32768 16384 32768 1"
for g in 64 128 256 1024; do echo "group_m=$g"; TNC_GROUP_M=$g python tools/gemm_bench.py $S; done
S2="16384 32768 16384 1"
for g in 16 64 256; do echo "shape2 group_m=$g"; TNC_GROUP_M=$g python tools/gemm_bench.py $S2; done
S3="4096 65536 65536 1"
for g in 16 64 256; do echo "shape3 group_m=$g"; TNC_GROUP_M=$g python tools/gemm_bench.py $S3; done
