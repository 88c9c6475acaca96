# Round profile capture: launch list of the bench command + full ncu of the
# dominant GEMM shape.  Usage: bash tools/capture_profiles.sh r01
R=${1:-r01}
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/${R}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/gemm_bench.py 32768 16384 32768 1 > gpurun_out/${R}_gemm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_cgemm -c 1 -o gpurun_out/${R}_tc_full python tools/gemm_bench.py 32768 16384 32768 1 > gpurun_out/${R}_ncu_tc.log 2>&1
echo "tc full rc=$?"
