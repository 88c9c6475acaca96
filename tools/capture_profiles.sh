# Round profile capture (run on the GPU box, each ncu only after its command
# exited 0 without ncu).  Usage: bash tools/capture_profiles.sh r01
#   1. launch list of the default bench command (C3)
#   2. DRAM bytes per tensor-core GEMM launch of one C3 slice (roofline.traffic)
#   3. full capture of the dominant C3 GEMM shape
#   4. full captures of K6 on C1a and C1c
#   5. full capture of one K4 absorb pass
R=${1:-r01}
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/${R}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tc_cgemm --csv \
  --log-file gpurun_out/${R}_tc_traffic.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${R}_ncu_traffic.log 2>&1
echo "tc traffic rc=$?"
python tools/gemm_bench.py 32768 16384 32768 1 > gpurun_out/${R}_gemm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_cgemm -c 1 -o gpurun_out/${R}_tc_full python tools/gemm_bench.py 32768 16384 32768 1 > gpurun_out/${R}_ncu_tc.log 2>&1
echo "tc full rc=$?"
for i in 0 2; do
  python tools/c1_one.py $i 6 2 > gpurun_out/${R}_k6_$i.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gather_tc -s 1 -c 1 -o gpurun_out/${R}_k6_c1_$i python tools/c1_one.py $i 6 3 >> gpurun_out/${R}_k6_$i.log 2>&1
  echo "k6 c1[$i] rc=$?"
done
# 5. full capture of one K4 absorb pass (rank-28 chain, 16 gates)
python tools/absorb_one.py > gpurun_out/${R}_absorb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:absorb_pass -c 1 -o gpurun_out/${R}_absorb_full python tools/absorb_one.py > gpurun_out/${R}_ncu_absorb.log 2>&1
echo "absorb rc=$?"
