set -x
for G in 8 16 32 64 128; do
  TNC_GROUP_M=$G python bench.py --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/sweep_g$G.json 2>/dev/null
  TNC_GROUP_M=$G ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tc_cgemm --csv --log-file gpurun_out/sweep_g$G.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
