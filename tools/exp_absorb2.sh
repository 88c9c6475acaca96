python -m pytest tests/test_gpu_fusion.py tests/test_gpu_edges.py -x -q 2>&1 | tail -3
python -m pytest tests/test_gpu_fullsize.py -x -q -k "c2 or chain or fused" 2>&1 | tail -2
for nb in 1 2; do echo "NBUF=$nb"; TNC_ABSORB_NBUF=$nb python bench.py --workload c2 --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-400; done
python tools/absorb_one.py > gpurun_out/abs_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:absorb -c 1 -o gpurun_out/absorb_r01c python tools/absorb_one.py > gpurun_out/ncu_absc.log 2>&1
echo "ncu rc=$?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tc_cgemm --csv --log-file gpurun_out/r01_tc_traffic.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_traffic.log 2>&1
echo "traffic rc=$?"
