# absorb (K4) kernel: parity tests, C2 bench for both buffering modes, one full ncu capture
python -m pytest tests/test_gpu_fusion.py tests/test_gpu_edges.py -x -q 2>&1 | tail -15
python -m pytest tests/test_gpu_fullsize.py -x -q -k "c2 or chain or fused" 2>&1 | tail -3
for nb in 1 2; do echo "NBUF=$nb"; TNC_ABSORB_NBUF=$nb python bench.py --workload c2 --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-900; done
python tools/absorb_one.py > gpurun_out/abs_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:absorb -c 1 -o gpurun_out/absorb_r01b python tools/absorb_one.py > gpurun_out/ncu_absb.log 2>&1
echo "ncu rc=$?"
