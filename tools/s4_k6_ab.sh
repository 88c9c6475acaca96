mkdir -p gpurun_out
for d in 1 2; do for sp in 0 1; do
  echo "== depth=$d spin=$sp"
  for i in 0 2; do TNC_GT_DEPTH=$d TNC_GT_SPIN=$sp python tools/c1_one.py $i 6 6 | tail -3 | tr '\n' ' '; echo; done
done; done
echo "== ymode sweep on C1c (depth=1 spin=1)"
for ym in 0 2; do TNC_GT_YMODE=$ym python tools/c1_one.py 2 6 6 | tail -2 | tr '\n' ' '; echo; done
timeout 600 python -m pytest tests/test_gpu_gather_tc.py tests/test_gpu_fullsize.py -x -q -m gpu 2>&1 | tail -3
