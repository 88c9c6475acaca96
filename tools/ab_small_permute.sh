for m in 1 0 1 0; do
  if [ $m = 1 ]; then export TNC_NO_SMALL_PERMUTE=1; echo "== tile kernel for small permutes"; else unset TNC_NO_SMALL_PERMUTE; echo "== small-permute kernel"; fi
  python bench.py --steps 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python tools/prep_times.py
  python bench.py --workload c1 --steps 20 --warmup 5 2>/dev/null | python tools/bench_line.py | grep C1c
done
unset TNC_NO_SMALL_PERMUTE
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_stream.py -x -q -m gpu 2>&1 | tail -2
