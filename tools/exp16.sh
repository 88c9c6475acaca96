python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py 2>&1 | tail -1 > gpurun_out/bench_c3_r01b.json; cut -c1-600 gpurun_out/bench_c3_r01b.json
python bench.py --workload c4 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | cut -c1-500
python bench.py --workload c2 --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-300
