python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -15
python -m pytest tests/test_gpu_fullsize.py -x -q -k "c1" 2>&1 | tail -3
python bench.py --workload c1 --steps 10 --warmup 3 2>&1 | cut -c1-700
