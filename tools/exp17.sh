python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -2
python tools/c1a_time.py
