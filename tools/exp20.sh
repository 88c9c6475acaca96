python -m pytest tests/test_gpu_parity.py -x -q -k "reuse" 2>&1 | tail -2
python bench.py --workload c4 --reuse 1 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 > gpurun_out/c4_reuse1.json; cut -c1-1500 gpurun_out/c4_reuse1.json
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
