# round evidence (usage: bash tools/round_evidence.sh): GPU suite, one bench line per BASELINE config, the 3xTF32 C3 line, the reference arm
mkdir -p gpurun_out
(timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gputest.log)
timeout 600 python bench.py --workload c1 --steps 10 --warmup 3 > gpurun_out/r02_bench_c1.jsonl 2> gpurun_out/r02_bench_c1.err; echo "c1 rc=$?"
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err; echo "c3 rc=$?"
TNC_TC_TF32=1 timeout 900 python bench.py --steps 5 > gpurun_out/r02_bench_c3_tf32.json 2> gpurun_out/r02_bench_c3_tf32.err; echo "c3 tf32 rc=$?"
timeout 900 python bench.py --workload c4 --steps 5 > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err; echo "ref rc=$?"
tail -3 gpurun_out/r02_gputest.log
