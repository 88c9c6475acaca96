L=paper_2504_09186_b200/libtnc_b200.so
cp $L /tmp/new.so
for rep in 1 2; do
for lib in build_base_libtnc_b200.so /tmp/new.so; do
  cp $lib $L; echo "== $lib"
  python bench.py --steps 6 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python tools/prep_times.py
done; done
cp /tmp/new.so $L
python bench.py --workload c1 --steps 20 --warmup 5 2>/dev/null | python tools/bench_line.py
