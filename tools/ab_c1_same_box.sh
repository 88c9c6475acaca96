# same-box A/B on C1: the session-start library, then the current one (optionally under env settings)
L=paper_2504_09186_b200/libtnc_b200.so
cp $L /tmp/new.so
echo "== base"; cp build_base_libtnc_b200.so $L; python bench.py --workload c1 --steps 20 --warmup 5 2>/dev/null | python tools/bench_line.py | grep -v C1b
cp /tmp/new.so $L
for cfg in "$@"; do
  echo "== new $cfg"; env $cfg python bench.py --workload c1 --steps 20 --warmup 5 2>/dev/null | python tools/bench_line.py | grep -v C1b
done
