# same-box A/B of prebuilt library variants on C1: usage: bash tools/ab_libs_same_box.sh lib1.so lib2.so ...
L=paper_2504_09186_b200/libtnc_b200.so
cp $L /tmp/new.so
for lib in "$@"; do
  echo "== $lib"; cp $lib $L; python bench.py --workload c1 --steps 20 --warmup 5 2>/dev/null | python tools/bench_line.py | grep -v C1b
done
cp /tmp/new.so $L
