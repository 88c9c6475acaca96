# Same-box A/B on C1: a baseline library, then the current one (optionally under env settings).
# Box-to-box spread on C1 is about 5 %, so only runs inside one gpurun call compare.
#   baseline: build another commit's library in a git worktree and copy it to
#   build_base_libtnc_b200.so at the repo root (*.so is git-ignored but travels with gpurun)
#   usage: bash tools/ab_c1_same_box.sh TNC_X=1 TNC_GT_OCC2=0 ...   (one current-library run per argument)
L=paper_2504_09186_b200/libtnc_b200.so
cp $L /tmp/new.so
echo "== base"; cp build_base_libtnc_b200.so $L; python bench.py --workload c1 --steps 20 --warmup 5 2>/dev/null | python tools/bench_line.py | grep -v C1b
cp /tmp/new.so $L
for cfg in "$@"; do
  echo "== new $cfg"; env $cfg python bench.py --workload c1 --steps 20 --warmup 5 2>/dev/null | python tools/bench_line.py | grep -v C1b
done
