# session probe: FFMA/FFMA2 rate, ncu full captures of K4 (rank-28 chain pass) and K6 (C1a, C1c)
mkdir -p gpurun_out
./build/ffma2_rate > gpurun_out/s4_ffma2_rate.txt 2>&1
python tools/absorb_one.py > gpurun_out/s4_absorb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:absorb_pass -c 1 -o gpurun_out/s4_absorb_full python tools/absorb_one.py > gpurun_out/s4_ncu_absorb.log 2>&1
echo "absorb rc=$?"
for i in 0 2; do
  python tools/c1_one.py $i 6 2 > gpurun_out/s4_k6_$i.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gather_tc -s 1 -c 1 -o gpurun_out/s4_k6_c1_$i python tools/c1_one.py $i 6 3 >> gpurun_out/s4_k6_$i.log 2>&1
  echo "k6 c1[$i] rc=$?"
done
