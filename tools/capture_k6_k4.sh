R=r02
for i in 0 2; do
  python tools/c1_one.py $i 6 2 > gpurun_out/${R}_k6_$i.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:gather_tc -s 1 -c 1 -o gpurun_out/${R}_k6_c1_$i -f python tools/c1_one.py $i 6 3 >> gpurun_out/${R}_k6_$i.log 2>&1
  echo "k6 c1[$i] rc=$?"
done
python tools/absorb_one.py > gpurun_out/${R}_absorb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:absorb_pass -c 1 -o gpurun_out/${R}_absorb_full -f python tools/absorb_one.py > gpurun_out/${R}_ncu_absorb.log 2>&1
echo "absorb rc=$?"
