ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/stream_c1a3 python tools/c1a_time.py > gpurun_out/ncu_stream3.log 2>&1
echo "ncu rc=$?"
