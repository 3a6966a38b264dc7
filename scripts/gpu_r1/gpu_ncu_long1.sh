mkdir -p gpurun_out
python scripts/one_long.py 1024 > gpurun_out/one_long.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:long_kernel -s 2 -c 1 -o gpurun_out/long1024 python scripts/one_long.py 1024 > gpurun_out/ncu_long1024.log 2>&1
echo "rc=$?"
