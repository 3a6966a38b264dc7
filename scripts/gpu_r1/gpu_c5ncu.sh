mkdir -p gpurun_out
CMD5="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD5 > gpurun_out/ncu_plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:long_kernel -s 4 -c 1 \
  -o gpurun_out/c5_long_full $CMD5 > gpurun_out/ncu_c5.log 2>&1
echo "ncu c5 rc=$?"; python -c "import json;d=json.load(open('/dev/stdin'));print(d['ms_per_step'])" < gpurun_out/ncu_plain5.log
