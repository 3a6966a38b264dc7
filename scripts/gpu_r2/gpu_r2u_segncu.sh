mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cdist"
$CMD > gpurun_out/segncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 3 -c 1 -o gpurun_out/seg_c2 $CMD > gpurun_out/segncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/segncu.log
