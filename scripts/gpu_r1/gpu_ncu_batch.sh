# ncu --set full capture of the c2 batch kernel (one launch after warm-up)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -s 3 -c 1 \
  -o gpurun_out/r1_c2_batch_full $CMD > gpurun_out/r1_ncu_full.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/r1_ncu_full.log
