# ncu --set full of the c2 batch kernel (two-column build)
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cdist"
timeout 300 $CMD > gpurun_out/r2g_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -s 6 -c 1 -o gpurun_out/r2g_c2 $CMD > gpurun_out/r2g_ncu.log 2>&1; echo "ncu rc=$?"
