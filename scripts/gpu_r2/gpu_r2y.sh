mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cdist"
for L in 2 8; do
FFD_SEG_L=$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 3 -c 1 -o gpurun_out/seg_c2_L$L $CMD > gpurun_out/segncu_L$L.log 2>&1; echo "ncu L=$L rc=$?"
done
