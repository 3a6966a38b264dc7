mkdir -p gpurun_out
for nm in "128 128 l2" "128 128 sql2" "384 256 l2" "384 256 sql2"; do python scripts/seg_probe1.py $nm; done
FFD_SEG_L=2 python scripts/seg_probe1.py 128 128 l2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 1 -c 1 -o gpurun_out/seg_u128 python scripts/seg_probe1.py 128 128 l2 > gpurun_out/segu.log 2>&1; echo "ncu rc=$?"
