mkdir -p gpurun_out
python scripts/seg_probe1.py 128 128 l2
python scripts/seg_probe1.py 128 128 l2 percurve
python scripts/seg_probe1.py 128 128 l2 percurve
FFD_SEG_L=2 python scripts/seg_probe1.py 128 128 l2
FFD_SEG_L=2 python scripts/seg_probe1.py 128 128 l2
FFD_SEG=0 python scripts/seg_probe1.py 128 128 l2 percurve
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 1 -c 1 -o gpurun_out/seg_u128pc python scripts/seg_probe1.py 128 128 l2 percurve > gpurun_out/segu.log 2>&1; echo "ncu rc=$?"
