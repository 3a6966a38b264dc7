# segmented batch kernel: parity tests, then c2 at L = 4 / 8 and without it
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_seg_gpu.py -x -q > gpurun_out/seg_tests.log 2>&1; echo "seg tests rc=$?"; tail -3 gpurun_out/seg_tests.log
for L in 2 4 8; do
FFD_SEG_L=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist > gpurun_out/seg_c2_L$L.json 2>gpurun_out/seg_c2.err; echo "c2 L=$L rc=$?"; cut -c1-330 gpurun_out/seg_c2_L$L.json | cut -c150-330
done
FFD_SEG=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist > gpurun_out/seg_c2_off.json 2>&1; echo "c2 noseg rc=$?"; cut -c150-330 gpurun_out/seg_c2_off.json
python scripts/seg_probe.py > gpurun_out/seg_probe3.jsonl 2>&1; grep batch gpurun_out/seg_probe3.jsonl
