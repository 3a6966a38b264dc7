mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_seg_gpu.py -x -q > gpurun_out/segac_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/segac_tests.log
for B in 1 0; do
FFD_SEG_BIG=$B timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist > gpurun_out/segac_c2_$B.json 2>gpurun_out/segac_c2.err; echo "c2 big=$B rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/segac_c2_$B.json')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clocks'])"
done
FFD_SEG_BIG=0 timeout 300 python -m pytest tests/test_seg_gpu.py -x -q > gpurun_out/segac_tests0.log 2>&1; echo "tests big=0 rc=$?"; tail -1 gpurun_out/segac_tests0.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cdist"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 6 -c 2 -o gpurun_out/seg_c2_ac $CMD > gpurun_out/segac_ncu.log 2>&1; echo "ncu rc=$?"
