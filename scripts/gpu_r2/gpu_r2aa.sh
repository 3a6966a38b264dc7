mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_seg_gpu.py tests/test_batch_gpu.py -x -q > gpurun_out/segab_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/segab_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist > gpurun_out/segab_c2.json 2>gpurun_out/segab_c2.err; echo "c2 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/segab_c2.json')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clocks'])"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cdist"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 3 -c 1 -o gpurun_out/seg_c2_ab $CMD > gpurun_out/segab_ncu.log 2>&1; echo "ncu rc=$?"
