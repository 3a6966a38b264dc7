mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_seg_gpu.py -x -q > gpurun_out/segad_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/segad_tests.log
for v in "FFD_X=0" "FFD_X=1"; do
env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist > gpurun_out/segad_c2.json 2>gpurun_out/segad_c2.err; echo "c2 [$v] rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/segad_c2.json')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
