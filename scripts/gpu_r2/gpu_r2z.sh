mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_seg_gpu.py tests/test_cdist_gpu.py -x -q > gpurun_out/segz_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/segz_tests.log
for L in 2 3; do
FFD_SEG_L=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist > gpurun_out/segz_c2_L$L.json 2>gpurun_out/segz_c2.err; echo "c2 L=$L rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/segz_c2_L$L.json')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clocks'])"
done
timeout 600 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/segz_c4.json 2>gpurun_out/segz_c4.err; echo "c4 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/segz_c4.json')); print(d['ms_per_step'], d['value'], d['roofline'])"
