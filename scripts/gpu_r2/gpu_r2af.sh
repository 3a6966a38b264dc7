mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_seg_gpu.py tests/test_batch_gpu.py -x -q > gpurun_out/segaf_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/segaf_tests.log
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/segaf_c3.json 2>gpurun_out/segaf_c3.err; echo "c3 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/segaf_c3.json')); print(d['ms_per_step'], d['value'], d['roofline']['frac'])"
FFD_SEG=0 timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/segaf_c3_off.json 2>&1; echo "c3 noseg rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/segaf_c3_off.json')); print(d['ms_per_step'], d['value'], d['roofline']['frac'])"
