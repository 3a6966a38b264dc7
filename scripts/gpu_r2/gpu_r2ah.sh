mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_longpair_gpu.py tests/test_dtw_gpu.py -x -q > gpurun_out/ah_tests.log 2>&1; echo "long+dtw tests rc=$?"; tail -1 gpurun_out/ah_tests.log
for i in 1 2; do
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ah_c5.json 2>gpurun_out/ah_c5.err; echo "c5 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/ah_c5.json')); print(d['ms_per_step'], d['value'], d['roofline'].get('frac'))"
done
