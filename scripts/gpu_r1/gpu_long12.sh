mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_longpair_gpu.py -x -q -k "config5 or f32 or int_exact" > gpurun_out/pytest_long12.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_long12.log
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c5_12.json 2> gpurun_out/c5_12.err; echo "c5 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/c5_12.json').read().splitlines()[-1])
print(d['value'], d['ms_per_step'], {k:(round(v['kernel_ms'],2), round(v['frac'],3)) for k,v in d['roofline']['per_norm'].items()})"
python scripts/trace_lags.py 262144
