mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_longpair_gpu.py -m gpu -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_long.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_long.log
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_c5.json'));print(d['value'],{k:round(v['kernel_ms'],2) for k,v in d['roofline']['per_norm'].items()},d['results'])"
python scripts/long_sweep.py 2>&1 | tail -6
