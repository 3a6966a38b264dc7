mkdir -p gpurun_out
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo "bench c5 rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_c5.json'));r=d['roofline'];print(d['value'],r['achieved'],r['kernel_ms'],{k:v['kernel_ms'] for k,v in r['per_norm'].items()},d['results'])"; tail -2 gpurun_out/bench_c5.err
timeout 600 python -m pytest tests/test_longpair_gpu.py tests/test_batch_gpu.py -m gpu -q -x --timeout 120 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_lb.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_lb.log
