mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/r1_bench_c5_v5.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/r1_bench_c5_v5.json'));print(d['value'],{k:(round(v['kernel_ms'],2),round(v['frac'],3)) for k,v in d['roofline']['per_norm'].items()},d['results'])"
python scripts/long_sweep.py 2>&1 | tail -4
