mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; grep -c watchdog gpurun_out/pytest_gpu.log
timeout 1200 python scripts/paper_sweeps.py > gpurun_out/r1_paper_sweeps.jsonl 2>&1; echo "sweeps rc=$?"; grep -c watchdog gpurun_out/r1_paper_sweeps.jsonl; grep '^{' gpurun_out/r1_paper_sweeps.jsonl | cut -c1-200
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_c5.json'));print(d['value'],{k:round(v['kernel_ms'],2) for k,v in d['roofline']['per_norm'].items()},d['results'])"
