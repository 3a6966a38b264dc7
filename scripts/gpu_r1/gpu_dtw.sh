mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python scripts/bench_dtw.py > gpurun_out/bench_dtw.jsonl 2>&1; echo "dtw bench rc=$?"; cat gpurun_out/bench_dtw.jsonl
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print(d['value'], d['roofline']['frac'])"
