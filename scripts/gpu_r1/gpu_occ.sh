mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for c in 2 3 1; do st=5; [ $c = 1 ] && st=200; timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_c$c.json'));print('c$c',d['value'],d['ms_per_step'],d['roofline']['frac'])"; done
timeout 900 python scripts/paper_sweeps.py --max-exp 13 > gpurun_out/sw.jsonl 2>&1; grep -E '"N": (16384|8192|1024), "P": 1024|"P": (2048|8192)' gpurun_out/sw.jsonl | cut -c1-140
