mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; grep -c watchdog gpurun_out/pytest_gpu.log
for c in 2 3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_c$c.json'));print('c$c',d['value'],d['roofline']['frac'])"; done
timeout 1200 python scripts/paper_sweeps.py > gpurun_out/r1_paper_sweeps.jsonl 2>&1; echo "sweeps rc=$?"; grep -c watchdog gpurun_out/r1_paper_sweeps.jsonl; grep '"E2"' gpurun_out/r1_paper_sweeps.jsonl | cut -c1-160
