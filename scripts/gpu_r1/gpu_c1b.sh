mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_c1b.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_c1b.log
timeout 600 python bench.py --config 1 --steps 200 --warmup 3 > gpurun_out/r1_bench_c1_v8.json 2> gpurun_out/c1.err; echo "c1 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r1_bench_c1_v8.json').read().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['gpu_launches_per_step'], d.get('graph_replay'), d['roofline']['kernel_ms'], d['e2e'])"
timeout 600 python bench.py > gpurun_out/r1_bench_default_v8.json 2> gpurun_out/c2.err; echo "c2 rc=$?"; cut -c1-300 gpurun_out/r1_bench_default_v8.json
