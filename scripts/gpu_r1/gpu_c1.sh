mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_c1.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_c1.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --config 1 --steps 200 --warmup 3 > gpurun_out/r1_bench_c1_v7.json 2> gpurun_out/c1.err; echo "c1 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r1_bench_c1_v7.json').read().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['gpu_launches_per_step'], d.get('graph_replay'), d['roofline']['kernel_ms'], d['config']['l2'])"
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_c5_v7.json 2> gpurun_out/c5.err; echo "c5 rc=$?"; cut -c1-300 gpurun_out/r1_bench_c5_v7.json
