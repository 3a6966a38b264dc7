mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_batch_gpu.py -x -q -k "host" > gpurun_out/pytest_host.log 2>&1; echo "host tests rc=$?"; tail -3 gpurun_out/pytest_host.log
timeout 600 python bench.py > gpurun_out/r1_bench_default_v10.json 2> gpurun_out/c2.err; echo "c2 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r1_bench_default_v10.json').read().splitlines()[-1])
print(d['value'], d['e2e'])"
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_c3_v10.json 2> gpurun_out/c3.err; echo "c3 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r1_bench_c3_v10.json').read().splitlines()[-1])
print(d['value'], d['e2e'])"
