set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2a_pytest.log
python bench.py --steps 20 --warmup 3 > gpurun_out/r2a_bench_c2.json 2> gpurun_out/r2a_bench_c2.err; echo rc=$?
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_c4.json 2>&1; echo rc=$?
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_c5.json 2>&1; echo rc=$?
python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_c3.json 2>&1; echo rc=$?
