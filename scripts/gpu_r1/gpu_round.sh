set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r1_pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r1_bench_c2.json 2> gpurun_out/r1_bench_c2.err; echo "bench rc=$?"
cat gpurun_out/r1_bench_c2.json
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_c4.json 2> gpurun_out/r1_bench_c4.err; echo "bench4 rc=$?"
cat gpurun_out/r1_bench_c4.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_c2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1_ncu_launch.log 2>&1; echo "ncu rc=$?"
