timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_cdist_gpu.py tests/test_batch_gpu.py tests/test_abi.py -x -q > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2c_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --gpus 1 --spawn --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_bench_spawn.json 2> gpurun_out/r2c_bench_spawn.err; echo "spawn rc=$?"
