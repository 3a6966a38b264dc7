timeout 900 python -m pytest tests/test_longpair_gpu.py -x -q > gpurun_out/r2b_long.log 2>&1; echo "long rc=$?"
tail -5 gpurun_out/r2b_long.log
timeout 600 python -m pytest tests -m gpu -x -q --deselect tests/test_longpair_gpu.py > gpurun_out/r2b_gpu.log 2>&1; echo "gpu rc=$?"
tail -3 gpurun_out/r2b_gpu.log
timeout 300 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_c5.json 2>&1; echo "c5 rc=$?"
