mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/bench_cdist_self.py > gpurun_out/r1_bench_cdist_self.json 2>&1; cat gpurun_out/r1_bench_cdist_self.json
