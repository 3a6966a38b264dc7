mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_dtw_gpu.py -x -q > gpurun_out/pytest_dtw.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_dtw.log
timeout 600 python scripts/bench_dtw.py > gpurun_out/r1_bench_dtw_v2.jsonl 2> gpurun_out/dtw.err; echo "dtw rc=$?"; cat gpurun_out/r1_bench_dtw_v2.jsonl
