mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python scripts/bench_dtw.py > gpurun_out/r1_bench_dtw.jsonl 2>&1; echo "dtw bench rc=$?"; cat gpurun_out/r1_bench_dtw.jsonl
timeout 1200 python scripts/paper_sweeps.py > gpurun_out/r1_paper_sweeps.jsonl 2> gpurun_out/r1_paper_sweeps.err; echo "sweeps rc=$?"; cat gpurun_out/r1_paper_sweeps.jsonl; tail -3 gpurun_out/r1_paper_sweeps.err
