# Σd upper-limit kernel: parity, the full GPU suite (after the R-set trim), sweeps, default bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_ds.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_ds.log
timeout 900 python scripts/paper_sweeps.py --oracle-pairs 4 > gpurun_out/r1_paper_sweeps_v2.jsonl 2> gpurun_out/sweeps.err; echo "sweeps rc=$?"
cut -c1-400 gpurun_out/r1_paper_sweeps_v2.jsonl; tail -3 gpurun_out/sweeps.err
timeout 600 python bench.py > gpurun_out/r1_bench_default_v6.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cut -c1-600 gpurun_out/r1_bench_default_v6.json
