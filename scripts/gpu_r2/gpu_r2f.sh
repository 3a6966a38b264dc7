# two-column batch path: quick smoke first (short timeout), then GPU tests + c2/c3 bench
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2f_smoke.log
timeout 180 python -m pytest tests/test_batch_gpu.py -x -q > gpurun_out/r2f_batch.log 2>&1; echo "batch rc=$?"; tail -2 gpurun_out/r2f_batch.log
timeout 120 python bench.py --steps 20 --warmup 3 --no-cdist --no-cpu-baseline > gpurun_out/r2f_c2.json 2>&1; echo "c2 rc=$?"
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_gpu.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/r2f_gpu.log
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_c3.json 2>&1; echo "c3 rc=$?"
