# re-entry check: GPU tests + default bench + c5 bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2s_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2s_pytest.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r2s_default.json 2> gpurun_out/r2s_default.err; echo "default rc=$?"
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/r2s_c5.json 2> gpurun_out/r2s_c5.err; echo "c5 rc=$?"
for f in gpurun_out/r2s_*.json; do echo $f; cut -c1-400 $f; done
