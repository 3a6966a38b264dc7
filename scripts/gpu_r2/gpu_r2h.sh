# compact two-column step loop: smoke, batch tests, c2 bench, ncu of the batch kernel
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2h_smoke.log
timeout 180 python -m pytest tests/test_batch_gpu.py -x -q > gpurun_out/r2h_batch.log 2>&1; echo "batch rc=$?"; tail -1 gpurun_out/r2h_batch.log
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cdist"
timeout 120 $CMD > gpurun_out/r2h_c2.json 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -s 6 -c 1 -o gpurun_out/r2h_c2 $CMD > gpurun_out/r2h_ncu.log 2>&1; echo "ncu rc=$?"
