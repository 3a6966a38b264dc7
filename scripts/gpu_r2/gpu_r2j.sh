# four columns per step, bank-conflict-free ring: per-launch c5 times at several R, then the long tests
for r in 0 8 16; do FFD_LONG_R=$r timeout 120 python scripts/c5_launches.py 5 >> gpurun_out/r2j_c5.jsonl 2>&1; echo "R=$r rc=$?"; done
cat gpurun_out/r2j_c5.jsonl
timeout 600 python -m pytest tests/test_longpair_gpu.py -x -q > gpurun_out/r2j_long.log 2>&1; echo "long rc=$?"; tail -2 gpurun_out/r2j_long.log
