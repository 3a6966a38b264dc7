mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_batch_gpu.py -m gpu -q -x -s --timeout 120 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_batch_wd.log 2>&1; echo "rc=$?"; grep -a "watchdog" gpurun_out/pytest_batch_wd.log | head -20; tail -5 gpurun_out/pytest_batch_wd.log
