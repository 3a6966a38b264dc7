# DTW long path + stream lead: DTW/long/batch tests, c5 timing
timeout 600 python -m pytest tests/test_dtw_gpu.py tests/test_longpair_gpu.py -x -q > gpurun_out/r2n_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2n_tests.log
timeout 120 python scripts/c5_launches.py 3 > gpurun_out/r2n_c5.json 2>&1; echo "c5 rc=$?"; cut -c1-600 gpurun_out/r2n_c5.json
