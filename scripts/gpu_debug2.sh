mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python -m pytest tests/test_batch_gpu.py -m gpu -q -x --timeout 120 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_batch_$i.log 2>&1; echo "pytest batch run $i rc=$?"; tail -3 gpurun_out/pytest_batch_$i.log
done
timeout 300 python -m pytest tests/test_batch_gpu.py -m gpu -q -x --timeout 120 --timeout-method=thread -p no:cacheprovider -k "odd_even" > gpurun_out/pytest_oddeven.log 2>&1; echo "oddeven alone rc=$?"; tail -3 gpurun_out/pytest_oddeven.log
