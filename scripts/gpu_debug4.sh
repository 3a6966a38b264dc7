mkdir -p gpurun_out
for i in 1 2 3; do
timeout 600 python -m pytest tests -m gpu -q -x --timeout 120 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_all_$i.log 2>&1; echo "run $i rc=$?"; grep -a "watchdog" gpurun_out/pytest_all_$i.log | head -5; tail -2 gpurun_out/pytest_all_$i.log
done
