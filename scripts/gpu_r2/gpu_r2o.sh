# cdist with two columns per step: parity, then c4 timing for 1/2 columns and two shapes
timeout 600 python -m pytest tests/test_cdist_gpu.py tests/test_dist_gpu.py -x -q > gpurun_out/r2o_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2o_tests.log
for cols in 1 2; do for shape in "4,32" "8,16"; do
  FFD_CDIST_COLS=$cols FFD_CDIST_SHAPE=$shape timeout 300 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2o_c4_${cols}_${shape}.json 2>&1; echo "cols=$cols shape=$shape rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/r2o_c4_${cols}_${shape}.json').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['roofline']['kernel_ms'],2), round(d['roofline']['frac'],3))"
done; done
