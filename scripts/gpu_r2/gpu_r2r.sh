# compact one-column window loop (libffd_cw.so) vs the default: c2 timing + parity
cd paper_2404_05708_b200
FFD_LIB=$PWD/libffd_cw.so timeout 300 python -m pytest ../tests/test_batch_gpu.py -x -q -k "not dims" > ../gpurun_out/r2r_tests.log 2>&1; echo "cw tests rc=$?"; tail -1 ../gpurun_out/r2r_tests.log
cd ..
for v in "" _cw "" _cw; do
  FFD_LIB=$PWD/paper_2404_05708_b200/libffd$v.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cdist > gpurun_out/r2r_c2$v.json 2>&1; echo "lib$v rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/r2r_c2$v.json').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3))"
done
