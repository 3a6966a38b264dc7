# two-column batch path with compact code (libffd_tc.so) vs the default: c2 timing, parity, ncu of tc
cd paper_2404_05708_b200
FFD_LIB=$PWD/libffd_tc.so timeout 300 python -m pytest ../tests/test_batch_gpu.py -x -q -k "int or sql2 or l2 or window or edge" > ../gpurun_out/r2q_tests.log 2>&1; echo "tc tests rc=$?"; tail -1 ../gpurun_out/r2q_tests.log
cd ..
for v in "" _tc; do
  FFD_LIB=$PWD/paper_2404_05708_b200/libffd$v.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cdist > gpurun_out/r2q_c2$v.json 2>&1; echo "lib$v rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/r2q_c2$v.json').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3))"
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cdist"
FFD_LIB=$PWD/paper_2404_05708_b200/libffd_tc.so timeout 300 $CMD > /dev/null 2>&1 && \
FFD_LIB=$PWD/paper_2404_05708_b200/libffd_tc.so timeout 900 ncu --set full --clock-control none -k regex:batch_kernel -s 6 -c 1 -o gpurun_out/r2q_c2_tc $CMD > gpurun_out/r2q_ncu.log 2>&1; echo "ncu rc=$?"
