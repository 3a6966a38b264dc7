# config 5 with a 4-step steady loop in the long-pair kernel (FFD_LONG_UNROLL=4) against 2
mkdir -p gpurun_out
for lib in libffd.so libffd_u8.so libffd.so libffd_u8.so; do
FFD_LIB=paper_2404_05708_b200/$lib timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/u4_c5.json 2>gpurun_out/u4_c5.err; echo "c5 $lib rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/u4_c5.json')); print(d['ms_per_step'], d['value'], d['roofline'].get('frac'))"
done
FFD_LIB=paper_2404_05708_b200/libffd_u8.so timeout 900 python -m pytest tests/test_longpair_gpu.py -x -q > gpurun_out/u4_tests.log 2>&1; echo "u8 long tests rc=$?"; tail -1 gpurun_out/u4_tests.log
