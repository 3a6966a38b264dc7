# config 5 with 7 band slots per CTA (R = 8: 1024 bands on 147 CTAs) against the default 8 (R = 7)
mkdir -p gpurun_out
FFD_LIB=paper_2404_05708_b200/libffd_w7.so timeout 900 python -m pytest tests/test_longpair_gpu.py -x -q > gpurun_out/w7_tests.log 2>&1; echo "w7 long tests rc=$?"; tail -1 gpurun_out/w7_tests.log
for lib in libffd.so libffd_w7.so; do
FFD_LIB=paper_2404_05708_b200/$lib timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/w7_c5_$lib.json 2>gpurun_out/w7_c5.err; echo "c5 $lib rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/w7_c5_$lib.json')); print(d['ms_per_step'], d['value'], d['roofline'].get('frac'), d['roofline'].get('per_norm_ms') or '')"
done
