# long kernel: coarse (1 us) naps until the producer's first position, then the fine poll; long/DTW tests + c5 bench x2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_longpair_gpu.py tests/test_dtw_gpu.py -x -q > gpurun_out/coarse_tests.log 2>&1; echo "long+dtw tests rc=$?"; tail -1 gpurun_out/coarse_tests.log
for i in 1 2; do
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/coarse_c5_$i.json 2>gpurun_out/coarse_c5.err; echo "c5 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/coarse_c5_$i.json')); print(d['ms_per_step'], d['value'], d['roofline'].get('frac'), d['clocks'])"
done
