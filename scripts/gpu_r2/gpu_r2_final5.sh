# after ffd_batch_sized (c1) and the rate-limited abort reads in the long kernel's spins: GPU tests, c1/c5/default bench
mkdir -p gpurun_out
V=${V:-v5}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu_$V.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest_gpu_$V.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_$V.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_smoke_$V.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/r2_clocks_$V.csv &
SMI=$!
timeout 900 python bench.py --config 1 --steps 200 --warmup 3 > gpurun_out/r2_bench_c1_$V.json 2> gpurun_out/r2_bench_c1_$V.err; echo "c1 rc=$?"
for i in 1 2; do
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/r2_bench_c5_${V}_$i.json 2> gpurun_out/r2_bench_c5_$V.err; echo "c5 rc=$?"
done
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench_default_$V.json 2> gpurun_out/r2_bench_default_$V.err; echo "default rc=$?"
kill $SMI
for f in gpurun_out/r2_bench_*_$V*.json; do echo $f; python -c "
import json,sys; d=json.load(open('$f')); print(d['ms_per_step'], d['value'], d.get('gpu_launches'), (d.get('graph_replay') or {}).get('ms_per_step'), (d.get('roofline') or {}).get('frac'), d.get('clocks'))"; done
