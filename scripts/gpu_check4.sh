# GPU tests + c2/c3/c5 benches + ncu of c2 and c5 kernels
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
for c in 2 3 5 4; do
  st=5; [ $c = 4 ] && st=2
  timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  echo "bench c$c rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_c$c.json'));r=d['roofline'];print(d['value'],r['achieved'],r['frac'],r['kernel_ms'],d['clocks'],r.get('per_norm',''))"; tail -2 gpurun_out/bench_c$c.err
done
if [ "${NCU:-1}" = 1 ]; then
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -s 6 -c 1 \
  -o gpurun_out/c2_batch_full $CMD > gpurun_out/ncu_c2.log 2>&1
echo "ncu c2 rc=$?"
CMD5="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD5 > gpurun_out/ncu_plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:long_kernel -s 4 -c 1 \
  -o gpurun_out/c5_long_full $CMD5 > gpurun_out/ncu_c5.log 2>&1
echo "ncu c5 rc=$?"
fi
