# GPU tests + bench lines for all configs (round-1 check)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-2 5 3 4}; do
  st=5; [ $c = 4 ] && st=2; [ $c = 1 ] && st=200
  timeout 900 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  echo "bench c$c rc=$?"; cut -c1-1200 gpurun_out/bench_c$c.json; tail -3 gpurun_out/bench_c$c.err
done
