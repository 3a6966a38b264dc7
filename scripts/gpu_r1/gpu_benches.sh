# bench lines for configs 5, 3, 1 + ncu --set full of the c2 main-tier batch kernel
mkdir -p gpurun_out
for c in 5 3 1; do
  st=3; [ $c = 1 ] && st=200
  timeout 900 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/r1_bench_c$c.json 2> gpurun_out/r1_bench_c$c.err
  echo "bench c$c rc=$?"; cat gpurun_out/r1_bench_c$c.json | cut -c1-1500; tail -3 gpurun_out/r1_bench_c$c.err
done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -s 6 -c 1 \
  -o gpurun_out/r1_c2_batch_full $CMD > gpurun_out/r1_ncu_full.log 2>&1
echo "ncu rc=$?"
