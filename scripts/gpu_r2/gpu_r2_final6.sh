# round-2 final refresh v6 (ffd_batch_maxlen, AbortPoll): GPU tests, smoke, every bench line, c2 launch list
# c2 launch list, ncu --set full of the c5 long kernel (L2)
mkdir -p gpurun_out
V=${V:-v6}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu_$V.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest_gpu_$V.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_$V.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_smoke_$V.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/r2_clocks_$V.csv &
SMI=$!
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench_default_$V.json 2> gpurun_out/r2_bench_default_$V.err; echo "default rc=$?"
for c in 1 3 5; do
  st=5; [ $c = 1 ] && st=200
  timeout 900 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/r2_bench_c${c}_$V.json 2> gpurun_out/r2_bench_c$c.err; echo "c$c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2_bench_reference_$V.json 2>&1; echo "ref rc=$?"
kill $SMI
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cdist"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r2_c2_launches_$V.csv $CMD > gpurun_out/r2_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for f in gpurun_out/r2_bench_*_$V.json; do echo $f; cut -c1-250 $f; done
