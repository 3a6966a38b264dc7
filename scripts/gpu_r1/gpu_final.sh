# refresh every bench line (v6), the c2 launch list, one ncu --set full of the c2 batch kernel
mkdir -p gpurun_out
V=${V:-v6}
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/r1_clocks_$V.csv &
SMI=$!
python bench.py > gpurun_out/r1_bench_default_$V.json 2> gpurun_out/bench_default.err; echo "default rc=$?"
for c in 1 3 4 5; do
  st=5; [ $c = 4 ] && st=2; [ $c = 1 ] && st=200
  timeout 900 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/r1_bench_c${c}_$V.json 2> gpurun_out/bench_c$c.err; echo "c$c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r1_bench_reference_$V.json 2>&1; echo "ref rc=$?"
kill $SMI
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r1_c2_launches_$V.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch_kernel -s 6 -c 1 -o gpurun_out/r1_c2_batch_$V $CMD > gpurun_out/ncu_c2.log 2>&1; echo "ncu full rc=$?"
for f in gpurun_out/r1_bench_*_$V.json; do echo $f; cut -c1-400 $f; done
