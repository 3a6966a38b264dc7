# long kernel with four columns per step: correctness first (short timeouts), then c5 at several R
timeout 300 python -m pytest tests/test_longpair_gpu.py -x -q -k "f32 or int_exact or rows_per_lane or many" > gpurun_out/r2i_long.log 2>&1; echo "long rc=$?"; tail -2 gpurun_out/r2i_long.log
for r in 0 8 16; do
  FFD_LONG_R=$r timeout 200 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_c5_r$r.json 2>&1; echo "c5 R=$r rc=$?"
done
timeout 600 python -m pytest tests/test_longpair_gpu.py -x -q > gpurun_out/r2i_long_all.log 2>&1; echo "long all rc=$?"; tail -2 gpurun_out/r2i_long_all.log
