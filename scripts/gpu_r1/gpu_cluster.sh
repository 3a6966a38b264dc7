mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_longpair_gpu.py -q -x -m gpu --timeout 300 --timeout-method=thread -p no:cacheprovider 2>&1 | tail -2
for c in 8 1; do
  echo "== FFD_LONG_CLUSTER=$c"
  FFD_LONG_CLUSTER=$c python scripts/trace_long.py 131072 > gpurun_out/tr_$c.txt 2>&1; head -c 300 gpurun_out/tr_$c.txt; echo
  FFD_LONG_CLUSTER=$c timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b5_$c.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/b5_$c.json'));print(d['value'],{k:round(v['kernel_ms'],2) for k,v in d['roofline']['per_norm'].items()},d['results'])"
done
