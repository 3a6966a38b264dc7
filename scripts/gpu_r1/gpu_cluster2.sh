mkdir -p gpurun_out
for c in 2 4 8 1; do
  echo "== FFD_LONG_CLUSTER=$c"
  FFD_LONG_CLUSTER=$c timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b5_$c.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/b5_$c.json'));print(d['value'],{k:round(v['kernel_ms'],2) for k,v in d['roofline']['per_norm'].items()},d['results'])"
done
