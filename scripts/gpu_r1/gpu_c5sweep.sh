mkdir -p gpurun_out
for g in 148 128 74 64 32; do
  FFD_LONG_CTAS=$g timeout 600 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_g$g.json 2> gpurun_out/bench_c5_g$g.err
  echo "G=$g rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_c5_g$g.json'));r=d['roofline'];print({k:round(v['kernel_ms'],2) for k,v in r['per_norm'].items()}, d['results'])"
done
