# round-2 closing check of HEAD with a fresh build: GPU tests, smoke, default bench line
mkdir -p gpurun_out
V=${V:-v7}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu_$V.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest_gpu_$V.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_$V.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_smoke_$V.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench_default_$V.json 2> gpurun_out/r2_bench_default_$V.err; echo "default rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2_bench_reference_$V.json 2>&1; echo "ref rc=$?"
for f in gpurun_out/r2_bench_*_$V.json; do echo $f; cut -c1-400 $f; done
