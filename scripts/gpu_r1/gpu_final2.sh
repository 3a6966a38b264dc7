# final round check: GPU tests, smoke, every bench line (V), launch list + ncu of c2
mkdir -p gpurun_out
V=${V:-v11}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest_gpu_$V.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r1_pytest_gpu_$V.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$V.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$V.log
V=$V bash scripts/gpu_final.sh
