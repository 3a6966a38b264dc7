# segmented batch kernel: parity tests, then c2 with and without it
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_seg_gpu.py -x -q > gpurun_out/seg_tests.log 2>&1; echo "seg tests rc=$?"; tail -15 gpurun_out/seg_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist > gpurun_out/seg_c2.json 2>gpurun_out/seg_c2.err; echo "c2 seg rc=$?"; cut -c1-600 gpurun_out/seg_c2.json; tail -3 gpurun_out/seg_c2.err
FFD_SEG=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist > gpurun_out/seg_c2_off.json 2>&1; echo "c2 noseg rc=$?"; cut -c1-300 gpurun_out/seg_c2_off.json
python scripts/seg_probe.py > gpurun_out/seg_probe2.jsonl 2>&1; grep batch gpurun_out/seg_probe2.jsonl
