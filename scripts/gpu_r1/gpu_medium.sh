mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_longpair_gpu.py tests/test_dtw_gpu.py -x -q -k "medium" > gpurun_out/pytest_medium.log 2>&1; echo "medium rc=$?"; tail -15 gpurun_out/pytest_medium.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_med.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_med.log
timeout 900 python scripts/paper_sweeps.py --oracle-pairs 4 > gpurun_out/r1_paper_sweeps_v3.jsonl 2> gpurun_out/sweeps.err; echo "sweeps rc=$?"
python -c "
import json
for l in open('gpurun_out/r1_paper_sweeps_v3.jsonl'):
    d=json.loads(l); print(d['exp'], d['N'], d['P'], d['gpu_gcells_per_s'], d['parity_1e-5'], d['dp_over_sumd_sql2'])"
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c5med.json 2> gpurun_out/c5med.err; echo "c5 rc=$?"; cut -c1-250 gpurun_out/c5med.json
