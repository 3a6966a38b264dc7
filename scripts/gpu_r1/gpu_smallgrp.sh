mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_sg.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_sg.log
timeout 900 python scripts/paper_sweeps.py --oracle-pairs 4 > gpurun_out/r1_paper_sweeps_v4.jsonl 2> gpurun_out/sweeps.err; echo "sweeps rc=$?"
python -c "
import json
for l in open('gpurun_out/r1_paper_sweeps_v4.jsonl'):
    d=json.loads(l); print(d['exp'], d['N'], d['P'], d['gpu_gcells_per_s'], d['parity_1e-5'], d['dp_over_sumd_sql2'])"
