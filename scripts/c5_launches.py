"""Per-launch device time of the config-5 long pair (each norm, several calls),
CUDA events around each ffd_batch call: shows run-to-run variance of the
long-pair kernel.  Usage: python scripts/c5_launches.py [calls] [norms, e.g. l2,l1]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_05708_b200 as ffd  # noqa: E402
import workload  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = workload.CONFIGS[5]
p_h, q_h = workload.gen_long_pair(cfg)
p, q = torch.from_numpy(p_h).cuda(), torch.from_numpy(q_h).cuda()
off = torch.tensor([0, 0], dtype=torch.int64, device="cuda")
lens = torch.tensor([p.shape[0], q.shape[0]], dtype=torch.int32, device="cuda")
out = torch.empty(1, device="cuda")
res = {"R": os.environ.get("FFD_LONG_R", "auto")}
norms = sys.argv[2].split(",") if len(sys.argv) > 2 else cfg.norms
for nm in norms:
    ffd.batch(p, q, off, lens, norm=nm, out=out, validate=False)
    ts = []
    for _ in range(calls):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ffd.batch(p, q, off, lens, norm=nm, out=out, validate=False)
        b.record()
        torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(b), 3))
    res[nm] = {"ms": ts, "value": float(out.item()), "gcells": p.shape[0] * q.shape[0] / (np.median(ts) * 1e-3) / 1e9}
print(json.dumps(res))
