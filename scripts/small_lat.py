"""Latency of small ffd_batch calls (config-1 scale) against the pair shape:
separates the fixed per-call cost from the per-step cost of one warp."""
import json, sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_05708_b200 as ffd

def run(B, n, m, reps=300):
    rng = np.random.default_rng(0)
    p = np.cumsum(rng.normal(size=(B * n, 2)), 0).astype(np.float32)
    q = np.cumsum(rng.normal(size=(B * m, 2)), 0).astype(np.float32)
    off = np.concatenate([np.arange(B) * n, np.arange(B) * m]).astype(np.int64)
    ln = np.concatenate([np.full(B, n), np.full(B, m)]).astype(np.int32)
    a = [torch.from_numpy(x).cuda() for x in (p, q, off, ln)]
    out = torch.empty(B, device="cuda")
    for _ in range(5):
        ffd.batch(*a, out=out)
    ffd.profile_take()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ffd.profile_enable(True)
    e0.record()
    for _ in range(reps):
        ffd.batch(*a, out=out)
    e1.record()
    torch.cuda.synchronize()
    ffd.profile_enable(False)
    km, kn = ffd.profile_take()
    print(json.dumps({"B": B, "n": n, "m": m, "us_per_call": round(e0.elapsed_time(e1) / reps * 1e3, 2),
                      "main_kernel_us": round(km / max(kn, 1) * 1e3, 2)}), flush=True)

for B, n, m in [(1, 16, 16), (16, 16, 16), (16, 64, 80), (16, 64, 800), (16, 64, 8000), (16, 640, 80),
                (1, 64, 80), (256, 64, 80), (4096, 64, 80)]:
    run(B, n, m)
