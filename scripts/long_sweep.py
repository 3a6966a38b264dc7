"""Time one pair (n, m = 262144) for several n: separates per-step cost from link/fill cost."""
import sys, os, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_05708_b200 as ffd
m = 262144
rng = np.random.default_rng(1)
q = np.cumsum(rng.normal(size=(m, 2)), 0).astype(np.float32)
qd = torch.from_numpy(q).cuda()
for n in [32, 128, 224, 512, 1024, 2048, 8192, 32768, 131072, 262144]:
    p = np.cumsum(rng.normal(size=(n, 2)), 0).astype(np.float32)
    pd = torch.from_numpy(p).cuda()
    off = torch.tensor([0, 0], dtype=torch.int64, device="cuda")
    lens = torch.tensor([n, m], dtype=torch.int32, device="cuda")
    for _ in range(2):
        ffd.batch(pd, qd, off, lens, norm="l2")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        out = ffd.batch(pd, qd, off, lens, norm="l2")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(json.dumps({"n": n, "ms": round(ms, 3), "ns_per_col": round(ms * 1e6 / m, 2),
                      "gcells": round(n * m / ms / 1e6, 1)}), flush=True)
