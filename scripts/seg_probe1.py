"""One uniform-shape batch through ffd.batch (for ncu): n m [norm] [int]"""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_05708_b200 as ffd
n, m = int(sys.argv[1]), int(sys.argv[2])
norm = sys.argv[3] if len(sys.argv) > 3 else "l2"
percurve = len(sys.argv) > 4 and sys.argv[4] == "percurve"  # every curve a walk from the origin
P = 100000
dev = torch.device("cuda", 0)
g = torch.Generator().manual_seed(1)
if norm == "sql2":
    p = torch.cumsum(torch.randint(-8, 9, (P * n, 2), generator=g), 0).int().to(dev)
    q = torch.cumsum(torch.randint(-8, 9, (P * m, 2), generator=g), 0).int().to(dev)
elif percurve:
    p = torch.cumsum(torch.randn(P, n, 2, generator=g), 1).reshape(-1, 2).float().to(dev)
    q = torch.cumsum(torch.randn(P, m, 2, generator=g), 1).reshape(-1, 2).float().to(dev)
else:
    p = torch.cumsum(torch.randn(P * n, 2, generator=g), 0).float().to(dev)
    q = torch.cumsum(torch.randn(P * m, 2, generator=g), 0).float().to(dev)
offs = torch.cat([torch.arange(P) * n, torch.arange(P) * m]).to(torch.int64).to(dev)
lens = torch.cat([torch.full((P,), n), torch.full((P,), m)]).to(torch.int32).to(dev)
for _ in range(3):
    ffd.batch(p, q, offs, lens, norm=norm, validate=False)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(5):
    ffd.batch(p, q, offs, lens, norm=norm, validate=False)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
print(json.dumps({"n": n, "m": m, "norm": norm, "ms": ms, "gcells": P * n * m / ms / 1e6}))
