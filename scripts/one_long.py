"""One pair (n, 262144) for profiling the long-pair kernel in isolation."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_05708_b200 as ffd
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = 262144
rng = np.random.default_rng(1)
p = torch.from_numpy(np.cumsum(rng.normal(size=(n, 2)), 0).astype(np.float32)).cuda()
q = torch.from_numpy(np.cumsum(rng.normal(size=(m, 2)), 0).astype(np.float32)).cuda()
off = torch.tensor([0, 0], dtype=torch.int64, device="cuda")
lens = torch.tensor([n, m], dtype=torch.int32, device="cuda")
for _ in range(3):
    out = ffd.batch(p, q, off, lens, norm="l2")
torch.cuda.synchronize()
print(out.item())
