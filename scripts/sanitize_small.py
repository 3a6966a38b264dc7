"""Small end-to-end exercise of every kernel for compute-sanitizer memcheck:
batch (fp32, int32 incl. the exact int64 tier, multi-band), DTW, cdist, cdist_self,
and long pairs (cluster links)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_05708_b200 as ffd

rng = np.random.default_rng(0)
def batch(lens, dim=2, kind="f", scale=1):
    B = len(lens) // 2
    lens = np.asarray(lens, np.int32)
    off = np.zeros(2 * B, np.int64); off[1:B] = np.cumsum(lens[:B - 1]); off[B + 1:] = np.cumsum(lens[B:-1])
    if kind == "i":
        p = (np.cumsum(rng.integers(-8, 9, size=(int(lens[:B].sum()), dim)), 0) * scale).astype(np.int32)
        q = (np.cumsum(rng.integers(-8, 9, size=(int(lens[B:].sum()), dim)), 0) * scale).astype(np.int32)
    else:
        p = np.cumsum(rng.normal(size=(int(lens[:B].sum()), dim)), 0).astype(np.float32)
        q = np.cumsum(rng.normal(size=(int(lens[B:].sum()), dim)), 0).astype(np.float32)
    return [torch.from_numpy(a).cuda() for a in (p, q, off, lens)]

a = batch(list(rng.integers(1, 700, 80)))
print(ffd.batch(*a, norm="l2").sum().item())
print(ffd.dtw_batch(*a, norm="l2").sum().item())
a = batch(list(rng.integers(1, 600, 80)), kind="i", scale=3000)
print(ffd.batch(*a, norm="sql2").sum().item())
a = batch([3000, 40, 2500, 3100, 50, 3000])          # long pairs (n > one band, m > scratch? no) + short
print(ffd.batch(*a, norm="l2").cpu().numpy())
a = batch([9000, 9500])                               # long-pair kernel
print(ffd.batch(*a, norm="l2").cpu().numpy())
A = torch.from_numpy(np.cumsum(rng.normal(size=(50, 40, 2)), 1).astype(np.float32)).cuda()
B = torch.from_numpy(np.cumsum(rng.normal(size=(70, 37, 2)), 1).astype(np.float32)).cuda()
print(ffd.cdist(A, B).sum().item(), ffd.cdist_self(A).sum().item())
torch.cuda.synchronize()
print("ok")
