"""Probe: segmented two-column streaming (the cdist kernel) vs the batch kernel on
uniform shapes, to size a segmented batch kernel.  Prints JSON lines."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_05708_b200 as ffd

dev = torch.device("cuda", 0)
g = torch.Generator(device="cpu").manual_seed(1)


def walk(n, L, D=2):
    return torch.cumsum(torch.randn(n, L, D, generator=g), dim=1).float().to(dev)


def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


for lenA, lenB, shape in [(128, 128, "4,32"), (128, 128, "8,16"), (256, 256, "16,16"), (256, 256, "32,12"),
                          (384, 256, "32,12"), (512, 256, "32,16"), (192, 256, "16,12")]:
    os.environ["FFD_CDIST_SHAPE"] = shape
    nA, nB = 4096, 2048
    A, B = walk(nA, lenA), walk(nB, lenB)
    ms = timeit(lambda: ffd.cdist(A, B, norm="l2"))
    cells = nA * nB * lenA * lenB
    print(json.dumps({"probe": "cdist", "shape": shape, "lenA": lenA, "lenB": lenB, "ms": ms,
                      "gcells": cells / ms / 1e6}), flush=True)
os.environ.pop("FFD_CDIST_SHAPE", None)
for n, m in [(128, 128), (256, 256), (384, 256), (512, 256)]:
    P = 100000
    p, q = walk(P, n).reshape(-1, 2), walk(P, m).reshape(-1, 2)
    offs = torch.cat([torch.arange(P) * n, torch.arange(P) * m]).to(torch.int64).to(dev)
    lens = torch.cat([torch.full((P,), n), torch.full((P,), m)]).to(torch.int32).to(dev)
    ms = timeit(lambda: ffd.batch(p, q, offs, lens, norm="l2", validate=False))
    print(json.dumps({"probe": "batch", "n": n, "m": m, "ms": ms, "gcells": P * n * m / ms / 1e6}), flush=True)
