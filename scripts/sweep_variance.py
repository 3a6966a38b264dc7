import sys, os, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2404_05708_b200 as ffd
sys.path.insert(0, os.path.join(os.getcwd(), 'scripts'))
from paper_sweeps import one_vs_many, time_gpu
for (N, P) in [(4096, 1024), (1024, 2048), (2048, 1024), (4097, 1024)]:
    p, q, off, lens = one_vs_many(N, P, P)
    res = []
    for rep in range(4):
        ms, _ = time_gpu(ffd, torch, p, q, off, lens, 20)
        res.append(round(N * P * P / (ms * 1e-3) / 1e9, 1))
    print(N, P, res, flush=True)
