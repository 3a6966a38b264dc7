"""DTW throughput (ffd_batch_dtw) on config-3-shaped inputs:
3-D fp32 Gaussian walks, lengths U[256,1024], L2 (sqrt per cell) and sq-L2, plus
the config-2 shape as fp32.  Prints one JSON line per case (cells/s, kernel ms)."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_05708_b200 as ffd
import workload

def case(cfg, norm, steps=5):
    b = workload.gen_batch(cfg)
    p = torch.from_numpy(b.p.astype(np.float32)).cuda()
    q = torch.from_numpy(b.q.astype(np.float32)).cuda()
    off = torch.from_numpy(b.offsets).cuda(); lens = torch.from_numpy(b.lengths).cuda()
    for _ in range(3):
        ffd.dtw_batch(p, q, off, lens, norm=norm)
    torch.cuda.synchronize()
    ffd.profile_take(); ffd.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        ffd.dtw_batch(p, q, off, lens, norm=norm)
    e1.record(); torch.cuda.synchronize(); ffd.profile_enable(False)
    kms, n = ffd.profile_take()
    ms = e0.elapsed_time(e1) / steps
    cells = b.cells()
    print(json.dumps({"case": f"dtw_{cfg.name}_{norm}", "pairs": b.num_pairs, "cells": cells, "ms_per_call": ms,
                      "kernel_ms": kms / max(n, 1), "gcells_per_s": cells / (kms / max(n, 1)) / 1e6}), flush=True)

case(workload.CONFIGS[3].scaled(pairs=100_000), "l2")
case(workload.CONFIGS[3].scaled(pairs=100_000), "sql2")
