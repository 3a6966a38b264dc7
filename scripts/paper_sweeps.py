"""The paper's own experiment shapes on B200.

E1: N curves p_i against ONE curve q (the one-vs-many batch of PAPER L259, expressed
    through ffd_batch's offsets: every q offset is 0, no copy), N = 2^5 .. 2^14,
    P = Q = 2^10, 2-D, steps uniform in {−1, 0, +1}², L2, fp32.
E2: N = 2^10, P = Q = 2^5 .. 2^13 (2^14 needs the long-pair path pair by pair).

For each point: the Σ_ij d_ij "upper limit" kernel (ffd_dist_sum, PAPER L300,
L304–L305) timed beside the DP, with a root per cell (the paper's hypot) and
without (the DP's own squared distance); GPU kernel time (CUDA events, after warm-up, as PAPER L277) and the
CPU oracle (the plain fp64 table, OpenMP over pairs) on a bounded number of the
same pairs — the paper's "relative improvement" axis (Fig. 1/2, whose data is
missing from PAPER.md) restated as GPU / oracle cells/s.  Prints JSON lines.

    python scripts/paper_sweeps.py [--max-exp 14] [--oracle-pairs 8]
"""
import argparse
import json
import os
import sys
import time

# the oracle's OpenMP threads must not spin on every core after each parallel
# region: they starved the host thread that enqueues the next point's GPU work
# (two E1/E2 points read 35 % low in r1_paper_sweeps_v5.jsonl)
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workload  # noqa: E402


def one_vs_many(N, P, Q, seed_first=0):
    """N unit-step walks of length P (p) and one of length Q (q), batch layout."""
    cfg = workload.CONFIGS[101].scaled(pairs=N, len_p=(P, P), len_q=(Q, Q))
    b = workload.gen_batch(cfg, first=seed_first)
    q = b.q[:Q].copy()                       # the single reference curve
    offsets = np.concatenate([b.offsets[:N], np.zeros(N, np.int64)])
    return b.p, q, offsets, b.lengths


def time_gpu(ffd, torch, p, q, off, lens, reps, fn="batch", norm="l2"):
    args = [torch.from_numpy(a).cuda() for a in (p, q, off, lens)]
    call = getattr(ffd, fn)
    # the GPU idles (and its clocks drop) while the CPU oracle runs between
    # points: keep it busy for ≥ 0.3 s before timing, and time ≥ 50 ms of calls
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    call(*args, norm=norm)
    e1.record()
    torch.cuda.synchronize()
    est = max(e0.elapsed_time(e1), 1e-3)
    for _ in range(max(3, int(300 / est))):
        call(*args, norm=norm)
    reps = max(reps, int(50 / est))
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        out = call(*args, norm=norm)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out.cpu().numpy()


def time_oracle(p, q, off, lens, k, threads):
    import oracle
    B = len(lens) // 2
    sel = np.arange(min(k, B))
    offs = np.concatenate([off[sel], off[B + sel]])
    ln = np.concatenate([lens[sel], lens[B + sel]])
    t0 = time.perf_counter()
    ref = oracle.batch(p, q, offs, ln, 2, "l2", threads=threads)
    return time.perf_counter() - t0, ref, sel


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-exp", type=int, default=14)
    ap.add_argument("--oracle-pairs", type=int, default=16)
    args = ap.parse_args()
    import torch
    import paper_2404_05708_b200 as ffd
    ffd.lib()
    threads = len(os.sched_getaffinity(0))
    points = [("E1", 2 ** e, 1024, 1024) for e in range(5, args.max_exp + 1)]
    points += [("E2", 1024, 2 ** e, 2 ** e) for e in range(5, min(args.max_exp, 13) + 1)]
    for exp, N, P, Q in points:
        p, q, off, lens = one_vs_many(N, P, Q)
        cells = N * P * Q
        ms, got = time_gpu(ffd, torch, p, q, off, lens, reps=5 if cells > 1e10 else 20)
        k = max(1, min(N, int(args.oracle_pairs * (1024 * 1024) / (P * Q))))
        t_cpu, ref, sel = time_oracle(p, q, off, lens, k, threads)
        ok = bool(np.all(np.abs(got[sel] - ref) <= 1e-5 * np.abs(ref)))
        gpu = cells / (ms * 1e-3) / 1e9
        cpu = len(sel) * P * Q / t_cpu / 1e9
        # the paper's "upper limit": Σ_ij d_ij alone, with
        # a root per cell (its hypot workload) and without (the DP's own d here)
        reps = 5 if cells > 1e10 else 20
        ms_l2, s_l2 = time_gpu(ffd, torch, p, q, off, lens, reps, "dist_sum", "l2")
        ms_sq, _ = time_gpu(ffd, torch, p, q, off, lens, reps, "dist_sum", "sql2")
        import oracle
        offs = np.concatenate([off[sel[:2]], off[N + sel[:2]]])
        ln = np.concatenate([lens[sel[:2]], lens[N + sel[:2]]])
        ref_s = oracle.dist_sum_batch(p, q, offs, ln, 2, "l2")
        ok_s = bool(np.all(np.abs(s_l2[sel[:2]] - ref_s) <= 39 * 2.0 ** -24 * ref_s))
        print(json.dumps({"exp": exp, "N": N, "P": P, "Q": Q, "cells": cells, "gpu_ms": round(ms, 4),
                          "gpu_gcells_per_s": round(gpu, 2), "oracle_gcells_per_s": round(cpu, 3),
                          "oracle_threads": threads, "oracle_pairs": int(len(sel)),
                          "gpu_over_oracle": round(gpu / cpu, 1), "parity_1e-5": ok,
                          "sumd_l2_gcells_per_s": round(cells / (ms_l2 * 1e-3) / 1e9, 2),
                          "sumd_sql2_gcells_per_s": round(cells / (ms_sq * 1e-3) / 1e9, 2),
                          "dp_over_sumd_sql2": round(ms_sq / ms, 3), "sumd_parity": ok_s}), flush=True)


if __name__ == "__main__":
    main()
