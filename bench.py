#!/usr/bin/env python
"""Benchmark: DP cells/s of the discrete Fréchet hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ffd|reference]

Default line (config 2 headline + config 4 beside it, the metric's "batched &
all-pairs"):
  * value: one "step" = one ffd_batch call over the whole config-2 batch (100k
    pairs, 2-D int32, lengths U[128,512], squared L2, exact) with inputs resident
    in HBM (512 MB > 126 MB L2: no flush needed).  With N GPUs every rank
    processes its own 100k-pair shard (weak scaling, no data-path collective).
  * all_pairs: config 4 (20k × 20k curves of 128 points, 2-D fp32 L2): rows of A
    sharded over the N ranks, each rank's block by ffd_cdist, then one NCCL
    all_gather_into_tensor of the matrix — INSIDE the timed region (strong
    scaling).  Its own roofline, e2e and cpu_baseline.
Times are CUDA events on the launching stream, max over ranks; rank 0 prints
ONE JSON line.  `--gpus N` without a torchrun environment re-executes itself
under `python -m torch.distributed.run --nproc-per-node N` (127.0.0.1).

--config 1/3/4/5 times that config alone.  --impl reference times the CPU
oracle (oracle/, the plain C table DP) on the host cores on a bounded sample of
the same workload — the slow reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workload  # noqa: E402

METRIC = "DP cells/sec (G cells/s) batched & all-pairs Fréchet; % of ALU roofline"
UNIT = "Gcells/s"
SM_MAX_MHZ_NOMINAL = 1965.0
# ALU roofline (profiles/r2_pipe_model.md): peak cells/s = SMs × 4 SMSPs × 32 lanes ×
# f_SM / (cycles per warp-cell on one SMSP), the cycles being the largest of the cell's ALU-pipe cycles,
# FMA-pipe cycles and issue slots, with the per-instruction pipe costs MEASURED by ncu
# (sm__pipe_alu_cycles_active / sm__pipe_fma_cycles_active of tools/microbench/pipes.cu): FMNMX and FMNMX3
# keep the ALU pipe 2 cycles, FADD2/FMUL2/FFMA2 the FMA pipe 2 cycles, FADD 1.  Every Fréchet cell needs
# min-of-three + max = 4 ALU cycles.
#            cell: (ALU cycles, FMA cycles, issue slots) per warp-cell
PIPE_MODEL = {"xsq_d2": (4, 3, 3.5), "f32_d2_sq": (4, 4, 4), "f32_d3_sq": (4, 6, 5),
              "f32_d2_l1": (4, 3, 4), "f32_d2_linf": (4, 2, 3)}
PEAK_SOURCE = "profiles/r2_pipe_model.md (ncu pipe counters of tools/microbench/pipes.cu)"


def cells_per_clk_per_sm(cell):
    return 4 * 32 / max(PIPE_MODEL[cell])


CELL_OF_CONFIG = {1: "f32_d2_sq", 2: "xsq_d2", 3: "f32_d3_sq", 4: "f32_d2_sq", 5: "f32_d2_sq"}
CELL_OF_NORM = {"l1": "f32_d2_l1", "l2": "f32_d2_sq", "linf": "f32_d2_linf"}
# roofline.traffic (dram bytes per launch of the dominant kernel) is not measurable inside a plain
# run; it is null here, and the ncu --set full captures of the same kernels, with their dram
# bytes against the algorithmic bytes, are committed under profiles/ (named per round).
TRAFFIC_PROFILES = {2: "profiles/r2_traffic_c2.csv", 4: "profiles/r2_c4_cdist_ncu_full.txt",
                    5: "profiles/r2_traffic_c5.csv", 3: "profiles/r2_traffic_c3.csv"}


L2_FLUSH_BELOW = 256 << 20  # inputs smaller than this could stay in L2 (126 MB) between steps


def timed_steps_flushed(torch, stream, dev, fn, steps):
    """ms per step, each step timed alone with CUDA events on `stream` after a
    256 MB write that evicts L2 (the flush itself is outside the timed events)."""
    junk = torch.empty(L2_FLUSH_BELOW // 4, dtype=torch.float32, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in evs:
        junk.fill_(1.0)
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs) / steps


def alu_roofline(cells_per_launch, kernel_ms, cell, sms, f_max, f_meas, kernel, traffic):
    """The roofline object for the dominant kernel."""
    achieved = cells_per_launch / (kernel_ms * 1e-3) / 1e9
    c = cells_per_clk_per_sm(cell)
    alu, fma, issue = PIPE_MODEL[cell]
    peak = sms * c * f_max / 1e9
    return {"bound": "alu", "achieved": achieved, "peak": peak, "unit": UNIT, "frac": achieved / peak,
            "traffic": traffic, "kernel": kernel, "kernel_ms": kernel_ms, "cell": cell,
            "peak_basis": f"{sms} SMs x 128 lanes / max(ALU {alu}, FMA {fma}, issue {issue}) cycles per warp-cell "
                          f"= {c:.2f} cells/clk/SM x {f_max/1e6:.0f} MHz (max SM clock); {PEAK_SOURCE}",
            "frac_at_measured_clock": achieved / (sms * c * f_meas / 1e9)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, index: int, period_s: float = 0.005):
        self.samples = []
        self.reasons = set()
        self.period = period_s
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
            "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_sample(cfg, target_cells: float):
    """First pairs of the workload totalling ≈ target_cells cells (bounded CPU sample)."""
    lp = workload.gen_lengths(cfg, "p")
    lq = workload.gen_lengths(cfg, "q")
    cum = np.cumsum(lp.astype(np.int64) * lq.astype(np.int64))
    k = int(np.searchsorted(cum, target_cells)) + 1
    k = max(1, min(k, cfg.pairs))
    return workload.gen_batch(cfg.scaled(pairs=k)), k


def run_oracle_timed(b, cfg, threads):
    import oracle
    t0 = time.perf_counter()
    oracle.batch(b.p, b.q, b.offsets, b.lengths, b.dim, cfg.norm, threads=threads)
    return time.perf_counter() - t0


def oracle_runner(cfg, target_cells: float, cores: int):
    """(callable timing one oracle pass, cells per pass, sample description) for a
    bounded sample of config `cfg` (batch: leading pairs; cdist: seeded entries;
    long pair: the leading sub-problem of the pair)."""
    import oracle
    if cfg.kind == "batch":
        b, k = oracle_sample(cfg, target_cells)
        return (lambda: run_oracle_timed(b, cfg, cores)), b.cells(), \
            f"first {k} pairs of {cfg.name} ({b.cells():.3g} cells), plain C table DP, OpenMP over pairs"
    if cfg.kind == "cdist":
        cnt = max(1, int(target_cells // (cfg.length * cfg.length)))
        ia = workload.sample_indices(cfg, 0, cnt, cfg.nA)
        ib = workload.sample_indices(cfg, 1, cnt, cfg.nB)
        A = workload.gen_set(cfg, "A")
        B = workload.gen_set(cfg, "B")

        def run():
            t0 = time.perf_counter()
            oracle.cdist_entries(A, B, ia, ib, cfg.norm, threads=cores)
            return time.perf_counter() - t0
        cells = cnt * cfg.length * cfg.length
        return run, cells, f"{cnt} seeded (a, b) entries of {cfg.name} ({cells:.3g} cells), plain C table DP"
    # long pair: leading s×s sub-problem, one per norm, run concurrently (one core each)
    p, q = workload.gen_long_pair(cfg)
    s = int(min(p.shape[0], (target_cells / len(cfg.norms)) ** 0.5))
    from concurrent.futures import ThreadPoolExecutor

    def run():
        t0 = time.perf_counter()
        with ThreadPoolExecutor(len(cfg.norms)) as ex:
            list(ex.map(lambda nm: oracle.pair(p[:s], q[:s], nm, form="linear"), cfg.norms))
        return time.perf_counter() - t0
    cells = s * s * len(cfg.norms)
    return run, cells, (f"leading {s}x{s} sub-problem of {cfg.name} under {'/'.join(cfg.norms)} "
                        f"({cells:.3g} cells), fp64 Alg. 5 linear form, one core per norm")


def cpu_baseline_line(args, cfg, ws):
    """The oracle timed on the host cores on a bounded sample (rank 0, N = 1 only),
    with all host threads and with one (t1)."""
    if ws != 1 or args.no_cpu_baseline:
        return None
    cores = cpu_cores()
    run, ccells, sample = oracle_runner(cfg, args.cpu_cells, cores)
    t = run()
    if cfg.kind == "long":
        cores = len(cfg.norms)
    line = {"value": ccells / t / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{sample} (oracle/ffd_oracle.c), {t:.1f} s"}
    if cfg.kind != "long":  # the long-pair sample already runs one core per norm
        run1, c1, sample1 = oracle_runner(cfg, args.cpu_cells / 10, 1)
        t1 = run1()
        line["t1"] = {"value": c1 / t1 / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
                      "sample": f"{sample1} (one thread), {t1:.1f} s"}
    return line


def bench_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = workload.CONFIGS[args.config]
    cores = cpu_cores()
    run, cells, sample = oracle_runner(cfg, 3e8, cores)
    for _ in range(args.warmup):
        run()
    t = sum(run() for _ in range(args.steps))
    value = cells * args.steps / t / 1e9
    if cfg.kind == "long":
        cores = len(cfg.norms)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int64" if cfg.dtype == "i32" else "f64",
        "data": "synthetic", "config": {"workload": cfg.name, "sample_cells": cells},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample + " (per step)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


class Ctx:
    """Per-process GPU / process-group context shared by the measurements."""

    def __init__(self):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.ws, self.rank, local = dist_env()
        if self.ws > 1:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        self.dev = torch.device("cuda", local if self.ws > 1 else 0)
        torch.cuda.set_device(self.dev)
        import paper_2404_05708_b200 as ffd
        ffd.lib()
        self.ffd = ffd
        self.stream = torch.cuda.current_stream(self.dev)
        self.sms = torch.cuda.get_device_properties(self.dev).multi_processor_count

    def barrier(self):
        if self.ws > 1:
            self.dist.barrier()

    def reduce(self, vals, op="max"):
        if self.ws == 1:
            return list(vals)
        t = self.torch.tensor(list(vals), dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return [float(x) for x in t.tolist()]

    def close(self):
        if self.ws > 1:
            self.dist.destroy_process_group()


def measure_batch(args, cx, cfg):
    """A batch config (1-3): every rank its own shard of cfg.pairs pairs (weak
    scaling, no collective).  Returns the JSON line (rank 0) or None."""
    torch, ffd, dev, stream = cx.torch, cx.ffd, cx.dev, cx.stream
    first = cx.rank * cfg.pairs

    def pinned(shape, dtype):
        t = torch.empty(shape, dtype=torch.from_numpy(np.zeros(0, dtype)).dtype, pin_memory=True)
        return t.numpy()

    b = workload.gen_batch(cfg, alloc=pinned, first=first)
    cells = b.cells()
    B = b.num_pairs
    p = torch.from_numpy(b.p).to(dev)
    q = torch.from_numpy(b.q).to(dev)
    off = torch.from_numpy(b.offsets).to(dev)
    lens = torch.from_numpy(b.lengths).to(dev)
    out = torch.empty(B, dtype=torch.int64 if cfg.dtype == "i32" else torch.float32, device=dev)
    # the inputs are generated by workload/ and checked once by the library's own validator
    assert ffd.validate(p, q, off, lens) == 0
    # the caller knows its length bounds (ffd_batch_maxlen: no long-pair launch when none can be long)
    mlen = (int(b.lengths[:B].max()), int(b.lengths[B:].max()))

    # ---- device-resident timing ------------------------------------------------
    for _ in range(args.warmup):
        ffd.batch(p, q, off, lens, norm=cfg.norm, out=out, validate=False, max_len=mlen)
    torch.cuda.synchronize()
    ffd.launches_taken()
    ffd.profile_take()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cx.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev.index)
    ffd.profile_enable(True)
    in_bytes = b.p.nbytes + b.q.nbytes + b.offsets.nbytes + b.lengths.nbytes
    flush = in_bytes < L2_FLUSH_BELOW
    host_ms = None
    with sampler:
        if flush:
            ms = timed_steps_flushed(torch, stream, dev,
                                     lambda: ffd.batch(p, q, off, lens, norm=cfg.norm, out=out, validate=False, max_len=mlen),
                                     args.steps)
        else:
            e0.record(stream)
            h0 = time.perf_counter()
            for _ in range(args.steps):
                ffd.batch(p, q, off, lens, norm=cfg.norm, out=out, validate=False, max_len=mlen)
            host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
    ffd.profile_enable(False)
    cx.barrier()
    launches = ffd.launches_taken() // args.steps
    kern_ms_total, kern_n = ffd.profile_take()
    kern_ms = kern_ms_total / max(kern_n, 1)
    checksum = int(out.sum().item()) if cfg.dtype == "i32" else float(out.double().sum().item())
    ms_max, kern_max = cx.reduce([ms, kern_ms])
    total_cells = cx.reduce([float(cells)], "sum")[0]
    value = total_cells / (ms_max * 1e-3) / 1e9

    # ---- the same step replayed from a CUDA graph (small, launch-bound batches):
    # ffd_batch is stream-capturable, so a serving loop can replay its launch
    # chain as one graph launch
    graph = None
    if B <= 4096:
        try:
            side = torch.cuda.Stream(dev)
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                ffd.batch(p, q, off, lens, norm=cfg.norm, out=out, validate=False, max_len=mlen)
            stream.wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                ffd.batch(p, q, off, lens, norm=cfg.norm, out=out, validate=False, max_len=mlen)
            for _ in range(args.warmup):
                g.replay()
            torch.cuda.synchronize()
            if flush:
                g_ms = timed_steps_flushed(torch, stream, dev, g.replay, args.steps)
            else:
                g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                g0.record(stream)
                for _ in range(args.steps):
                    g.replay()
                g1.record(stream)
                torch.cuda.synchronize()
                g_ms = g0.elapsed_time(g1) / args.steps
            g_ms = cx.reduce([g_ms])[0]
            graph = {"ms_per_step": g_ms, "value": total_cells / (g_ms * 1e-3) / 1e9,
                     "unit": "Gcells/s", "api": "ffd_batch_maxlen captured once into a CUDA graph, replayed per step"}
        except Exception as e:  # reported, never silently replaced
            graph = {"error": f"{type(e).__name__}: {e}"[:200]}

    # ---- end to end through the C ABI with host buffers (ffd_batch_host) -------
    out_h = torch.empty(B, dtype=out.dtype, pin_memory=True).numpy()
    for _ in range(max(1, min(args.warmup, 2))):
        ffd.batch_host(b.p, b.q, b.offsets, b.lengths, norm=cfg.norm, out=out_h)
    cx.barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(args.steps):
        ffd.batch_host(b.p, b.q, b.offsets, b.lengths, norm=cfg.norm, out=out_h)
    e3.record(stream)
    torch.cuda.synchronize()
    cx.barrier()
    e2e_ms = cx.reduce([e2.elapsed_time(e3) / args.steps])[0]
    e2e_ok = bool(np.array_equal(out_h, out.cpu().numpy()))
    h2d = b.p.nbytes + b.q.nbytes + b.offsets.nbytes + b.lengths.nbytes
    d2h = out_h.nbytes
    if cx.rank != 0:
        return None

    clocks = sampler.summary()
    f_meas = (clocks["sm_mhz"] or SM_MAX_MHZ_NOMINAL) * 1e6
    f_max = (clocks["sm_max_mhz"] or SM_MAX_MHZ_NOMINAL) * 1e6
    cell = CELL_OF_CONFIG[cfg.cid]
    # 2-D batches above 4096 pairs: their single-band pairs (≤ 512 points) run on the
    # segmented two-column kernel (csrc/seg.cuh), the rest on the batch kernel; the
    # timed span covers both launches
    seg = B > 4096 and (cfg.dim == 2 or (cfg.dim == 3 and cfg.dtype == "f32" and cfg.norm in ("sql2", "l2")))
    kname = (f"seg_kernel + batch_kernel ({cell} cell)" if seg else f"batch_kernel ({cell} cell)")
    roofline = alu_roofline(cells, kern_max, cell, cx.sms, f_max, f_meas, kname, None)
    roofline["algorithmic_bytes"] = h2d + out.numel() * out.element_size()
    roofline["traffic_ncu"] = TRAFFIC_PROFILES.get(cfg.cid)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": cx.ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64" if cfg.dtype == "i32" else "f32",
        "data": "synthetic",
        "config": {"workload": cfg.name, "pairs_per_gpu": B, "cells_per_gpu_step": cells,
                   "arithmetic": ("int32 coordinates, exact int64 results: fp32 instructions on translated "
                                  "coordinates whose every partial is an integer < 2^24 (exact), int64 tier "
                                  "for pairs outside that window" if cfg.dtype == "i32" else "fp32"),
                   "dim": cfg.dim, "norm": cfg.norm, "lengths": list(cfg.len_p),
                   "l2": ("L2 flushed (256 MB write) before every timed step; steps timed one by one"
                          if flush else
                          "inputs larger than L2 (%.0f MB per GPU)" % ((b.p.nbytes + b.q.nbytes) / 1e6)),
                   "parallelism": f"pairs sharded over {cx.ws} GPU(s), no collective on the data path",
                   "api": f"batch() -> ffd_batch_maxlen with the batch's length bounds {list(mlen)}"},
        "clocks": clocks,
        "roofline": roofline,
        "cpu_baseline": cpu_baseline_line(args, cfg, cx.ws),
        "e2e": {"value": total_cells / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "matches_device_result": e2e_ok,
                "api": "ffd_batch_host (pinned host buffers, H2D + kernels + D2H per step)"},
        "gpu_launches": launches * args.steps,
        "gpu_launches_per_step": launches,
        "host_enqueue_ms_per_step": host_ms,
        "checksum": checksum,
    }
    if graph is not None:
        line["graph_replay"] = graph
    return line


def measure_cdist(args, cx, steps):
    """Config 4: all-pairs δ between two sets of 20k curves (L=128), rows of A sharded
    over the ranks, one NCCL all_gather_into_tensor assembles the matrix inside the
    timed region (SURVEY §8(a) a7 + a9; strong scaling).  Returns a dict (rank 0)."""
    torch, ffd, dev, stream = cx.torch, cx.ffd, cx.dev, cx.stream
    from paper_2404_05708_b200.dist import assemble, row_range
    cfg = workload.CONFIGS[4]
    if args.cdist_rows:
        cfg = cfg.scaled(nA=args.cdist_rows)
    A_h = workload.gen_set(cfg, "A")
    B_h = workload.gen_set(cfg, "B")
    A = torch.from_numpy(A_h).to(dev)
    B = torch.from_numpy(B_h).to(dev)
    r0, r1, blk = row_range(cfg.nA, cx.ws, cx.rank)
    block = torch.empty((blk, cfg.nB), dtype=torch.float32, device=dev)
    cells_rank = (r1 - r0) * cfg.nB * cfg.length * cfg.length
    total_cells = cfg.nA * cfg.nB * cfg.length * cfg.length

    def step():
        if r1 > r0:
            ffd.cdist(A, B, cfg.norm, rows=(r0, r1), out=block)
        if cx.ws > 1:
            return assemble(block, cfg.nA)
        return block

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ffd.launches_taken()
    ffd.profile_take()
    cx.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev.index)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ffd.profile_enable(True)
    with sampler:
        e0.record(stream)
        for _ in range(steps):
            full = step()
        e1.record(stream)
        torch.cuda.synchronize()
    ffd.profile_enable(False)
    cx.barrier()
    ms = e0.elapsed_time(e1) / steps
    kern_ms_total, kern_n = ffd.profile_take()
    kern_ms = kern_ms_total / max(kern_n, 1)
    launches = ffd.launches_taken() // steps
    ms_max, kern_max = cx.reduce([ms, kern_ms])
    checksum = float(full.double().sum().item())
    # the fused distribution (dist.cdist(distribution="p2p")): every rank's kernel
    # stores its results into all ranks' symmetric-memory matrices over NVLink,
    # one device barrier publishes them — no gather in the step
    p2p = None
    if cx.ws > 1:
        from paper_2404_05708_b200 import dist as fdist
        try:
            for _ in range(args.warmup):
                fdist.cdist(A, B, cfg.norm, distribution="p2p")
            torch.cuda.synchronize()
            cx.barrier()
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(stream)
            for _ in range(steps):
                fp = fdist.cdist(A, B, cfg.norm, distribution="p2p")
            p1.record(stream)
            torch.cuda.synchronize()
            p_ms = cx.reduce([p0.elapsed_time(p1) / steps])[0]
            same = bool(torch.equal(fp, full))
            p2p = {"value": total_cells / (p_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": p_ms,
                   "matches_allgather_matrix": same,
                   "api": "dist.cdist(distribution='p2p'): ffd_cdist_to into every rank's symmetric-memory "
                          "matrix + one device barrier"}
        except Exception as e:  # reported, never silently replaced
            p2p = {"error": f"{type(e).__name__}: {e}"[:300]}
    # the gather alone (max over ranks): what the collective adds to the step
    gather_ms = None
    if cx.ws > 1:
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cx.barrier()
        g0.record(stream)
        for _ in range(steps):
            assemble(block, cfg.nA)
        g1.record(stream)
        torch.cuda.synchronize()
        gather_ms = cx.reduce([g0.elapsed_time(g1) / steps])[0]
    # end to end: host A, B -> device, compute + gather, full matrix -> host
    out_h = torch.empty((cfg.nA, cfg.nB), dtype=torch.float32, pin_memory=True)
    A_p = torch.from_numpy(A_h).pin_memory()
    B_p = torch.from_numpy(B_h).pin_memory()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(1, steps // 4)
    cx.barrier()
    e2.record(stream)
    for _ in range(e2e_steps):
        A.copy_(A_p, non_blocking=True)
        B.copy_(B_p, non_blocking=True)
        f = step()
        out_h.copy_(f, non_blocking=True)
    e3.record(stream)
    torch.cuda.synchronize()
    e2e_ms = cx.reduce([e2.elapsed_time(e3) / e2e_steps])[0]
    if cx.rank != 0:
        return None
    clocks = sampler.summary()
    f_max = (clocks["sm_max_mhz"] or SM_MAX_MHZ_NOMINAL) * 1e6
    f_meas = (clocks["sm_mhz"] or SM_MAX_MHZ_NOMINAL) * 1e6
    roofline = alu_roofline(cells_rank, kern_max, CELL_OF_CONFIG[4], cx.sms, f_max, f_meas,
                            "cdist_kernel (fp32 L2, W=4 R=32)", None)
    roofline["algorithmic_bytes"] = A_h.nbytes + B_h.nbytes + (r1 - r0) * cfg.nB * 4
    roofline["traffic_ncu"] = TRAFFIC_PROFILES.get(4)
    return {
        "metric": METRIC, "value": total_cells / (ms_max * 1e-3) / 1e9, "unit": UNIT, "n_gpus": cx.ws,
        "steps": steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong", "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "nA": cfg.nA, "nB": cfg.nB, "length": cfg.length,
                   "cells_per_step": total_cells, "norm": cfg.norm,
                   "parallelism": f"rows of A over {cx.ws} GPU(s) + all_gather_into_tensor (NCCL) in the step",
                   "l2": "every step writes the 1.6 GB output, which evicts L2 between steps; "
                         "B (20 MB) is L2-resident within a step by design"},
        "clocks": clocks,
        "kernel_ms_per_rank": kern_max,
        "all_gather_ms": gather_ms,
        "p2p_distribution": p2p,
        "cpu_baseline": cpu_baseline_line(args, cfg, cx.ws),
        "roofline": roofline,
        "e2e": {"value": total_cells / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": A_h.nbytes + B_h.nbytes,
                "d2h_bytes_per_step": cfg.nA * cfg.nB * 4,
                "api": "dist.cdist path: H2D of A and B, ffd_cdist per rank, all-gather, D2H of the matrix"},
        "gpu_launches": launches * steps, "gpu_launches_per_step": launches,
        "checksum": checksum,
    }


def bench_ffd(args):
    """The default line: config 2 (headline value) with config 4 beside it."""
    cx = Ctx()
    cfg = workload.CONFIGS[args.config]
    line = measure_batch(args, cx, cfg)
    if args.config == 2 and not args.no_cdist:
        ap = measure_cdist(args, cx, args.steps)
        if line is not None:
            line["all_pairs"] = ap
            line["gpu_launches_all_pairs"] = ap["gpu_launches"]
    if line is not None:
        print(json.dumps(line), flush=True)
    cx.close()
    return 0


def bench_cdist(args):
    cx = Ctx()
    line = measure_cdist(args, cx, args.steps)
    if line is not None:
        line["vs_baseline"] = None
        print(json.dumps(line), flush=True)
    cx.close()
    return 0


def bench_long(args):
    """Config 5: one pair n = m = 262,144 (2-D fp32), the long-pair wavefront kernel
    (SURVEY §8(a) a8), under L1, L2 and L∞; one step = the three calls.  Replicas only
    (the pair does not shard): with N ranks every rank runs its own copy."""
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)
    import paper_2404_05708_b200 as ffd
    ffd.lib()
    cfg = workload.CONFIGS[5]
    p_h, q_h = workload.gen_long_pair(cfg)
    n, m = p_h.shape[0], q_h.shape[0]
    p = torch.from_numpy(p_h).to(dev)
    q = torch.from_numpy(q_h).to(dev)
    off = torch.tensor([0, 0], dtype=torch.int64, device=dev)
    lens = torch.tensor([n, m], dtype=torch.int32, device=dev)
    outs = {nm: torch.empty(1, dtype=torch.float32, device=dev) for nm in cfg.norms}
    assert ffd.validate(p, q, off, lens) == 0  # once; the timed calls skip the synchronous check
    stream = torch.cuda.current_stream(dev)
    cells = n * m

    def step():
        for nm in cfg.norms:
            ffd.batch(p, q, off, lens, norm=nm, out=outs[nm], validate=False)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ffd.launches_taken()
    ffd.profile_take()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev.index)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        ms = timed_steps_flushed(torch, stream, dev, step, args.steps)
    launches = ffd.launches_taken() // args.steps
    # per-norm duration of the dominant (long-pair) kernel: a second, instrumented pass
    per_norm = {nm: [] for nm in cfg.norms}
    for _ in range(args.steps):
        for nm in cfg.norms:
            ffd.profile_enable(True)
            ffd.batch(p, q, off, lens, norm=nm, out=outs[nm], validate=False)
            ffd.profile_enable(False)
            per_norm[nm].append(ffd.profile_take()[0])
    ffd.launches_taken()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t[0])
    vals = {nm: float(outs[nm].item()) for nm in cfg.norms}
    # end to end: host points in, three results out, per step
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p_pin = torch.from_numpy(p_h).pin_memory()
    q_pin = torch.from_numpy(q_h).pin_memory()
    res_h = torch.empty(len(cfg.norms), dtype=torch.float32, pin_memory=True)
    e2.record(stream)
    for _ in range(args.steps):
        p.copy_(p_pin, non_blocking=True)
        q.copy_(q_pin, non_blocking=True)
        step()
        res_h.copy_(torch.cat([outs[nm] for nm in cfg.norms]), non_blocking=True)
    e3.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e2.elapsed_time(e3) / args.steps
    # N > 1: the same pair with its rows split over the ranks (SURVEY §8(f) f4,
    # dist.long_pair: the band chain continues across GPUs through NVLink rings)
    sharded = None
    if ws > 1:
        from paper_2404_05708_b200 import dist as fdist
        try:
            for nm in cfg.norms:
                fdist.long_pair(p, q, nm)
            torch.cuda.synchronize()
            dist.barrier()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for _ in range(args.steps):
                res = {nm: fdist.long_pair(p, q, nm) for nm in cfg.norms}
            s1.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([s0.elapsed_time(s1) / args.steps], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sh_ms = float(t[0])
            sharded = {"value": 3 * cells / (sh_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": sh_ms,
                       "scaling": "strong", "matches_one_gpu": all(float(res[nm].item()) == float(outs[nm].item())
                                                                   for nm in cfg.norms),
                       "api": "dist.long_pair: rows split over the ranks, ffd_long_pair_shard, symmetric-memory rings"}
        except Exception as e:  # reported, never silently replaced
            sharded = {"error": f"{type(e).__name__}: {e}"[:300]}
    if rank == 0:
        clocks = sampler.summary()
        f_max = (clocks["sm_max_mhz"] or SM_MAX_MHZ_NOMINAL) * 1e6
        f_meas = (clocks["sm_mhz"] or SM_MAX_MHZ_NOMINAL) * 1e6
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        # median over the instrumented steps: one slow launch (a cooperative grid
        # waiting for SMs) must not stand for the kernel
        kern = {nm: float(np.median(per_norm[nm])) for nm in cfg.norms}
        per = {nm: alu_roofline(cells, kern[nm], CELL_OF_NORM[nm], sms, f_max, f_meas,
                                f"long_kernel (fp32 {nm})", None) for nm in cfg.norms}
        line = {
            "metric": METRIC, "value": ws * 3 * cells / (ms_max * 1e-3) / 1e9, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "n": n, "m": m, "norms": list(cfg.norms),
                       "cells_per_step": 3 * cells, "parallelism": "replicas only (one pair per GPU)",
                       "l2": "L2 flushed (256 MB write) before every timed step (inputs are 4.2 MB); steps timed one by one"},
            "clocks": clocks,
            "cpu_baseline": cpu_baseline_line(args, cfg, ws),
            "roofline": dict(per["l2"], per_norm={nm: {k: per[nm][k] for k in
                                                        ("kernel_ms", "achieved", "peak", "frac", "cell")}
                                                   for nm in cfg.norms}),
            "e2e": {"value": ws * 3 * cells / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": p_h.nbytes + q_h.nbytes, "d2h_bytes_per_step": 4 * len(cfg.norms)},
            "results": vals,
            "sharded_one_pair": sharded,
            "gpu_launches": launches * args.steps, "gpu_launches_per_step": launches,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def spawn_ranks(n: int):
    """Re-execute this command under torchrun with n ranks on this node (127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)]
    cmd += [a for a in sys.argv[1:] if a != "--spawn"]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ffd", choices=["ffd", "reference"])
    ap.add_argument("--cpu-cells", type=float, default=3e9, help="cells in the oracle cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cdist", action="store_true", help="default line: skip the config-4 all_pairs leg")
    ap.add_argument("--cdist-rows", type=int, default=0, help="config 4: use only this many A curves")
    ap.add_argument("--spawn", action="store_true",
                    help="run under torchrun even for --gpus 1 (the multi-rank launch path)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and (args.gpus > 1 or args.spawn):
        spawn_ranks(args.gpus)  # does not return
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; timing {ws} rank(s)", file=sys.stderr)
    if args.impl == "reference":
        return bench_reference(args)
    kind = workload.CONFIGS[args.config].kind
    if kind == "cdist":
        return bench_cdist(args)
    if kind == "long":
        return bench_long(args)
    return bench_ffd(args)


if __name__ == "__main__":
    sys.exit(main())
