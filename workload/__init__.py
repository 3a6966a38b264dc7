"""Seeded synthetic workloads for BASELINE.json configs 1–5 and the paper's sweeps.

Shared by the tests (oracle side) and bench.py / tests (CUDA side).  Holds no
part of the method's arithmetic: it only draws random-walk curves (C code in
ffd_gen.c, counter-based SplitMix64).

Batch layout (the ffd_batch ABI): p points [Σn, dim], q points [Σm, dim],
offsets int64[2B] (first B: p offsets, next B: q offsets, in points),
lengths int32[2B] (same order).  cdist layout: dense [n, L, dim].
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ffd_gen.c")
_LIB = os.path.join(_HERE, "libffd_gen.so")

SEED = 240405708  # arxiv id, fixed for every config


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fopenmp", "-shared", "-fPIC",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P, I64, I32, U64, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double
        L.ffdgen_lengths.argtypes = [U64, U64, I64, I64, I32, I32, P]
        L.ffdgen_walks_f32.argtypes = [U64, U64, I64, I64, P, P, I32, D, D, P]
        L.ffdgen_walks_i32.argtypes = [U64, U64, I64, I64, P, P, I32, I32, I32, P]
        L.ffdgen_walks_unit_f32.argtypes = [U64, U64, I64, I64, P, P, I32, P]
        L.ffdgen_indices.argtypes = [U64, U64, I64, I64, P]
        L.ffdgen_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config (or a scaled-down variant of it)."""
    cid: int
    name: str
    kind: str            # "batch" | "cdist" | "long"
    dim: int
    dtype: str           # "f32" | "i32"
    norm: str            # "l1" | "l2" | "linf" | "sql2"
    walk: str            # "gauss" | "int" | "unit"
    pairs: int = 0
    len_p: tuple = (1, 1)
    len_q: tuple = (1, 1)
    sigma: float = 1.0
    start_sigma: float = 0.0
    step: tuple = (-8, 8)
    nA: int = 0
    nB: int = 0
    length: int = 0
    norms: tuple = field(default_factory=tuple)

    def scaled(self, **kw) -> "Config":
        return replace(self, **kw)


CONFIGS = {
    1: Config(1, "c1_batch16_f32_2d_l2", "batch", 2, "f32", "l2", "gauss", pairs=16,
              len_p=(64, 64), len_q=(80, 80), sigma=1.0),
    2: Config(2, "c2_batch100k_i32_2d_sql2", "batch", 2, "i32", "sql2", "int", pairs=100_000,
              len_p=(128, 512), len_q=(128, 512), step=(-8, 8)),
    3: Config(3, "c3_batch1M_f32_3d_l2", "batch", 3, "f32", "l2", "gauss", pairs=1_000_000,
              len_p=(256, 1024), len_q=(256, 1024), sigma=1.0, start_sigma=10.0),
    4: Config(4, "c4_cdist20k_f32_2d_l2", "cdist", 2, "f32", "l2", "gauss", nA=20_000, nB=20_000,
              length=128, sigma=1.0),
    5: Config(5, "c5_longpair_262144_f32_2d", "long", 2, "f32", "l2", "gauss", pairs=1,
              len_p=(262_144, 262_144), len_q=(262_144, 262_144), sigma=1.0,
              norms=("l1", "l2", "linf")),
    # the paper's own sweep shape: unit steps, fp32, L2
    101: Config(101, "paper_E1_unit_walks", "batch", 2, "f32", "l2", "unit", pairs=1024,
                len_p=(1024, 1024), len_q=(1024, 1024)),
}


def _tag(cid: int, what: int) -> int:
    return cid * 16 + what


def gen_lengths(cfg: Config, which: str, count: int | None = None, first: int = 0) -> np.ndarray:
    count = cfg.pairs if count is None else count
    lo, hi = cfg.len_p if which == "p" else cfg.len_q
    out = np.empty(count, np.int32)
    lib().ffdgen_lengths(SEED, _tag(cfg.cid, 0 if which == "p" else 1), first, count, lo, hi, _ptr(out))
    return out


def _walks(cfg: Config, what: int, lengths: np.ndarray, offsets: np.ndarray, out: np.ndarray,
           first: int = 0):
    n = lengths.shape[0]
    lengths = np.ascontiguousarray(lengths, np.int32)
    offsets = np.ascontiguousarray(offsets, np.int64)
    tag = _tag(cfg.cid, what)
    if cfg.walk == "int":
        assert out.dtype == np.int32
        lib().ffdgen_walks_i32(SEED, tag, first, n, _ptr(lengths), _ptr(offsets), cfg.dim,
                               cfg.step[0], cfg.step[1], _ptr(out))
    elif cfg.walk == "unit":
        assert out.dtype == np.float32
        lib().ffdgen_walks_unit_f32(SEED, tag, first, n, _ptr(lengths), _ptr(offsets), cfg.dim, _ptr(out))
    else:
        assert out.dtype == np.float32
        lib().ffdgen_walks_f32(SEED, tag, first, n, _ptr(lengths), _ptr(offsets), cfg.dim,
                               cfg.sigma, cfg.start_sigma, _ptr(out))


def np_dtype(cfg: Config):
    return np.int32 if cfg.dtype == "i32" else np.float32


@dataclass
class Batch:
    p: np.ndarray          # [Σn, dim]
    q: np.ndarray          # [Σm, dim]
    offsets: np.ndarray    # int64[2B]
    lengths: np.ndarray    # int32[2B]
    dim: int
    norm: str

    @property
    def num_pairs(self) -> int:
        return self.offsets.shape[0] // 2

    def cells(self) -> int:
        B = self.num_pairs
        return int(np.dot(self.lengths[:B].astype(np.int64), self.lengths[B:].astype(np.int64)))


def gen_batch(cfg: Config, alloc=None, first: int = 0) -> Batch:
    """Generate pairs first..first+cfg.pairs-1 of a batch config (pair k depends
    only on k).  `alloc(shape, dtype)` may return writable numpy views (e.g. of
    pinned torch tensors); default np.empty."""
    alloc = alloc or (lambda shape, dtype: np.empty(shape, dtype))
    B = cfg.pairs
    lp = gen_lengths(cfg, "p", first=first)
    lq = gen_lengths(cfg, "q", first=first)
    op = np.zeros(B, np.int64)
    oq = np.zeros(B, np.int64)
    if B > 1:
        np.cumsum(lp[:-1], out=op[1:])
        np.cumsum(lq[:-1], out=oq[1:])
    dt = np_dtype(cfg)
    p = alloc((int(lp.sum()), cfg.dim), dt)
    q = alloc((int(lq.sum()), cfg.dim), dt)
    _walks(cfg, 2, lp, op, p, first=first)
    _walks(cfg, 3, lq, oq, q, first=first)
    return Batch(p, q, np.concatenate([op, oq]), np.concatenate([lp, lq]), cfg.dim, cfg.norm)


def gen_set(cfg: Config, which: str, alloc=None) -> np.ndarray:
    """Dense curve set [n, L, dim] for cdist configs (which: "A" | "B")."""
    alloc = alloc or (lambda shape, dtype: np.empty(shape, dtype))
    n = cfg.nA if which == "A" else cfg.nB
    L = cfg.length
    out = alloc((n, L, cfg.dim), np_dtype(cfg))
    lengths = np.full(n, L, np.int32)
    offsets = np.arange(n, dtype=np.int64) * L
    _walks(cfg, 4 if which == "A" else 5, lengths, offsets, out.reshape(-1, cfg.dim))
    return out


def gen_long_pair(cfg: Config):
    """The single long pair of config 5: (p [n, dim], q [m, dim])."""
    n, m = cfg.len_p[0], cfg.len_q[0]
    p = np.empty((n, cfg.dim), np_dtype(cfg))
    q = np.empty((m, cfg.dim), np_dtype(cfg))
    _walks(cfg, 6, np.array([n], np.int32), np.zeros(1, np.int64), p)
    _walks(cfg, 7, np.array([m], np.int32), np.zeros(1, np.int64), q)
    return p, q


def sample_indices(cfg: Config, what: int, count: int, n: int) -> np.ndarray:
    out = np.empty(count, np.int64)
    lib().ffdgen_indices(SEED, _tag(cfg.cid, 8 + what), count, n, _ptr(out))
    return out
