"""ctypes binding of the plain C oracle (oracle/ffd_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py.  The product package
(paper_2404_05708_b200) never imports this module.

Every function here is argument marshalling around the C oracle; the
arithmetic lives in ffd_oracle.c, which cites PAPER.md line by line.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ffd_oracle.c")
_LIB = os.path.join(_HERE, "libffd_oracle.so")

L1, L2, LINF, SQL2 = 1, 2, 3, 4
NORMS = {"l1": L1, "l2": L2, "linf": LINF, "sql2": SQL2}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C11, -ffp-contract=off, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "ffd_oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
             "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _declare(_lib)
    return _lib


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_INT = ctypes.c_int


def _declare(L):
    L.orc_point_dist_f32.restype = ctypes.c_double
    L.orc_point_dist_f32.argtypes = [_P, _P, _INT, _INT]
    L.orc_point_dist_i32.restype = _INT
    L.orc_point_dist_i32.argtypes = [_P, _P, _INT, _INT, _P]
    for n in ("orc_dist_matrix_f32", "orc_dist_matrix_i32"):
        getattr(L, n).restype = _INT
        getattr(L, n).argtypes = [_P, _I64, _P, _I64, _INT, _INT, _P]
    for n in ("orc_frechet_table_d", "orc_frechet_linear_d", "orc_frechet_alg2_d",
              "orc_frechet_inplace_d", "orc_frechet_brute_d", "orc_hausdorff_d",
              "orc_dtw_table_d", "orc_dtw_alg_d", "orc_dtw_brute_d"):
        getattr(L, n).restype = ctypes.c_double
        getattr(L, n).argtypes = [_P, _I64, _I64]
    for n in ("orc_frechet_table_i", "orc_frechet_linear_i", "orc_frechet_brute_i"):
        getattr(L, n).restype = _I64
        getattr(L, n).argtypes = [_P, _I64, _I64]
    L.orc_frechet_full_table_d.restype = None
    L.orc_frechet_full_table_d.argtypes = [_P, _I64, _I64, _P]
    for n in ("orc_pair_f32", "orc_pair_linear_f32", "orc_pair_i32", "orc_pair_linear_i32",
              "orc_pair_f32mirror", "orc_pair_dtw_f32", "orc_pair_dtw_f32mirror",
              "orc_pair_dist_sum_f32"):
        getattr(L, n).restype = _INT
        getattr(L, n).argtypes = [_P, _I64, _P, _I64, _INT, _INT, _P]
    for n in ("orc_batch_f32", "orc_batch_f32mirror", "orc_batch_i32", "orc_batch_dtw_f32",
              "orc_batch_dtw_f32mirror", "orc_batch_dist_sum_f32"):
        getattr(L, n).restype = _INT
        getattr(L, n).argtypes = [_P, _P, _P, _P, _I64, _INT, _INT, _P, _INT]
    for n in ("orc_cdist_entries_f32", "orc_cdist_entries_f32mirror"):
        getattr(L, n).restype = _INT
        getattr(L, n).argtypes = [_P, _I32, _P, _I32, _INT, _INT, _P, _P, _I64, _P, _INT]


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _norm(norm) -> int:
    return NORMS[norm] if isinstance(norm, str) else int(norm)


class OracleError(RuntimeError):
    def __init__(self, status):
        super().__init__(f"oracle status {status}")
        self.status = status


# ---- distance matrix -------------------------------------------------------

def dist_matrix(p, q, norm="l2"):
    """d_ij = f(p_i, q_j).  float32 input -> fp64 d; int32 -> int64 d."""
    p = np.asarray(p)
    q = np.asarray(q)
    dim = p.shape[1]
    if p.dtype.kind == "i":
        p, q = _c(p, np.int32), _c(q, np.int32)
        d = np.empty((p.shape[0], q.shape[0]), np.int64)
        st = lib().orc_dist_matrix_i32(_ptr(p), p.shape[0], _ptr(q), q.shape[0], dim, _norm(norm), _ptr(d))
    else:
        p, q = _c(p, np.float32), _c(q, np.float32)
        d = np.empty((p.shape[0], q.shape[0]), np.float64)
        st = lib().orc_dist_matrix_f32(_ptr(p), p.shape[0], _ptr(q), q.shape[0], dim, _norm(norm), _ptr(d))
    if st:
        raise OracleError(st)
    return d


# ---- δ from a given distance matrix ---------------------------------------

def _from_d(fn_d, fn_i, d):
    d = np.asarray(d)
    P, Q = d.shape
    if d.dtype.kind == "i":
        if fn_i is None:
            raise TypeError("integer form not provided")
        d = _c(d, np.int64)
        return int(fn_i(_ptr(d), P, Q))
    d = _c(d, np.float64)
    return float(fn_d(_ptr(d), P, Q))


def frechet_table_d(d):
    return _from_d(lib().orc_frechet_table_d, lib().orc_frechet_table_i, d)


def frechet_linear_d(d):
    return _from_d(lib().orc_frechet_linear_d, lib().orc_frechet_linear_i, d)


def frechet_alg2_d(d):
    return _from_d(lib().orc_frechet_alg2_d, None, d)


def frechet_inplace_d(d):
    return _from_d(lib().orc_frechet_inplace_d, None, d)


def frechet_brute_d(d):
    return _from_d(lib().orc_frechet_brute_d, lib().orc_frechet_brute_i, d)


def hausdorff_d(d):
    return _from_d(lib().orc_hausdorff_d, None, d)


def full_table_d(d):
    d = _c(d, np.float64)
    P, Q = d.shape
    C = np.empty((P + 1, Q + 1), np.float64)
    lib().orc_frechet_full_table_d(_ptr(d), P, Q, _ptr(C))
    return C


def dtw_table_d(d):
    return _from_d(lib().orc_dtw_table_d, None, d)


def dtw_alg_d(d):
    return _from_d(lib().orc_dtw_alg_d, None, d)


def dtw_brute_d(d):
    return _from_d(lib().orc_dtw_brute_d, None, d)


def dtw_pair(p, q, norm="l2", mirror=False):
    """DTW(p, q) of float32 curves with lazily evaluated d: fp64 table, or the
    fp32 mirror of the kernels' operation order (mirror=True)."""
    p, q = _c(p, np.float32), _c(q, np.float32)
    out = np.zeros(1, np.float32 if mirror else np.float64)
    fn = lib().orc_pair_dtw_f32mirror if mirror else lib().orc_pair_dtw_f32
    st = fn(_ptr(p), p.shape[0], _ptr(q), q.shape[0], p.shape[1], _norm(norm), _ptr(out))
    if st:
        raise OracleError(st)
    return out[0].item()


def dtw_batch(p, q, offsets, lengths, dim, norm="l2", threads=0, mirror=False, check=True):
    """DTW of every pair of a batch (float32 curves), layout as batch()."""
    offsets = _c(offsets, np.int64)
    lengths = _c(lengths, np.int32)
    B = offsets.shape[0] // 2
    p, q = _c(p, np.float32), _c(q, np.float32)
    out = np.empty(B, np.float32 if mirror else np.float64)
    fn = lib().orc_batch_dtw_f32mirror if mirror else lib().orc_batch_dtw_f32
    st = fn(_ptr(p), _ptr(q), _ptr(offsets), _ptr(lengths), B, dim, _norm(norm), _ptr(out), threads)
    if st and check:
        raise OracleError(st)
    return out


def dist_sum_pair(p, q, norm="l2"):
    """Σ_ij d(p_i, q_j) of float32 curves in fp64."""
    p, q = _c(p, np.float32), _c(q, np.float32)
    out = np.zeros(1, np.float64)
    st = lib().orc_pair_dist_sum_f32(_ptr(p), p.shape[0], _ptr(q), q.shape[0], p.shape[1],
                                     _norm(norm), _ptr(out))
    if st:
        raise OracleError(st)
    return out[0].item()


def dist_sum_batch(p, q, offsets, lengths, dim, norm="l2", threads=0, check=True):
    """Σ_ij d_ij of every pair of a batch (float32 curves), layout as batch()."""
    offsets = _c(offsets, np.int64)
    lengths = _c(lengths, np.int32)
    B = offsets.shape[0] // 2
    p, q = _c(p, np.float32), _c(q, np.float32)
    out = np.empty(B, np.float64)
    st = lib().orc_batch_dist_sum_f32(_ptr(p), _ptr(q), _ptr(offsets), _ptr(lengths), B, dim,
                                      _norm(norm), _ptr(out), threads)
    if st and check:
        raise OracleError(st)
    return out


# ---- pairs -----------------------------------------------------------------

def pair(p, q, norm="l2", form="table"):
    """δ_dF(p, q) with lazily evaluated d.  form: table | linear | mirror."""
    p = np.asarray(p)
    q = np.asarray(q)
    dim = p.shape[1]
    L = lib()
    if p.dtype.kind == "i":
        p, q = _c(p, np.int32), _c(q, np.int32)
        out = np.zeros(1, np.int64)
        fn = {"table": L.orc_pair_i32, "linear": L.orc_pair_linear_i32}[form]
    else:
        p, q = _c(p, np.float32), _c(q, np.float32)
        if form == "mirror":
            out = np.zeros(1, np.float32)
            fn = L.orc_pair_f32mirror
        else:
            out = np.zeros(1, np.float64)
            fn = {"table": L.orc_pair_f32, "linear": L.orc_pair_linear_f32}[form]
    st = fn(_ptr(p), p.shape[0], _ptr(q), q.shape[0], dim, _norm(norm), _ptr(out))
    if st:
        raise OracleError(st)
    return out[0].item()


def batch(p, q, offsets, lengths, dim, norm="l2", threads=0, mirror=False, check=True):
    """out[k] = δ(p[offsets[k]:+lengths[k]], q[offsets[B+k]:+lengths[B+k]]).

    p, q: flat point arrays [Σ, dim] (float32 or int32).  Returns float64 (or
    float32 for mirror=True) / int64 array of length B."""
    offsets = _c(offsets, np.int64)
    lengths = _c(lengths, np.int32)
    B = offsets.shape[0] // 2
    L = lib()
    if np.asarray(p).dtype.kind == "i":
        p, q = _c(p, np.int32), _c(q, np.int32)
        out = np.empty(B, np.int64)
        st = L.orc_batch_i32(_ptr(p), _ptr(q), _ptr(offsets), _ptr(lengths), B, dim, _norm(norm), _ptr(out), threads)
    else:
        p, q = _c(p, np.float32), _c(q, np.float32)
        if mirror:
            out = np.empty(B, np.float32)
            st = L.orc_batch_f32mirror(_ptr(p), _ptr(q), _ptr(offsets), _ptr(lengths), B, dim, _norm(norm), _ptr(out), threads)
        else:
            out = np.empty(B, np.float64)
            st = L.orc_batch_f32(_ptr(p), _ptr(q), _ptr(offsets), _ptr(lengths), B, dim, _norm(norm), _ptr(out), threads)
    if st and check:
        raise OracleError(st)
    return out


def cdist_entries(A, B, ia, ib, norm="l2", threads=0, mirror=False):
    """out[k] = δ(A[ia[k]], B[ib[k]]) for dense sets A [nA, lenA, dim], B [nB, lenB, dim]."""
    A = _c(A, np.float32)
    Bs = _c(B, np.float32)
    ia = _c(ia, np.int64)
    ib = _c(ib, np.int64)
    n = ia.shape[0]
    L = lib()
    if mirror:
        out = np.empty(n, np.float32)
        st = L.orc_cdist_entries_f32mirror(_ptr(A), A.shape[1], _ptr(Bs), Bs.shape[1], A.shape[2], _norm(norm),
                                           _ptr(ia), _ptr(ib), n, _ptr(out), threads)
    else:
        out = np.empty(n, np.float64)
        st = L.orc_cdist_entries_f32(_ptr(A), A.shape[1], _ptr(Bs), Bs.shape[1], A.shape[2], _norm(norm),
                                     _ptr(ia), _ptr(ib), n, _ptr(out), threads)
    if st:
        raise OracleError(st)
    return out
