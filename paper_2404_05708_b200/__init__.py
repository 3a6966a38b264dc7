"""B200-native discrete Fréchet distance (arxiv 2404.05708) — Python binding.

Thin ctypes marshalling over the C ABI of include/ffd.h (libffd.so, built
in-tree by ``python -m paper_2404_05708_b200.build``).  Every step of the
computation runs in the library's CUDA kernels; PyTorch only provides device
memory and streams.  There is no CPU fallback: if the library or a GPU is
missing, calls raise.

    batch(p, q, offsets, lengths, norm)        -> Tensor[B]   (ffd_batch_maxlen)
    dtw_batch(p, q, offsets, lengths, norm)    -> Tensor[B]   (ffd_batch_dtw)
    dist_sum(p, q, offsets, lengths, norm)     -> Tensor[B] f64 (ffd_dist_sum)
    batch_host(p, q, offsets, lengths, norm)   -> ndarray[B]  (ffd_batch_host)
    cdist(A, B, norm, rows=None)               -> Tensor      (ffd_cdist)
    cdist_self(A, norm, rows=None)             -> Tensor      (ffd_cdist_self)
    cdist_to(A, B, outs, ...)                  -> None        (ffd_cdist_to: results into
                                                   full matrices on this GPU and NVLink peers)
    validate(p, q, offsets, lengths)           -> status      (ffd_validate_batch)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FFD_LIB", os.path.join(_HERE, "libffd.so"))

L1, L2, LINF, SQL2 = 1, 2, 3, 4
NORMS = {"l1": L1, "l2": L2, "linf": LINF, "sql2": SQL2}
F32, I32 = 0, 1

STATUS = {0: "ok", -1: "invalid argument", -2: "unsupported", -3: "CUDA error", -4: "empty curve",
          -5: "non-finite coordinate", -6: "integer overflow", -7: "out of range",
          -8: "workspace too small"}


class FFDError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        super().__init__(f"{what}: ffd status {status} ({STATUS.get(status, '?')})")
        self.status = status


_lib = None


def lib():
    """Load libffd.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2404_05708_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        P, I64, I32_, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
        L.ffd_batch.argtypes = [P, P, P, P, I64, I32_, I32_, I32_, P, P, SZ, P]
        L.ffd_batch.restype = ctypes.c_int
        L.ffd_batch_maxlen.argtypes = [P, P, P, P, I64, I64, I64, I32_, I32_, I32_, P, P, SZ, P]
        L.ffd_batch_maxlen.restype = ctypes.c_int
        L.ffd_batch_dtw.argtypes = [P, P, P, P, I64, I32_, I32_, I32_, P, P, SZ, P]
        L.ffd_batch_dtw.restype = ctypes.c_int
        L.ffd_batch_dtw_f64.argtypes = [P, P, P, P, I64, I32_, I32_, I32_, P, P, SZ, P]
        L.ffd_batch_dtw_f64.restype = ctypes.c_int
        L.ffd_dist_sum.argtypes = [P, P, P, P, I64, I32_, I32_, I32_, P, P]
        L.ffd_dist_sum.restype = ctypes.c_int
        L.ffd_batch_workspace_bytes.argtypes = [I64]
        L.ffd_batch_workspace_bytes.restype = SZ
        L.ffd_batch_host.argtypes = [P, I64, P, I64, P, P, I64, I32_, I32_, I32_, P, P]
        L.ffd_batch_host.restype = ctypes.c_int
        L.ffd_cdist.argtypes = [P, I64, I32_, P, I64, I32_, I32_, I32_, I32_, I64, I64, P, I64, P, SZ, P]
        L.ffd_cdist.restype = ctypes.c_int
        L.ffd_cdist_self.argtypes = [P, I64, I32_, I32_, I32_, I32_, I64, I64, P, I64, P, SZ, P]
        L.ffd_cdist_self.restype = ctypes.c_int
        L.ffd_cdist_to.argtypes = [P, I64, I32_, P, I64, I32_, I32_, I32_, I32_, I64, I64, I32_, I64, I32_,
                                   ctypes.POINTER(ctypes.c_void_p), I32_, I64, P, SZ, P]
        L.ffd_cdist_to.restype = ctypes.c_int
        L.ffd_cdist_workspace_bytes.argtypes = []
        L.ffd_cdist_workspace_bytes.restype = SZ
        L.ffd_long_pair_ring_bytes.argtypes = [I32_, I32_]
        L.ffd_long_pair_ring_bytes.restype = SZ
        L.ffd_long_pair_row_align.argtypes = []
        L.ffd_long_pair_row_align.restype = I32_
        L.ffd_long_pair_shard.argtypes = [P, I32_, P, I32_, I32_, I32_, I32_, I32_, I32_, P, SZ, ctypes.c_uint32,
                                          P, SZ, ctypes.c_uint32, P, P]
        L.ffd_long_pair_shard.restype = ctypes.c_int
        L.ffd_validate_batch.argtypes = [P, I64, P, I64, P, P, I64, I32_, I32_, P]
        L.ffd_validate_batch.restype = ctypes.c_int
        L.ffd_status_string.argtypes = [ctypes.c_int]
        L.ffd_status_string.restype = ctypes.c_char_p
        L.ffd_take_launch_count.argtypes = []
        L.ffd_take_launch_count.restype = I64
        L.ffd_version.restype = ctypes.c_int
        L.ffd_profile_enable.argtypes = [ctypes.c_int]
        L.ffd_profile_enable.restype = ctypes.c_int
        L.ffd_profile_take.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64)]
        L.ffd_profile_take.restype = ctypes.c_int
        _lib = L
    return _lib


EXPORTED = ["ffd_batch", "ffd_batch_maxlen", "ffd_batch_dtw", "ffd_batch_dtw_f64", "ffd_dist_sum", "ffd_batch_workspace_bytes", "ffd_batch_host", "ffd_cdist",
            "ffd_cdist_workspace_bytes", "ffd_cdist_self", "ffd_cdist_to", "ffd_long_pair_ring_bytes",
            "ffd_long_pair_row_align", "ffd_long_pair_shard", "ffd_validate_batch", "ffd_status_string",
            "ffd_take_launch_count", "ffd_version", "ffd_profile_enable", "ffd_profile_take"]


def _norm(norm) -> int:
    return NORMS[norm] if isinstance(norm, str) else int(norm)


def _torch():
    import torch
    return torch


def _stream_ptr(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.int32:
        return I32
    raise TypeError(f"coordinates must be float32 or int32, got {t.dtype}")


def _check(status: int, what: str):
    if status != 0:
        raise FFDError(status, what)


_ws_cache: dict = {}


def workspace(nbytes: int, device, stream=None):
    """Cached device workspace (grows on demand), one per (device, stream): calls
    on different streams run concurrently and must not share scratch.  The
    buffer is allocated on its stream, so the caching allocator only reuses a
    replaced buffer in that stream's order."""
    torch = _torch()
    dev = torch.device(device)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    key = (dev.index, s.cuda_stream)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        with torch.cuda.stream(s):
            buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
        _ws_cache[key] = buf
    return buf


def profile_enable(on: bool = True):
    lib().ffd_profile_enable(1 if on else 0)


def profile_take():
    """(summed dominant-kernel ms, number of timed launches) since the last take."""
    ms = ctypes.c_double(0.0)
    n = ctypes.c_int64(0)
    _check(lib().ffd_profile_take(ctypes.byref(ms), ctypes.byref(n)), "ffd_profile_take")
    return ms.value, n.value


def launches_taken() -> int:
    """Kernels the library launched on this thread since the previous call."""
    return int(lib().ffd_take_launch_count())


def _batch_args(p, q, offsets, lengths):
    """Common marshalling of the batch layout: dtypes, devices, shapes, contiguity."""
    torch = _torch()
    if not (p.is_cuda and q.is_cuda and offsets.is_cuda and lengths.is_cuda):
        raise ValueError("batch() takes CUDA tensors; use batch_host() for host arrays")
    dt = _dtype_code(p)
    if q.dtype != p.dtype or offsets.dtype != torch.int64 or lengths.dtype != torch.int32:
        raise TypeError("dtype mismatch (p/q same dtype, offsets int64, lengths int32)")
    if p.dim() != 2 or q.dim() != 2 or p.shape[1] != q.shape[1]:
        raise ValueError(f"p and q must be [points, dim] with the same dim, got {tuple(p.shape)}, {tuple(q.shape)}")
    if offsets.numel() % 2 or offsets.numel() != lengths.numel():
        raise ValueError("offsets and lengths must both hold 2*B entries")
    return dt, p.contiguous(), q.contiguous(), offsets.contiguous(), lengths.contiguous()


def batch(p, q, offsets, lengths, norm="l2", out=None, stream=None, measure="frechet", validate=True,
          max_len=None):
    """δ_dF for B pairs (ffd_batch).  p [Σn, dim], q [Σm, dim] float32/int32 CUDA
    tensors; offsets int64[2B]; lengths int32[2B].  Returns float32[B] (fp32
    input) or int64[B] (int32 input).  measure="dtw": dynamic time warping
    (ffd_batch_dtw, PAPER Appendix B; float32 input only); measure="dtw_f64": the
    same with fp64 sums (ffd_batch_dtw_f64, float64[B]).  validate=True first
    runs ffd_validate_batch (synchronous) and raises FFDError on empty curves,
    offsets out of range, non-finite coordinates or int64 overflow; with
    validate=False such pairs give NaN / INT64_MIN (or are undefined).  Inside a
    CUDA-graph capture the (synchronous) validation is skipped.  max_len: a bound
    on every curve length (int, or (max p-length, max q-length)); Fréchet calls
    ffd_batch_maxlen with it (default: the point counts of p and q), which skips
    the long-pair launch when no pair within it can be long — a pair longer
    than a bound it breaks gets NaN / INT64_MIN."""
    torch = _torch()
    dt, p, q, offsets, lengths = _batch_args(p, q, offsets, lengths)
    B = offsets.numel() // 2
    dim = p.shape[1]
    fns = {"frechet": "ffd_batch", "dtw": "ffd_batch_dtw", "dtw_f64": "ffd_batch_dtw_f64"}
    if measure not in fns:
        raise ValueError(f"unknown measure {measure!r}")
    if validate and not torch.cuda.is_current_stream_capturing():  # (a synchronous check cannot be captured)
        _check(int(lib().ffd_validate_batch(p.data_ptr(), p.shape[0], q.data_ptr(), q.shape[0],
                                            offsets.data_ptr(), lengths.data_ptr(), B, dim, dt,
                                            _stream_ptr(stream))), "ffd_validate_batch")
    if out is None:
        odt = torch.float64 if measure == "dtw_f64" else (torch.int64 if dt == I32 else torch.float32)
        out = torch.empty(B, dtype=odt, device=p.device)
    ws_bytes = lib().ffd_batch_workspace_bytes(B)
    ws = workspace(ws_bytes, p.device, stream)
    if measure == "frechet":  # length bounds let the library skip the long-pair launch of small batches
        mn, mm = (p.shape[0], q.shape[0]) if max_len is None else (max_len if isinstance(max_len, tuple)
                                                                   else (max_len, max_len))
        _check(lib().ffd_batch_maxlen(p.data_ptr(), q.data_ptr(), offsets.data_ptr(), lengths.data_ptr(), B,
                                      int(mn), int(mm), dim, _norm(norm), dt, out.data_ptr(), ws.data_ptr(),
                                      ws.numel(), _stream_ptr(stream)), "ffd_batch_maxlen")
        return out
    fn = getattr(lib(), fns[measure])
    _check(fn(p.data_ptr(), q.data_ptr(), offsets.data_ptr(), lengths.data_ptr(), B, dim,
              _norm(norm), dt, out.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(stream)), fns[measure])
    return out


def dtw_batch(p, q, offsets, lengths, norm="l2", out=None, stream=None, validate=True, precision="f32"):
    """Dynamic time warping of B pairs (ffd_batch_dtw, or ffd_batch_dtw_f64 with
    precision="f64": fp64 sums, bit-exact against the fp64 oracle): same layout as batch()."""
    if precision not in ("f32", "f64"):
        raise ValueError("precision must be 'f32' or 'f64'")
    return batch(p, q, offsets, lengths, norm=norm, out=out, stream=stream,
                 measure="dtw" if precision == "f32" else "dtw_f64", validate=validate)


def dist_sum(p, q, offsets, lengths, norm="l2", out=None, stream=None):
    """Σ_ij d(p_i, q_j) of B pairs (ffd_dist_sum, the paper's "upper limit"
    baseline): same layout as batch(), float32 curves, float64 result."""
    torch = _torch()
    if _dtype_code(p) != F32:
        raise FFDError(-2, "ffd_dist_sum")
    _, p, q, offsets, lengths = _batch_args(p, q, offsets, lengths)
    B = offsets.shape[0] // 2
    if out is None:
        out = torch.empty(B, dtype=torch.float64, device=p.device)
    _check(lib().ffd_dist_sum(p.data_ptr(), q.data_ptr(), offsets.data_ptr(), lengths.data_ptr(), B,
                              p.shape[1], _norm(norm), F32, out.data_ptr(), _stream_ptr(stream)),
           "ffd_dist_sum")
    return out


def batch_host(p: np.ndarray, q: np.ndarray, offsets: np.ndarray, lengths: np.ndarray, norm="l2",
               out: np.ndarray | None = None, stream=None) -> np.ndarray:
    """ffd_batch_host: host buffers in and out (copies inside the call)."""
    p = np.ascontiguousarray(p)
    q = np.ascontiguousarray(q)
    offsets = np.ascontiguousarray(offsets, np.int64)
    lengths = np.ascontiguousarray(lengths, np.int32)
    dt = I32 if p.dtype == np.int32 else F32
    B = offsets.shape[0] // 2
    if out is None:
        out = np.empty(B, np.int64 if dt == I32 else np.float32)
    _check(lib().ffd_batch_host(p.ctypes.data, p.shape[0], q.ctypes.data, q.shape[0], offsets.ctypes.data,
                                lengths.ctypes.data, B, p.shape[1], _norm(norm), dt, out.ctypes.data,
                                _stream_ptr(stream)), "ffd_batch_host")
    return out


def cdist(A, B, norm="l2", rows=None, out=None, ld_out=None, stream=None):
    """ffd_cdist on one shard: rows = (row_begin, row_end) of A (default all).
    A [nA, lenA, dim], B [nB, lenB, dim] CUDA tensors.  Returns the block
    [row_end-row_begin, nB] (float32, or int64 for int32 input)."""
    torch = _torch()
    dt = _dtype_code(A)
    A, B = A.contiguous(), B.contiguous()
    nA, lenA, dim = A.shape
    nB, lenB, _ = B.shape
    r0, r1 = (0, nA) if rows is None else rows
    ld = nB if ld_out is None else ld_out
    if out is None:
        out = torch.empty((r1 - r0, ld), dtype=torch.int64 if dt == I32 else torch.float32, device=A.device)
    wsb = lib().ffd_cdist_workspace_bytes()
    ws = workspace(wsb, A.device, stream) if wsb else None
    _check(lib().ffd_cdist(A.data_ptr(), nA, lenA, B.data_ptr(), nB, lenB, dim, _norm(norm), dt, r0, r1,
                           out.data_ptr(), ld, ws.data_ptr() if ws is not None else None, wsb,
                           _stream_ptr(stream)), "ffd_cdist")
    return out


def cdist_self(A, norm="l2", rows=None, out=None, ld_out=None, stream=None):
    """ffd_cdist_self: all-pairs δ of a set against itself (each unordered pair in
    the shard evaluated once).  Returns the block [row_end-row_begin, nA]."""
    torch = _torch()
    dt = _dtype_code(A)
    A = A.contiguous()
    nA, lenA, dim = A.shape
    r0, r1 = (0, nA) if rows is None else rows
    ld = nA if ld_out is None else ld_out
    if out is None:
        out = torch.empty((r1 - r0, ld), dtype=torch.int64 if dt == I32 else torch.float32, device=A.device)
    wsb = lib().ffd_cdist_workspace_bytes()
    ws = workspace(wsb, A.device, stream) if wsb else None
    _check(lib().ffd_cdist_self(A.data_ptr(), nA, lenA, dim, _norm(norm), dt, r0, r1, out.data_ptr(), ld,
                                ws.data_ptr() if ws is not None else None, wsb, _stream_ptr(stream)),
           "ffd_cdist_self")
    return out


def cdist_to(A, B, outs, ld_out, norm="l2", rows=None, self_mode=False, col_offset=0, mirror=False,
             stream=None):
    """ffd_cdist_to: rows [r0, r1) of A against the curves of B (column col_offset + b)
    written straight into every matrix of `outs` — device pointers (ints) of full
    row-major matrices with ld_out elements per row: this GPU's and NVLink peers'
    (symmetric memory / CUDA IPC).  mirror=True also writes the transposed place;
    self_mode=True: B is A's rows [col_offset, col_offset + nB), each unordered pair
    inside the shard evaluated once."""
    dt = _dtype_code(A)
    if B.dtype != A.dtype:
        raise TypeError("A and B must have the same dtype")
    A, B = A.contiguous(), B.contiguous()
    nA, lenA, dim = A.shape
    nB, lenB, dimB = B.shape
    if dimB != dim:
        raise ValueError("A and B must have the same dim")
    r0, r1 = (0, nA) if rows is None else rows
    ptrs = (ctypes.c_void_p * len(outs))(*[int(x) for x in outs])
    wsb = lib().ffd_cdist_workspace_bytes()
    ws = workspace(wsb, A.device, stream) if wsb else None
    _check(lib().ffd_cdist_to(A.data_ptr(), nA, lenA, B.data_ptr(), nB, lenB, dim, _norm(norm), dt, r0, r1,
                              1 if self_mode else 0, col_offset, 1 if mirror else 0, ptrs, len(outs), ld_out,
                              ws.data_ptr() if ws is not None else None, wsb, _stream_ptr(stream)),
           "ffd_cdist_to")


def long_pair_ring_bytes(n: int, m: int) -> int:
    """Bytes of one cross-GPU ring of ffd_long_pair_shard for an n×m pair."""
    return int(lib().ffd_long_pair_ring_bytes(n, m))


def long_pair_row_align() -> int:
    return int(lib().ffd_long_pair_row_align())


def long_pair_shard(p, q, rows, norm="l2", in_ring=None, in_tag=0, out_ring=None, out_tag=0, out=None,
                    stream=None):
    """ffd_long_pair_shard: rows = (row_begin, row_end) of the rows curve (the shorter
    of p, q) on this GPU; in_ring: a local uint8 CUDA tensor (or None for the first
    range); out_ring: (pointer, bytes) of the next GPU's ring (or None for the last
    range).  Returns `out` (float32[1]); only the range ending at the last row
    writes δ into it."""
    torch = _torch()
    if _dtype_code(p) != F32 or q.dtype != p.dtype:
        raise FFDError(-2, "ffd_long_pair_shard")
    p, q = p.contiguous(), q.contiguous()
    if out is None:
        out = torch.full((1,), float("nan"), dtype=torch.float32, device=p.device)
    in_ptr, in_b = (in_ring.data_ptr(), in_ring.numel()) if in_ring is not None else (None, 0)
    out_ptr, out_b = (int(out_ring[0]), int(out_ring[1])) if out_ring is not None else (None, 0)
    _check(lib().ffd_long_pair_shard(p.data_ptr(), p.shape[0], q.data_ptr(), q.shape[0], p.shape[1], _norm(norm),
                                     F32, rows[0], rows[1], in_ptr, in_b, in_tag & 0xffffffff, out_ptr, out_b,
                                     out_tag & 0xffffffff, out.data_ptr(), _stream_ptr(stream)),
           "ffd_long_pair_shard")
    return out


def validate(p, q, offsets, lengths, stream=None) -> int:
    """ffd_validate_batch (synchronous); returns the status code."""
    dt, p, q, offsets, lengths = _batch_args(p, q, offsets, lengths)
    B = offsets.numel() // 2
    return int(lib().ffd_validate_batch(p.data_ptr(), p.shape[0], q.data_ptr(), q.shape[0], offsets.data_ptr(),
                                        lengths.data_ptr(), B, p.shape[1], dt, _stream_ptr(stream)))
