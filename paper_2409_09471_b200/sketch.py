"""Khatri-Rao structured sketch of TT vectors on the B200 (mirrors ttkrylov/sketch.py)."""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _lib
from .errors import ShapeMismatch
from .tt import TTOperator, TTVector, default_device


class KhatriRaoSketch:
    """Row-wise Khatri-Rao product of Gaussian factor matrices (sketch.py:18-35).

    Factors are held on the device as (rows, n_k) fp64 tensors."""

    def __init__(self, factors, seed=None, device=None):
        if device is None:
            device = factors[0].device if isinstance(factors[0], torch.Tensor) else default_device()
        fs = []
        for f in factors:
            t = f.to(dtype=torch.float64, device=device) if isinstance(f, torch.Tensor) else \
                torch.as_tensor(np.asarray(f, dtype=np.float64), device=device)
            fs.append(t.contiguous())
        rows = {int(f.shape[0]) for f in fs}
        if len(rows) != 1:
            raise ShapeMismatch("all factors must have the same row count")
        self.factors = fs
        self.rows = rows.pop()
        self.seed = seed

    @property
    def dims(self) -> tuple[int, ...]:
        return tuple(int(f.shape[1]) for f in self.factors)


def kr_sketch_new(dims, rows: int, seed=0, device=None) -> KhatriRaoSketch:
    """Factor entries N(0, rows^(-1/d)) drawn on the host from default_rng(seed) (sketch.py:38-47)."""
    if rows < 1:
        raise ValueError("rows must be >= 1")
    dims = list(dims)
    std = float(rows) ** (-0.5 / len(dims))
    rng = np.random.default_rng(seed)
    factors = [rng.normal(0.0, std, size=(rows, n)) for n in dims]
    return KhatriRaoSketch(factors, seed=seed, device=device)


def kr_apply_rows(s: KhatriRaoSketch, vs, row_lo: int, row_hi: int, out=None) -> torch.Tensor:
    """Sketch rows [row_lo, row_hi) of a batch of TT vectors -> (len(vs), row_hi-row_lo) device tensor."""
    vs = list(vs)
    for v in vs:
        if s.dims != v.dims:
            raise ShapeMismatch(f"sketch dims {s.dims} do not match vector {v.dims}")
    if not (0 <= row_lo <= row_hi <= s.rows):
        raise ValueError("bad row range")
    dev = s.factors[0].device
    if out is None:
        out = torch.empty((len(vs), row_hi - row_lo), dtype=torch.float64, device=dev)
    if not vs or row_hi == row_lo:
        return out
    _lib.require_cuda(s.factors[0], "sketch factors")
    lib = _lib.load()
    d = len(s.dims)
    n = _lib.int_array(s.dims)
    ranks = _lib.int_array([r for v in vs for r in v.ranks])
    nbytes = lib.ttk_kr_sketch_ws_bytes(d, n, row_lo, row_hi, len(vs), ranks)
    ws = _lib.workspace(nbytes, dev)
    _lib.check(lib.ttk_kr_sketch(d, n, row_lo, row_hi, _lib.ptr_array(s.factors), len(vs), ranks,
                                 _lib.ptr_array([c for v in vs for c in v.cores]), out.data_ptr(),
                                 ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev)))
    return out


def kr_apply_batch(s: KhatriRaoSketch, vs) -> torch.Tensor:
    """Sketch of every vector in `vs`: (len(vs), rows) device tensor, one launch."""
    return kr_apply_rows(s, vs, 0, s.rows)


def kr_apply_device(s: KhatriRaoSketch, v: TTVector) -> torch.Tensor:
    """Length-s device vector (no host sync)."""
    return kr_apply_rows(s, [v], 0, s.rows)[0]


def kr_apply(s: KhatriRaoSketch, v: TTVector) -> np.ndarray:
    """Apply the sketch to a TT vector, returning a dense length-s host vector (sketch.py:50-70)."""
    if s.dims != v.dims:
        raise ShapeMismatch(f"sketch dims {s.dims} do not match vector {v.dims}")
    return kr_apply_device(s, v).cpu().numpy()


_FT_LOCK = threading.Lock()


def _premultiplied_factors(s: KhatriRaoSketch, a: TTOperator):
    """Ft_k[j, al, i', be] = sum_i F_k[j, i] D_k[al, i, i', be] for every core (one
    batched DMMA GEMM per core); cached on the sketch for the last operator used,
    keyed by the operator cores' storage and version counters (an in-place edit
    of a core invalidates it) and built under a lock (concurrent solvers)."""
    key = tuple((c.data_ptr(), c._version, tuple(c.shape)) for c in a.op_cores) + \
        tuple((f.data_ptr(), f._version) for f in s.factors)
    with _FT_LOCK:
        hit = getattr(s, "_ft_cache", None)
        if hit is not None and hit[0] == key:
            return hit[1]
        fts = _build_premultiplied(s, a)
        s._ft_cache = (key, fts)
        return fts


def _build_premultiplied(s: KhatriRaoSketch, a: TTOperator):
    lib = _lib.load()
    dev = s.factors[0].device
    fts = []
    for F, D in zip(s.factors, a.op_cores):
        p0, m, n, p1 = (int(x) for x in D.shape)
        S = s.rows
        ft = torch.empty((S, p0, n, p1), dtype=torch.float64, device=dev)
        ws = _lib.workspace(max(int(lib.ttk_gemm_strided_ws_bytes(p0, S, n * p1, m)), 8), dev)
        _lib.check(lib.ttk_gemm_strided(p0, S, n * p1, m, 1.0, F.data_ptr(), m, 1, 0, D.data_ptr(), n * p1, 1,
                                        m * n * p1, 0.0, ft.data_ptr(), p0 * n * p1, 1, n * p1,
                                        ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev)))
        fts.append(ft)
    return fts


def kr_apply_matvec_device(s: KhatriRaoSketch, a: TTOperator, v: TTVector) -> torch.Tensor:
    """Sketch of A v as a length-s device vector, without materialising A v
    (SURVEY 8(f) #3): equal to kr_apply_device(s, tt_matvec(a, v)) up to rounding."""
    if a.col_dims != v.dims:
        raise ShapeMismatch(f"operator col_dims {a.col_dims} do not match {v.dims}")
    if s.dims != a.row_dims:
        raise ShapeMismatch(f"sketch dims {s.dims} do not match operator row_dims {a.row_dims}")
    _lib.require_cuda(v.cores[0], "TT vector")
    lib = _lib.load()
    dev = s.factors[0].device
    fts = _premultiplied_factors(s, a)
    d = v.d
    rho, r = list(a.ranks), list(v.ranks)
    out = torch.empty(s.rows, dtype=torch.float64, device=dev)
    ws = _lib.workspace(int(lib.ttk_kr_sketch_matvec_ws_bytes(d, s.rows, _lib.int_array(rho), _lib.int_array(r))),
                        dev)
    _lib.check(lib.ttk_kr_sketch_matvec(d, _lib.int_array(list(v.dims)), s.rows, _lib.ptr_array(fts),
                                        _lib.int_array(rho), _lib.int_array(r), _lib.ptr_array(v.cores),
                                        out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev)))
    return out


def kr_apply_matvec(s: KhatriRaoSketch, a: TTOperator, v: TTVector) -> np.ndarray:
    """kr_apply(s, tt_matvec(a, v)) as a host vector, A v never materialised."""
    return kr_apply_matvec_device(s, a, v).cpu().numpy()
