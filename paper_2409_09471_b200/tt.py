"""TT vectors/operators on the B200 and their exact arithmetic.

Mirrors the reference module ttkrylov/tt.py: same class and function names,
argument meaning and error behaviour, but the cores are CUDA fp64 torch
tensors and every operation runs through the sm_100a kernels of
libttk_b200.so (include/ttk_b200.h).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ShapeMismatch, SizeLimit

DENSE_CAP = 1_000_000  # tt.py:16
ZERO_REL = 1e-14       # tt.py:355, the rounding zero test (quirk Q1)


def default_device():
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")


def _as_core(c, device, order):
    if isinstance(c, torch.Tensor):
        t = c.to(dtype=torch.float64)
        if device is not None and t.device != torch.device(device):
            t = t.to(device)
    else:
        t = torch.as_tensor(np.asarray(c, dtype=np.float64), device=device)
    if t.dim() != order:
        return t
    return t.contiguous()


@dataclass(frozen=True)
class RoundSpec:
    """Rounding control: relative Frobenius tolerance and optional rank cap (tt.py:30-41)."""

    rel_tol: float = 0.0
    max_rank: int | None = None

    def __post_init__(self):
        if self.rel_tol < 0:
            raise ValueError("rel_tol must be nonnegative")
        if self.max_rank is not None and self.max_rank < 1:
            raise ValueError("max_rank must be >= 1 when given")


class TTVector:
    """A d-mode tensor in TT format; core k is a (r_{k-1}, n_k, r_k) fp64 tensor (tt.py:44-79)."""

    def __init__(self, cores, device=None):
        cores = list(cores)
        if not cores:
            raise ValueError("need at least one core")
        if device is None:
            device = cores[0].device if isinstance(cores[0], torch.Tensor) else default_device()
        cores = [_as_core(c, device, 3) for c in cores]
        for k, c in enumerate(cores):
            if c.dim() != 3:
                raise ShapeMismatch(f"core {k} must be order 3, got shape {tuple(c.shape)}")
        if cores[0].shape[0] != 1 or cores[-1].shape[2] != 1:
            raise ShapeMismatch("boundary ranks must equal 1")
        for k in range(len(cores) - 1):
            if cores[k].shape[2] != cores[k + 1].shape[0]:
                raise ShapeMismatch(f"rank chain broken between cores {k} and {k + 1}")
        self.cores = cores

    @property
    def d(self) -> int:
        return len(self.cores)

    @property
    def dims(self) -> tuple[int, ...]:
        return tuple(int(c.shape[1]) for c in self.cores)

    @property
    def ranks(self) -> tuple[int, ...]:
        return (1,) + tuple(int(c.shape[2]) for c in self.cores)

    @property
    def device(self):
        return self.cores[0].device

    def copy(self) -> "TTVector":
        return TTVector([c.clone() for c in self.cores])

    def numpy(self):
        return [c.detach().cpu().numpy() for c in self.cores]

    def __repr__(self):
        return f"TTVector(dims={self.dims}, ranks={self.ranks})"


class TTOperator:
    """A linear map between d-mode tensors; core k is (rho_{k-1}, m_k, n_k, rho_k) (tt.py:82-124)."""

    def __init__(self, op_cores, device=None):
        op_cores = list(op_cores)
        if not op_cores:
            raise ValueError("need at least one core")
        if device is None:
            device = op_cores[0].device if isinstance(op_cores[0], torch.Tensor) else default_device()
        op_cores = [_as_core(c, device, 4) for c in op_cores]
        for k, c in enumerate(op_cores):
            if c.dim() != 4:
                raise ShapeMismatch(f"op core {k} must be order 4, got shape {tuple(c.shape)}")
        if op_cores[0].shape[0] != 1 or op_cores[-1].shape[3] != 1:
            raise ShapeMismatch("boundary op-ranks must equal 1")
        for k in range(len(op_cores) - 1):
            if op_cores[k].shape[3] != op_cores[k + 1].shape[0]:
                raise ShapeMismatch(f"op-rank chain broken between cores {k} and {k + 1}")
        self.op_cores = op_cores

    @property
    def d(self) -> int:
        return len(self.op_cores)

    @property
    def row_dims(self) -> tuple[int, ...]:
        return tuple(int(c.shape[1]) for c in self.op_cores)

    @property
    def col_dims(self) -> tuple[int, ...]:
        return tuple(int(c.shape[2]) for c in self.op_cores)

    @property
    def ranks(self) -> tuple[int, ...]:
        return (1,) + tuple(int(c.shape[3]) for c in self.op_cores)

    @property
    def device(self):
        return self.op_cores[0].device

    def copy(self) -> "TTOperator":
        return TTOperator([c.clone() for c in self.op_cores])

    def band_tables(self, max_w: int = 2):
        """(w, [band_k], kinds) for the structure-aware matvec, or None when a
        core is not square or some block is wider than half-bandwidth max_w.
        Built on the device once and cached: the cores must not be modified
        afterwards.  band_k[al, be, i, t] = D_k[al, i, i+t-w, be] (zero outside
        the matrix); kinds: bytes, per core and block 0 zero / 1 diagonal /
        2 banded."""
        key = ("_bands", max_w)
        if getattr(self, "_band_key", None) == key:
            return self._bands
        res = None
        if all(c.shape[1] == c.shape[2] for c in self.op_cores):
            w = 0
            for c in self.op_cores:
                idx = (c != 0).any(dim=3).any(dim=0).nonzero()
                if idx.numel():
                    w = max(w, int((idx[:, 0] - idx[:, 1]).abs().max()))
            if w <= max_w:
                bands, kinds = [], []
                for c in self.op_cores:
                    rho0, n, _, rho1 = c.shape
                    off = torch.arange(-w, w + 1, device=c.device)
                    j = torch.arange(n, device=c.device)[:, None] + off[None, :]
                    valid = (j >= 0) & (j < n)
                    g = c.permute(0, 3, 1, 2)  # (rho0, rho1, i, j)
                    bt = torch.gather(g, 3, j.clamp(0, n - 1).expand(rho0, rho1, n, 2 * w + 1))
                    bt = (bt * valid).contiguous()
                    bands.append(bt)
                    nz = bt != 0                                # (rho0, rho1, n, 2w+1)
                    any_nz = nz.any(dim=3).any(dim=2)
                    off_diag = torch.cat([nz[..., :w], nz[..., w + 1:]], dim=3).any(dim=3).any(dim=2)
                    kinds.append((any_nz.to(torch.uint8) + off_diag.to(torch.uint8)).flatten().cpu())
                res = (w, bands, bytes(torch.cat(kinds).tolist()))
        self._band_key, self._bands = key, res
        return res

    def numpy(self):
        return [c.detach().cpu().numpy() for c in self.op_cores]

    def __repr__(self):
        return (f"TTOperator(row_dims={self.row_dims}, col_dims={self.col_dims}, "
                f"ranks={self.ranks})")


# ---------------------------------------------------------------------------
# construction helpers (tt.py:131-164); Gaussian draws stay on the host
# (numpy default_rng) so seeded inputs are identical to the reference's.


def attainable_ranks(dims, ranks):
    """Clip interior ranks to the unfolding sizes in exact integers (tt.py:152-156
    without the int64 cumprod overflow, quirk Q2)."""
    dims = list(dims)
    out = [int(r) for r in ranks]
    for k in range(1, len(dims)):
        out[k - 1] = int(min(out[k - 1], math.prod(dims[:k]), math.prod(dims[k:])))
    return out


def tt_zero(dims, device=None) -> TTVector:
    return TTVector([torch.zeros((1, n, 1), dtype=torch.float64, device=device or default_device())
                     for n in dims])


def tt_rank_one(vectors, device=None) -> TTVector:
    return TTVector([np.asarray(v, dtype=np.float64).reshape(1, -1, 1) for v in vectors], device=device)


def tt_random(dims, ranks, seed=0, device=None) -> TTVector:
    """i.i.d. standard normal cores drawn k = 0..d-1 from default_rng(seed) (tt.py:141-159)."""
    dims = list(dims)
    d = len(dims)
    ranks = list(ranks) if d > 1 else []
    if len(ranks) != max(d - 1, 0):
        raise ValueError("ranks must have length d-1")
    full = [1] + attainable_ranks(dims, ranks) + [1]
    rng = np.random.default_rng(seed)
    return TTVector([rng.standard_normal((full[k], dims[k], full[k + 1])) for k in range(d)],
                    device=device)


def identity_operator(dims, device=None) -> TTOperator:
    return TTOperator([np.eye(n).reshape(1, n, n, 1) for n in dims], device=device)


def kron_sum_operator(factors, device=None) -> TTOperator:
    """Kronecker sum of square matrices with op-ranks 2 (tt.py:413-447)."""
    mats = [np.asarray(f, dtype=np.float64) for f in factors]
    for i, f in enumerate(mats):
        if f.ndim != 2 or f.shape[0] != f.shape[1]:
            raise ShapeMismatch(f"factor {i} is not square: shape {f.shape}")
    d = len(mats)
    if d == 0:
        raise ValueError("need at least one factor")
    if d == 1:
        n = mats[0].shape[0]
        return TTOperator([mats[0].reshape(1, n, n, 1)], device=device)
    cores = []
    for i, f in enumerate(mats):
        n = f.shape[0]
        eye = np.eye(n)
        if i == 0:
            c = np.zeros((1, n, n, 2))
            c[0, :, :, 0], c[0, :, :, 1] = f, eye
        elif i == d - 1:
            c = np.zeros((2, n, n, 1))
            c[0, :, :, 0], c[1, :, :, 0] = eye, f
        else:
            c = np.zeros((2, n, n, 2))
            c[0, :, :, 0], c[1, :, :, 0], c[1, :, :, 1] = eye, f, eye
        cores.append(c)
    return TTOperator(cores, device=device)


def max_rank(v) -> int:
    return max(v.ranks)


# ---------------------------------------------------------------------------
# dense conversions (tt.py:171-200) -- small test instances only


def tt_to_dense(v: TTVector, max_entries: int = DENSE_CAP) -> torch.Tensor:
    total = math.prod(v.dims)
    if total > max_entries:
        raise SizeLimit(f"dense tensor would have {total} entries (cap {max_entries})")
    m = v.cores[0].reshape(v.dims[0], -1)
    for c in v.cores[1:]:
        m = (m @ c.reshape(c.shape[0], -1)).reshape(-1, c.shape[2])
    return m.reshape(v.dims)


def tt_op_to_dense(a: TTOperator, max_entries: int = DENSE_CAP) -> torch.Tensor:
    nrow, ncol = math.prod(a.row_dims), math.prod(a.col_dims)
    if nrow * ncol > max_entries:
        raise SizeLimit(f"dense matrix would have {nrow * ncol} entries (cap {max_entries})")
    rows, cols = a.row_dims[0], a.col_dims[0]
    m = a.op_cores[0].reshape(rows * cols, -1)
    for c in a.op_cores[1:]:
        rho, mk, nk, rho2 = c.shape
        m = (m @ c.reshape(rho, -1)).reshape(rows, cols, mk, nk, rho2).permute(0, 2, 1, 3, 4)
        rows, cols = rows * mk, cols * nk
        m = m.reshape(rows * cols, rho2)
    return m.reshape(rows, cols)


# ---------------------------------------------------------------------------
# arithmetic


def _check_cuda_vec(v: TTVector, what="TT vector"):
    _lib.require_cuda(v.cores[0], what)


def tt_matvec(a: TTOperator, v: TTVector, out=None, structured: bool = False) -> TTVector:
    """Apply the operator core by core; output ranks multiply, no rounding (tt.py:302-314).

    ``out``: optional preallocated output cores (reused across calls).
    ``structured``: use the banded kernel (``ttk_matvec_banded``) when every
    operator block has half-bandwidth <= 2 (identity / tridiagonal operators,
    SURVEY 8(f) #3); same result up to summation order, otherwise the dense
    DMMA contraction (the default, the path the north star measures)."""
    if a.col_dims != v.dims:
        raise ShapeMismatch(f"operator col_dims {a.col_dims} do not match {v.dims}")
    _check_cuda_vec(v)
    lib = _lib.load()
    d = v.d
    rho, r = list(a.ranks), list(v.ranks)
    m, n = list(a.row_dims), list(a.col_dims)
    dev = v.device
    shapes = [(r[k] * rho[k], m[k], r[k + 1] * rho[k + 1]) for k in range(d)]
    if out is None:
        out = [torch.empty(sh, dtype=torch.float64, device=dev) for sh in shapes]
    elif [tuple(c.shape) for c in out] != shapes:
        raise ShapeMismatch("preallocated matvec output has the wrong shapes")
    bt = a.band_tables() if structured else None
    if bt is not None:
        _lib.check(lib.ttk_matvec_banded(d, _lib.int_array(rho), _lib.int_array(n), _lib.int_array(r), bt[0],
                                          _lib.ptr_array(bt[1]), bt[2], _lib.ptr_array(v.cores),
                                          _lib.ptr_array(out), _lib.stream_ptr(dev)))
        return TTVector(out)
    _lib.check(lib.ttk_matvec(d, _lib.int_array(rho), _lib.int_array(m), _lib.int_array(n),
                              _lib.int_array(r), _lib.ptr_array(a.op_cores), _lib.ptr_array(v.cores),
                              _lib.ptr_array(out), _lib.stream_ptr(dev)))
    return TTVector(out)


def tt_combine(terms, coeffs) -> TTVector:
    """sum_t coeff_t * term_t as one block-diagonal concatenation.

    Equal, core for core, to the reference's left-to-right chain
    tt_add(..tt_add(t0, tt_scale(t1, c1)).., tt_scale(tp, cp)) used by the
    explicit Arnoldi update (solvers.py:361-366); coeff 1.0 terms are copied
    unscaled.  One kernel launch writes every output core."""
    terms = list(terms)
    coeffs = [float(c) for c in coeffs]
    if len(terms) != len(coeffs) or not terms:
        raise ValueError("need matching, nonempty terms and coeffs")
    dims = terms[0].dims
    for t in terms[1:]:
        if t.dims != dims:
            raise ShapeMismatch(f"dims differ: {dims} vs {t.dims}")
    _check_cuda_vec(terms[0])
    lib = _lib.load()
    d = len(dims)
    dev = terms[0].device
    if len(terms) > 16:  # kernel handles 16 terms per launch; fold the rest
        head = tt_combine(terms[:16], coeffs[:16])
        return tt_combine([head] + terms[16:], [1.0] + coeffs[16:])
    ranks = [t.ranks for t in terms]
    out = []
    for k in range(d):
        if d == 1:
            shape = (1, dims[0], 1)
        else:
            r0 = 1 if k == 0 else sum(rk[k] for rk in ranks)
            r1 = 1 if k == d - 1 else sum(rk[k + 1] for rk in ranks)
            shape = (r0, dims[k], r1)
        out.append(torch.empty(shape, dtype=torch.float64, device=dev))
    flat_ranks = [x for rk in ranks for x in rk]
    flat_in = [c for t in terms for c in t.cores]
    _lib.check(lib.ttk_tt_concat(d, len(terms), _lib.double_array(coeffs), _lib.int_array(dims),
                                 _lib.int_array(flat_ranks), _lib.ptr_array(flat_in),
                                 _lib.ptr_array(out), _lib.stream_ptr(dev)))
    return TTVector(out)


def tt_add(a: TTVector, b: TTVector) -> TTVector:
    """Exact sum; interior ranks add (tt.py:254-275)."""
    if a.dims != b.dims:
        raise ShapeMismatch(f"dims differ: {a.dims} vs {b.dims}")
    return tt_combine([a, b], [1.0, 1.0])


def tt_scale(a: TTVector, alpha: float) -> TTVector:
    """Scale the denoted tensor; the last core absorbs the factor (tt.py:278-282)."""
    _check_cuda_vec(a)
    lib = _lib.load()
    cores = [c.clone() for c in a.cores[:-1]]
    last = torch.empty_like(a.cores[-1])
    _lib.check(lib.ttk_scale(last.data_ptr(), a.cores[-1].data_ptr(), last.numel(), float(alpha),
                             _lib.stream_ptr(a.device)))
    return TTVector(cores + [last])


def tt_dots(x: TTVector, ys) -> torch.Tensor:
    """<x, y_i> for every partner, one sweep with grouped GEMMs per core.

    Returns a device tensor (no host sync).  Reference tt_dot, tt.py:285-294."""
    ys = list(ys)
    for y in ys:
        if y.dims != x.dims:
            raise ShapeMismatch(f"dims differ: {x.dims} vs {y.dims}")
    _check_cuda_vec(x)
    lib = _lib.load()
    d, dev = x.d, x.device
    out = torch.empty(len(ys), dtype=torch.float64, device=dev)
    if not ys:
        return out
    dims = _lib.int_array(x.dims)
    xr = _lib.int_array(x.ranks)
    yr = _lib.int_array([r for y in ys for r in y.ranks])
    nbytes = lib.ttk_tt_dots_ws_bytes(d, dims, xr, len(ys), yr)
    ws = _lib.workspace(nbytes, dev)
    _lib.check(lib.ttk_tt_dots(d, dims, xr, _lib.ptr_array(x.cores), len(ys), yr,
                               _lib.ptr_array([c for y in ys for c in y.cores]), out.data_ptr(),
                               ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev)))
    return out


def tt_dot(a: TTVector, b: TTVector) -> float:
    """Euclidean inner product via left-to-right core contraction (tt.py:285-294)."""
    if a.dims != b.dims:
        raise ShapeMismatch(f"dims differ: {a.dims} vs {b.dims}")
    return float(tt_dots(a, [b])[0].item())


def tt_norm(a: TTVector) -> float:
    """Frobenius norm of the denoted tensor (tt.py:297-299)."""
    return float(math.sqrt(max(tt_dot(a, a), 0.0)))


# ---------------------------------------------------------------------------
# rounding (tt.py:203-211, 321-368)


def tt_round(v: TTVector, spec: RoundSpec, zero_rel: float | None = ZERO_REL) -> TTVector:
    """TT-SVD recompression on the device (tt.py:337-368).

    Right-to-left Householder-QR sweep, then left-to-right truncated SVDs with
    the per-mode budget rel_tol*||v||/sqrt(d-1) and the max_rank cap.
    ``zero_rel`` keeps the reference's cancellation test (tt.py:348-356);
    pass None to disable it (reference quirk Q1: the test fires on every
    BASELINE-size input)."""
    d = v.d
    if d == 1:
        return v.copy()
    _check_cuda_vec(v)
    lib = _lib.load()
    dev = v.device
    dims = _lib.int_array(v.dims)
    ranks = _lib.int_array(v.ranks)
    outs = [torch.empty(max(c.numel(), c.shape[1]), dtype=torch.float64, device=dev) for c in v.cores]
    out_ranks = (_lib.ctypes.c_int * (d + 1))()
    ws = _lib.workspace(lib.ttk_tt_round_ws_bytes(d, dims, ranks), dev)
    _lib.check(lib.ttk_tt_round(d, dims, ranks, _lib.ptr_array(v.cores), float(spec.rel_tol),
                                int(spec.max_rank or 0), -1.0 if zero_rel is None else float(zero_rel),
                                _lib.ptr_array(outs), out_ranks, ws.data_ptr(), ws.numel(),
                                _lib.stream_ptr(dev)))
    r = list(out_ranks)
    cores = [outs[k][: r[k] * v.dims[k] * r[k + 1]].view(r[k], v.dims[k], r[k + 1]) for k in range(d)]
    return TTVector(cores)


def tt_norm_orthogonal(v: TTVector, core: int = -1) -> float:
    """||v|| of an orthogonalised TT: the Frobenius norm of the core that
    carries it (last core after tt_round / rto_sweeps, which leave cores
    0..d-2 left-orthonormal; core 0 after tt_truncate_left_orth, which leaves
    cores 1..d-1 right-orthonormal).  One fixed-order device reduction
    instead of a full dot sweep."""
    _check_cuda_vec(v)
    lib = _lib.load()
    c = v.cores[core]
    out = torch.empty(1, dtype=torch.float64, device=v.device)
    ws = _lib.workspace(4096, v.device)
    _lib.check(lib.ttk_sumsq(c.data_ptr(), c.numel(), out.data_ptr(), ws.data_ptr(), ws.numel(),
                             _lib.stream_ptr(v.device)))
    return float(math.sqrt(max(out.item(), 0.0)))


def tt_norm_left_orthogonal(v: TTVector) -> float:
    """||v|| when cores 0..d-2 are left-orthonormal (norm in the last core)."""
    return tt_norm_orthogonal(v, -1)
