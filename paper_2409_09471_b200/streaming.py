"""Streaming two-sided sketches of TT vectors on the B200 (mirrors ttkrylov/streaming.py).

TT-DRMs are drawn on the host with numpy default_rng (identical draws to the
reference) and uploaded once; partial contractions, Psi/Omega assembly,
pair combination and the generalised-Nystrom recovery run on the device.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .errors import DegenerateRecovery, ShapeMismatch
from .tt import RoundSpec, TTVector, attainable_ranks, default_device, tt_round, tt_zero, ZERO_REL

PINV_RCOND = 1e-12  # streaming.py:17


class TTDRM:
    """Random Gaussian TT used as a dimension-reduction map (streaming.py:24-35)."""

    def __init__(self, dims, ranks, cores, seed=None):
        self.dims = tuple(dims)
        self.ranks = tuple(ranks)
        self.cores = cores
        self.seed = seed


def tt_drm_new(dims, ranks, seed=0, device=None) -> TTDRM:
    """Core k ~ N(0, 1/(l_{k-1} n_k l_k)), drawn k = 0..d-1 on the host (streaming.py:38-53)."""
    dims = list(dims)
    d = len(dims)
    ranks = list(ranks)
    if len(ranks) != d - 1:
        raise ValueError("ranks must have length d-1")
    if any(r < 1 for r in ranks):
        raise ValueError("ranks must be positive")
    full = [1] + ranks + [1]
    rng = np.random.default_rng(seed)
    device = device or default_device()
    cores = []
    for k in range(d):
        var = 1.0 / (full[k] * dims[k] * full[k + 1])
        c = rng.normal(0.0, np.sqrt(var), size=(full[k], dims[k], full[k + 1]))
        cores.append(torch.as_tensor(c, device=device))
    return TTDRM(dims, tuple(full), cores, seed=seed)


class StreamFrame:
    """Left/right TT-DRM pair fixed for a sketch stream (streaming.py:56-97)."""

    def __init__(self, right: TTDRM, left: TTDRM):
        if right.dims != left.dims:
            raise ShapeMismatch("left/right DRM dims differ")
        for lm, rm in zip(left.ranks[1:-1], right.ranks[1:-1]):
            if lm <= rm:
                raise ValueError("left ranks must exceed recovery ranks")
        self.right = right
        self.left = left
        self.dims = right.dims

    @property
    def recovery_ranks(self):
        return self.right.ranks

    @classmethod
    def create(cls, dims, recovery_ranks, oversampling: int = 20, seed=0, device=None) -> "StreamFrame":
        """Recovery ranks clipped in exact integers (no int64 overflow, quirk Q2)."""
        dims = list(dims)
        ranks = list(recovery_ranks)
        if len(ranks) != len(dims) - 1:
            raise ValueError("recovery_ranks must have length d-1")
        if oversampling < 1:
            raise ValueError("oversampling must be >= 1")
        ranks = attainable_ranks(dims, ranks)
        lranks = [r + oversampling for r in ranks]
        s_right, s_left = np.random.SeedSequence(seed).spawn(2)
        return cls(right=tt_drm_new(dims, ranks, seed=s_right, device=device),
                   left=tt_drm_new(dims, lranks, seed=s_left, device=device))


class SketchPair:
    """Per-mode sketches Psi_mu ((l_{mu-1} n_mu) x r_mu) and Omega_mu (device tensors)."""

    def __init__(self, psi, omega, dims):
        self.psi = psi
        self.omega = omega
        self.dims = tuple(dims)

    def copy(self) -> "SketchPair":
        return SketchPair([p.clone() for p in self.psi], [o.clone() for o in self.omega], self.dims)


def stream_sketch(t: TTVector, frame: StreamFrame) -> SketchPair:
    """Two-sided partial-contraction sketches (streaming.py:117-142)."""
    if t.dims != frame.dims:
        raise ShapeMismatch(f"tensor dims {t.dims} do not match frame {frame.dims}")
    _lib.require_cuda(t.cores[0], "TT vector")
    lib = _lib.load()
    d, dev = t.d, t.device
    lr, rr = list(frame.left.ranks), list(frame.right.ranks)
    psi = [torch.empty((lr[mu] * t.dims[mu], rr[mu + 1]), dtype=torch.float64, device=dev) for mu in range(d)]
    omega = [torch.empty((lr[mu], rr[mu]), dtype=torch.float64, device=dev) for mu in range(1, d)]
    dims = _lib.int_array(t.dims)
    tr = _lib.int_array(t.ranks)
    li, ri = _lib.int_array(lr), _lib.int_array(rr)
    ws = _lib.workspace(lib.ttk_stream_sketch_ws_bytes(d, dims, tr, li, ri), dev)
    _lib.check(lib.ttk_stream_sketch(d, dims, tr, _lib.ptr_array(t.cores), li, _lib.ptr_array(frame.left.cores),
                                     ri, _lib.ptr_array(frame.right.cores), _lib.ptr_array(psi),
                                     _lib.ptr_array(omega), ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev)))
    return SketchPair(psi, omega, t.dims)


def _axpy(tensors, coeffs):
    lib = _lib.load()
    out = torch.empty_like(tensors[0])
    _lib.check(lib.ttk_axpy_multi(len(tensors), _lib.double_array(coeffs), _lib.ptr_array(tensors),
                                  out.numel(), out.data_ptr(), _lib.stream_ptr(out.device)))
    return out


def combine_pairs(pairs, coeffs) -> SketchPair:
    """Entrywise weighted sum of sketch pairs from one frame (streaming.py:145-163)."""
    if len(pairs) != len(coeffs) or not pairs:
        raise ValueError("need matching, nonempty pairs and coeffs")
    first = pairs[0]
    for p in pairs[1:]:
        if p.dims != first.dims:
            raise ShapeMismatch("pairs come from different frames")
        for a, b in zip(p.psi, first.psi):
            if a.shape != b.shape:
                raise ShapeMismatch("pairs come from different frames")
        for a, b in zip(p.omega, first.omega):
            if a.shape != b.shape:
                raise ShapeMismatch("pairs come from different frames")
    coeffs = [float(c) for c in coeffs]
    psi = [_axpy([p.psi[k] for p in pairs], coeffs) for k in range(len(first.psi))]
    omega = [_axpy([p.omega[k] for p in pairs], coeffs) for k in range(len(first.omega))]
    return SketchPair(psi, omega, first.dims)


def stream_recover(pair: SketchPair, spec: RoundSpec = RoundSpec(), zero_rel: float | None = ZERO_REL) -> TTVector:
    """Generalised-Nystrom recovery with symmetric S^{-1/2} pinv split, then
    tt_round (streaming.py:166-205)."""
    d = len(pair.psi)
    dims = pair.dims
    dev = pair.psi[0].device
    _lib.require_cuda(pair.psi[0], "sketch pair")
    lib = _lib.load()
    lr = [1] + [int(o.shape[0]) for o in pair.omega] + [1]
    rr = [1] + [int(o.shape[1]) for o in pair.omega] + [1]
    di, li, ri = _lib.int_array(dims), _lib.int_array(lr), _lib.int_array(rr)
    cap = [max(lr[mu], rr[mu]) * dims[mu] * rr[mu + 1] for mu in range(d)]
    outs = [torch.empty(max(c, 1), dtype=torch.float64, device=dev) for c in cap]
    out_ranks = (_lib.ctypes.c_int * (d + 1))()
    is_zero = _lib.ctypes.c_int(0)
    ws = _lib.workspace(lib.ttk_stream_recover_ws_bytes(d, di, li, ri), dev)
    _lib.check(lib.ttk_stream_recover_cores(d, di, li, ri, _lib.ptr_array(pair.psi), _lib.ptr_array(pair.omega),
                                            PINV_RCOND, _lib.ptr_array(outs), out_ranks,
                                            _lib.ctypes.byref(is_zero), ws.data_ptr(), ws.numel(),
                                            _lib.stream_ptr(dev)))
    if is_zero.value:
        return tt_zero(dims, device=dev)
    r = list(out_ranks)
    cores = [outs[k][: r[k] * dims[k] * r[k + 1]].view(r[k], dims[k], r[k + 1]) for k in range(d)]
    return tt_round(TTVector(cores), spec, zero_rel=zero_rel)
