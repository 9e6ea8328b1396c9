"""Randomize-then-orthogonalize TT rounding on the B200.

Absent from the reference (SPEC.md:313 lists it as a non-goal); restated from
PAPER.md:435-445 and SURVEY.md Appendix B, with the CPU restatement in
oracle/ttoracle.py (rto_sweeps / rto_round) as the checker:

  1. right partial contractions W_c = X_{>=c}^T G_{>=c} with a Gaussian TT-DRM
     G (streaming.py:133-136 recurrence), two chained DMMA GEMMs per core;
  2. left-to-right: Y_c = Z_c W_c, Q_c = TSQR(Y_c) (explicit Householder Q),
     M_c = Q_c^T Z_c, Z_{c+1} = M_c x_1 X_c;
  3. right-to-left TT-SVD truncation of the left-orthogonal result
     (tt_truncate_left_orth; no orthogonalisation sweep needed).
"""

from __future__ import annotations

import math
import threading

import torch

from . import _lib
from .errors import ShapeMismatch
from .streaming import TTDRM, tt_drm_new
from .tt import RoundSpec, TTVector, attainable_ranks


def rto_ranks(dims, in_ranks, ell):
    """Sketch ranks l_c (c = 1..d-1): min(ell_c, R_c, attainable), then
    l_c <= l_{c-1} n_{c-1} so every QR is tall (oracle.rto_ranks)."""
    d = len(dims)
    if isinstance(ell, int):
        ell = [ell] * (d - 1)
    ls = [int(min(e, r)) for e, r in zip(ell, in_ranks[1:-1])]
    ls = attainable_ranks(list(dims), ls)
    prev = 1
    for c in range(d - 1):
        ls[c] = max(1, min(ls[c], prev * dims[c]))
        prev = ls[c]
    return ls


def rto_flops(dims, in_ranks, ls) -> float:
    """Algorithmic FLOPs of the two sweeps (QR counted as 4ml^2 - 4l^3/3)."""
    d = len(dims)
    L = [1] + list(ls) + [1]
    R = list(in_ranks)
    f = 0.0
    for c in range(d - 1, 0, -1):
        f += 2.0 * R[c] * dims[c] * R[c + 1] * L[c + 1] + 2.0 * R[c] * dims[c] * L[c + 1] * L[c]
    for c in range(1, d):
        m, l = L[c - 1] * dims[c - 1], L[c]
        f += 2.0 * m * R[c] * l + (4.0 * m * l * l - 4.0 * l ** 3 / 3.0) + 2.0 * l * m * R[c]
        f += 2.0 * l * R[c] * dims[c] * R[c + 1]
    return f


class CounterDRM:
    """Gaussian TT-DRM generated on the device from a counter-based RNG
    (csrc/drm.cu, ttk_drm_gaussian): entry (i, j, l) of core k depends only on
    (seed, k, i, j, l) in the full index space, with variance 1/(R_{k-1} n_k R_k)
    of the full ranks as tt_drm_new draws it.  ``block(ls)`` returns the
    leading (l_{k-1} x n_k x l_k) blocks -- identical to slicing the full map --
    so a solver whose sketch ranks grow never draws the cap-sized DRM.
    ``cores`` materialises the full map (tests hand it to the CPU oracle)."""

    def __init__(self, dims, ranks, seed=0, device=None):
        self.dims = tuple(int(n) for n in dims)
        d = len(self.dims)
        ranks = list(ranks)
        if len(ranks) != d - 1 or any(r < 1 for r in ranks):
            raise ValueError("ranks must be d-1 positive integers")
        self.ranks = tuple([1] + ranks + [1])
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self.device = torch.device(device) if device is not None else torch.device("cuda", 0)
        _lib.require_cuda(torch.empty(0, device=self.device), "CounterDRM")

    def block(self, ls):
        L = [1] + [int(x) for x in ls] + [1]
        if len(L) != len(self.ranks) or any(a > b for a, b in zip(L, self.ranks)):
            raise ShapeMismatch(f"sketch ranks {L} exceed the DRM ranks {self.ranks}")
        lib = _lib.load()
        st = _lib.stream_ptr(self.device)
        R = self.ranks
        out = []
        for k, n in enumerate(self.dims):
            g = torch.empty((L[k], n, L[k + 1]), dtype=torch.float64, device=self.device)
            scale = 1.0 / math.sqrt(float(R[k]) * n * R[k + 1])
            _lib.check(lib.ttk_drm_gaussian(self.seed, k, n, R[k], R[k + 1], L[k], L[k + 1], scale,
                                            g.data_ptr(), st))
            out.append(g)
        return out

    @property
    def cores(self):
        return self.block(self.ranks[1:-1])


def _drm_slices(drm_cores, ls, device):
    full = [1] + list(ls) + [1]
    out = []
    for k, g in enumerate(drm_cores):
        if g.shape[0] < full[k] or g.shape[2] < full[k + 1]:
            raise ShapeMismatch(f"DRM core {k} of shape {tuple(g.shape)} is smaller than the sketch ranks")
        s = g[: full[k], :, : full[k + 1]]
        out.append(s if s.is_contiguous() else s.contiguous())
    return out


def rto_sweeps(v: TTVector, drm) -> TTVector:
    """Left-orthogonal TT with the DRM's ranks (clamped by rto_ranks)."""
    d = v.d
    _lib.require_cuda(v.cores[0], "TT vector")
    if isinstance(drm, CounterDRM):
        if drm.dims != v.dims:
            raise ShapeMismatch("DRM dims do not match the vector")
        if d == 1:
            return v.copy()
        ls = rto_ranks(v.dims, v.ranks, list(drm.ranks[1:-1]))
        G = drm.block(ls)
    else:
        if isinstance(drm, TTDRM):
            drm = drm.cores
        if tuple(int(g.shape[1]) for g in drm) != v.dims:
            raise ShapeMismatch("DRM dims do not match the vector")
        if d == 1:
            return v.copy()
        ls = rto_ranks(v.dims, v.ranks, [int(g.shape[2]) for g in drm[:-1]])
        G = _drm_slices(drm, ls, v.device)
    lib = _lib.load()
    dev = v.device
    L = [1] + ls + [1]
    out = [torch.empty((L[k], v.dims[k], L[k + 1]), dtype=torch.float64, device=dev) for k in range(d)]
    dims = _lib.int_array(v.dims)
    R = _lib.int_array(v.ranks)
    Lc = _lib.int_array(L)
    ws = _lib.workspace(lib.ttk_rto_ws_bytes(d, dims, R, Lc), dev)
    _lib.check(lib.ttk_rto_sweeps(d, dims, R, _lib.ptr_array(v.cores), Lc, _lib.ptr_array(G),
                                  _lib.ptr_array(out), ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev)))
    return TTVector(out)


def tt_truncate_left_orth(v: TTVector, spec: RoundSpec) -> TTVector:
    """TT-SVD truncation of a LEFT-orthogonal TT, right to left (cores 0..d-2
    left-orthonormal, e.g. rto_sweeps output): per core one TSQR of the
    transposed right unfolding, a Jacobi SVD of its R factor and two GEMMs;
    budget rel_tol ||v|| / sqrt(d-1) and the max_rank cap as tt_round
    (tt.py:357-364).  Oracle: oracle.truncate_left_orth."""
    d = v.d
    if d == 1:
        return v.copy()
    _lib.require_cuda(v.cores[0], "TT vector")
    lib = _lib.load()
    dev = v.device
    dims = _lib.int_array(v.dims)
    ranks = _lib.int_array(v.ranks)
    outs = [torch.empty(max(c.numel(), c.shape[1]), dtype=torch.float64, device=dev) for c in v.cores]
    out_ranks = (_lib.ctypes.c_int * (d + 1))()
    ws = _lib.workspace(lib.ttk_tt_truncate_ws_bytes(d, dims, ranks), dev)
    _lib.check(lib.ttk_tt_truncate(d, dims, ranks, _lib.ptr_array(v.cores), float(spec.rel_tol),
                                   int(spec.max_rank or 0), _lib.ptr_array(outs), out_ranks, ws.data_ptr(),
                                   ws.numel(), _lib.stream_ptr(dev)))
    r = list(out_ranks)
    return TTVector([outs[k][: r[k] * v.dims[k] * r[k + 1]].view(r[k], v.dims[k], r[k + 1]) for k in range(d)])


def tt_round_rto(v: TTVector, spec: RoundSpec, ell=None, drm=None, seed=0) -> TTVector:
    """Randomized rounding: RTO sweeps at sketch rank ``ell`` (or with the
    given DRM), then the right-to-left TT-SVD truncation to ``spec``.

    ell defaults to max_rank + 20 (oversampling as in the reference's
    StreamFrame, streaming.py:78).  The DRM is drawn on the host with
    tt_drm_new(dims, l, seed) so CPU and GPU see identical sketches."""
    if drm is None:
        if ell is None:
            if spec.max_rank is None:
                raise ValueError("tt_round_rto needs ell, drm or spec.max_rank")
            ell = spec.max_rank + 20
        ls = rto_ranks(v.dims, v.ranks, ell)
        drm = tt_drm_new(v.dims, ls, seed=seed, device=v.device)
    return tt_truncate_left_orth(rto_sweeps(v, drm), spec)


_PIPE_STREAMS = {}
_PIPE_LOCK = threading.Lock()


def _pipe_streams(dev):
    """(upload, matvec) side streams of the caller's current stream: independent
    callers on their own streams (bench.py inflight, concurrent solves) get
    their own pair, so their pipelines do not serialise on shared streams."""
    key = (dev.index, torch.cuda.current_stream(dev).cuda_stream)
    with _PIPE_LOCK:
        pair = _PIPE_STREAMS.get(key)
        if pair is None:
            pair = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
            _PIPE_STREAMS[key] = pair
    return pair


def _drm_block(v_dims, v_ranks, drm, dev):
    """Sketch ranks and DRM cores for rto_sweeps (same rules as rto_sweeps)."""
    if isinstance(drm, CounterDRM):
        if drm.dims != tuple(v_dims):
            raise ShapeMismatch("DRM dims do not match the vector")
        ls = rto_ranks(v_dims, v_ranks, list(drm.ranks[1:-1]))
        return ls, drm.block(ls)
    if isinstance(drm, TTDRM):
        drm = drm.cores
    if tuple(int(g.shape[1]) for g in drm) != tuple(v_dims):
        raise ShapeMismatch("DRM dims do not match the vector")
    ls = rto_ranks(v_dims, v_ranks, [int(g.shape[2]) for g in drm[:-1]])
    return ls, _drm_slices(drm, ls, dev)


def tt_matvec_round_rto(a, v: TTVector, spec: RoundSpec, drm, chunk: int | None = None, device=None) -> TTVector:
    """tt_truncate_left_orth(rto_sweeps(tt_matvec(a, v), drm), spec) as one
    stream-overlapped pipeline -- the matvec + randomized rounding step of
    tt_sgmres (solvers.py:356-368 with the rounding of SURVEY App. B).

    * operator and vector cores may live in (pinned) host memory: they are
      uploaded core by core from the right on a copy stream, and each chunk of
      ``chunk`` cores (default 4) is contracted (ttk_matvec_range) as soon as it
      has landed; device-resident inputs default to one launch over all cores
      (r01, config 3: chunks of 4 cost 0.6 ms more in launch efficiency than
      the overlap with the right sweep recovers);
    * the RTO right sweep waits per core (ttk_rto_sweeps_ev), so it starts on
      the last cores while the first ones are still uploading / contracting;
    * with host inputs the result comes back in pinned host memory, each core
      copied as soon as the truncation finalises it (ttk_tt_truncate_host).
    Same arithmetic and result as the three calls in sequence."""
    torch.cuda.nvtx.range_push("ttk/matvec_round_rto")
    try:
        return _matvec_round_rto(a, v, spec, drm, chunk, device)
    finally:
        torch.cuda.nvtx.range_pop()


def _matvec_round_rto(a, v, spec, drm, chunk, device):
    if a.col_dims != v.dims:
        raise ShapeMismatch(f"operator col_dims {a.col_dims} do not match {v.dims}")
    host = v.device.type == "cpu"
    if host != (a.op_cores[0].device.type == "cpu"):
        raise ValueError("operator and vector must both be in host memory or both on the device")
    if not host:
        _lib.require_cuda(v.cores[0], "TT vector")
    dev = (torch.device(device) if device is not None
           else (torch.device("cuda", torch.cuda.current_device()) if host else v.device))
    lib = _lib.load()
    d = v.d
    rho, r = list(a.ranks), list(v.ranks)
    m, n = list(a.row_dims), list(a.col_dims)
    cur = torch.cuda.current_stream(dev)
    up, mvs = _pipe_streams(dev)
    if host:
        xs = [torch.empty(tuple(c.shape), dtype=torch.float64, device=dev) for c in v.cores]
        ops = [torch.empty(tuple(c.shape), dtype=torch.float64, device=dev) for c in a.op_cores]
        ev_up = [torch.cuda.Event() for _ in range(d)]
        up.wait_stream(cur)  # the buffers were allocated on `cur`
        with torch.cuda.stream(up):
            for k in reversed(range(d)):
                ops[k].copy_(a.op_cores[k], non_blocking=True)
                xs[k].copy_(v.cores[k], non_blocking=True)
                ev_up[k].record(up)
        for t in ops + xs:
            t.record_stream(up)
    else:
        xs, ops, ev_up = list(v.cores), list(a.op_cores), None
    yr = [r[k] * rho[k] for k in range(d + 1)]
    y = [torch.empty((yr[k], m[k], yr[k + 1]), dtype=torch.float64, device=dev) for k in range(d)]
    # the DRM block is drawn on `cur` before the matvec stream starts
    ls, G = _drm_block(m, yr, drm, dev)
    mvs.wait_stream(cur)
    rho_a, m_a, n_a, r_a = (_lib.int_array(x) for x in (rho, m, n, r))
    D_p, C_p, Y_p = _lib.ptr_array(ops), _lib.ptr_array(xs), _lib.ptr_array(y)
    ev_mv = [None] * d
    if chunk is None:
        chunk = 4 if host else d
    chunk = max(1, int(chunk))
    for k1 in range(d, 0, -chunk):
        k0 = max(0, k1 - chunk)
        if ev_up is not None:
            mvs.wait_event(ev_up[k0])  # uploads run right to left: core k0 lands last
        _lib.check(lib.ttk_matvec_range(d, rho_a, m_a, n_a, r_a, D_p, C_p, Y_p, k0, k1, mvs.cuda_stream))
        e = torch.cuda.Event()
        e.record(mvs)
        for k in range(k0, k1):
            ev_mv[k] = e
    # RTO sweeps on `cur`, each core awaited on its matvec chunk's event
    L = [1] + ls + [1]
    z = [torch.empty((L[k], m[k], L[k + 1]), dtype=torch.float64, device=dev) for k in range(d)]
    if d == 1:
        cur.wait_event(ev_mv[0])
        z[0].copy_(y[0])
    else:
        dims_a, yr_a, L_a = _lib.int_array(m), _lib.int_array(yr), _lib.int_array(L)
        ws = _lib.workspace(lib.ttk_rto_ws_bytes(d, dims_a, yr_a, L_a), dev)
        ready = (_lib.ctypes.c_void_p * d)(*[e.cuda_event for e in ev_mv])
        _lib.check(lib.ttk_rto_sweeps_ev(d, dims_a, yr_a, _lib.ptr_array(y), L_a, _lib.ptr_array(G),
                                         _lib.ptr_array(z), ws.data_ptr(), ws.numel(), ready, cur.cuda_stream))
    for t in ops + xs + y:  # read on `mvs` / `cur`: keep the blocks until both are done
        t.record_stream(mvs)
    zt = TTVector(z)
    if not host:
        return tt_truncate_left_orth(zt, spec)
    # truncation with every final core streamed into pinned host memory
    dims_a, ranks_a = _lib.int_array(zt.dims), _lib.int_array(zt.ranks)
    outs = [torch.empty(max(c.numel(), c.shape[1]), dtype=torch.float64, device=dev) for c in z]
    hosts = [torch.empty(max(c.numel(), c.shape[1]), dtype=torch.float64, pin_memory=True) for c in z]
    out_ranks = (_lib.ctypes.c_int * (d + 1))()
    if d == 1:
        hosts[0].copy_(z[0].reshape(-1))
        return TTVector([hosts[0][: m[0]].view(1, m[0], 1)])
    ws = _lib.workspace(lib.ttk_tt_truncate_ws_bytes(d, dims_a, ranks_a), dev)
    _lib.check(lib.ttk_tt_truncate_host(d, dims_a, ranks_a, _lib.ptr_array(z), float(spec.rel_tol),
                                        int(spec.max_rank or 0), _lib.ptr_array(outs), out_ranks,
                                        _lib.ptr_array(hosts), ws.data_ptr(), ws.numel(), cur.cuda_stream))
    rr = list(out_ranks)
    return TTVector([hosts[k][: rr[k] * m[k] * rr[k + 1]].view(rr[k], m[k], rr[k + 1]) for k in range(d)])
