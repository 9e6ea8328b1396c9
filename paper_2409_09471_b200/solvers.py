"""TT-sGMRES on the B200 (mirrors ttkrylov/solvers.py: SolverConfig, SolveReport,
tt_sgmres, make_solver_frame, sketched_lsq, true_residual).

The Krylov loop keeps every TT vector on the device; per iteration it runs
the matvec, one batched dot sweep, the Khatri-Rao sketch of the unrounded
matvec output, one concatenation launch for the explicit Arnoldi update,
the rounding (TT-SVD, or randomize-then-orthogonalize + TT-SVD truncation)
and the streaming sketch of the new basis vector.  Only the s x k sketched
least-squares problem (s <= a few hundred) is solved on the host, as in the
reference (solvers.py:399-400).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ShapeMismatch
from .rto import CounterDRM, rto_ranks, rto_sweeps, tt_truncate_left_orth
from .sketch import KhatriRaoSketch, kr_apply
from .streaming import StreamFrame, combine_pairs, stream_recover, stream_sketch, tt_drm_new
from .tt import (ZERO_REL, RoundSpec, TTOperator, TTVector, tt_combine, tt_dots, tt_matvec, tt_norm,
                 tt_norm_orthogonal, tt_round, tt_scale)

PHASES = ("matvec", "sketch", "orth", "round", "lsq", "recovery")

_LSQ_RCOND = 1e-12          # solvers.py:43
_BREAKDOWN_FACTOR = 1e-14   # solvers.py:44
_CONDITION_WATERMARK = 1e-10  # solvers.py:45


@dataclass
class SolverConfig:
    """Solver knobs (solvers.py:48-79) plus the B200 extensions:

    rounding      "svd" (reference TT-SVD tt_round) or "rto" (randomize-then-
                  orthogonalize sweeps at sketch rank max_rank + rto_oversampling,
                  one TT-DRM per solve drawn with seed+2, then the right-to-left
                  TT-SVD truncation of the left-orthogonal result)
    zero_rel      the reference's rounding zero test (tt.py:348-356); None
                  disables it (reference quirk Q1 -- needed at BASELINE sizes)
    """

    maxit: int = 200
    tol: float = 1e-6
    ell: int = 1
    eta: float = 0.3
    max_rank: int | None = None
    sketch_rows: int | None = None
    oversampling: int = 20
    solution_rank: int | None = None
    combine_mode: str = "explicit"
    seed: int = 0
    track_true_residual: bool = False
    force_iterations: bool = False
    rounding: str = "svd"
    zero_rel: float | None = ZERO_REL
    rto_oversampling: int = 20
    rto_ell: int | None = None

    def __post_init__(self):
        if not (0 < self.tol < 1):
            raise ValueError("tol must lie in (0, 1)")
        if self.ell < 1:
            raise ValueError("ell must be >= 1")
        if not (0 < self.eta <= 1):
            raise ValueError("eta must lie in (0, 1]")
        if self.maxit < 1:
            raise ValueError("maxit must be >= 1")
        if self.combine_mode not in ("explicit", "stta"):
            raise ValueError("combine_mode must be 'explicit' or 'stta'")
        if self.rounding not in ("svd", "rto"):
            raise ValueError("rounding must be 'svd' or 'rto'")
        if self.rounding == "rto" and self.max_rank is None and self.rto_ell is None:
            raise ValueError("rto rounding needs max_rank or rto_ell")
        if self.sketch_rows is None:
            self.sketch_rows = 2 * self.maxit
        if self.sketch_rows <= self.maxit:
            raise ValueError("sketch_rows must exceed maxit")


@dataclass
class SolveReport:
    """Per-iteration history plus run-level outcomes of one solve (solvers.py:82-102)."""

    converged: bool = False
    iterations: int = 0
    res_sketched: list = field(default_factory=list)
    res_true: list | None = None
    basis_rank: list = field(default_factory=list)
    times: dict = field(default_factory=lambda: {p: [] for p in PHASES})
    seed: int = 0
    warnings: list = field(default_factory=list)
    max_resident_basis: int = 0
    wall_time: float = 0.0
    time_to_tol: dict = field(default_factory=dict)

    @property
    def peak_rank(self) -> int:
        return max(self.basis_rank, default=0)

    def phase_totals(self) -> dict:
        return {p: float(sum(v)) for p, v in self.times.items()}


class _PhaseTimer:
    """CUDA-event phase timer (the reference's _PhaseTimer, solvers.py:105-116,
    with the same phase names): events are recorded on the stream without host
    syncs and resolved once at the end of the solve; every phase is also an
    NVTX range ("ttk/<phase>") for Nsight timelines."""

    def __init__(self, report, device):
        self.report = report
        self.device = device
        self.rows = []
        self.cur = []
        self.open = False

    def mark(self, phase):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.current_stream(self.device))
        self.cur.append((phase, ev))
        if self.open:
            torch.cuda.nvtx.range_pop()
            self.open = False
        if phase is not None:
            torch.cuda.nvtx.range_push("ttk/" + phase)
            self.open = True

    def flush(self):
        self.rows.append(self.cur)
        self.cur = []

    def resolve(self):
        torch.cuda.synchronize(self.device)
        for row in self.rows:
            acc = {p: 0.0 for p in PHASES}
            for (p0, e0), (_, e1) in zip(row, row[1:]):
                if p0 is not None:
                    acc[p0] += e0.elapsed_time(e1) * 1e-3
            for p in PHASES:
                self.report.times[p].append(acc[p])


def sketched_lsq(w: np.ndarray, rhs: np.ndarray):
    """min_y ||w y - rhs|| via the SVD pseudo-inverse, rcond 1e-12 (solvers.py:119-126)."""
    y, res, _ = _lsq_svd(w, rhs)
    return y, res


def _lsq_svd(w, rhs):
    if w.ndim != 2 or w.shape[0] < w.shape[1]:
        raise ValueError("need a tall (s >= k) matrix")
    y, _, _, sv = np.linalg.lstsq(w, rhs, rcond=_LSQ_RCOND)
    return y, float(np.linalg.norm(w @ y - rhs)), sv


def true_residual(a: TTOperator, b: TTVector, x: TTVector, zero_rel: float | None = ZERO_REL) -> float:
    """||b - A x|| / ||b||, one rounding at 1e-12 (solvers.py:137-141)."""
    r = tt_round(tt_combine([b, tt_matvec(a, x)], [1.0, -1.0]), RoundSpec(1e-12), zero_rel=zero_rel)
    nb = tt_norm(b)
    return tt_norm(r) / nb if nb > 0 else tt_norm(r)


def default_solution_rank(b: TTVector, cfg: SolverConfig) -> int:
    if cfg.solution_rank is not None:
        return cfg.solution_rank
    return max(max(b.ranks) * 2, 20)


def make_solver_frame(b: TTVector, cfg: SolverConfig, seed) -> StreamFrame:
    """One frame per run; recovery ranks cover b and twice the solution rank
    (solvers.py:150-155, clipped in exact integers -- quirk Q2)."""
    sol = default_solution_rank(b, cfg)
    ranks = [max(r, 2 * sol) for r in b.ranks[1:-1]]
    return StreamFrame.create(b.dims, ranks, oversampling=cfg.oversampling, seed=seed, device=b.device)


def _is_zero(v) -> bool:
    if v is None:
        return True
    return all(not bool(torch.any(c != 0)) for c in v.cores)


def solver_rto_drm(dims, cfg: SolverConfig, device=None):
    """The per-solve TT-DRM of the 'rto' rounding mode: sketch ranks
    l = max_rank + rto_oversampling (or rto_ell), clipped to attainable and
    progressive l_c <= l_{c-1} n_{c-1}; seed cfg.seed + 2."""
    cap = cfg.rto_ell if cfg.rto_ell is not None else cfg.max_rank + cfg.rto_oversampling
    d = len(dims)
    ls = rto_ranks(list(dims), [1] + [10 ** 9] * (d - 1) + [1], cap)
    # generated on the device block by block as the sketch ranks grow (rto.CounterDRM):
    # a host draw of the cap-sized map cost ~2.6 s per config-5 solve
    return CounterDRM(dims, ls, seed=cfg.seed + 2, device=device)


class _SketchedRun:
    """Explicit/STTA sketched GMRES with sketch-only basis memory (solvers.py:292-431)."""

    def __init__(self, a, b, x0, cfg, sketch, frame, precond=None):
        if sketch.dims != b.dims:
            raise ShapeMismatch("sketch dims do not match the right-hand side")
        if a.col_dims != b.dims or a.row_dims != b.dims:
            raise ShapeMismatch("operator dims do not match the right-hand side")
        self.a, self.b, self.cfg, self.sketch, self.frame = a, b, cfg, sketch, frame
        self.precond = precond
        self.x0 = None if _is_zero(x0) else x0
        self.report = SolveReport(seed=cfg.seed)
        self.device = b.device
        self.timer = _PhaseTimer(self.report, self.device)
        self.window = []
        self.w_cols = []
        self.pairs = []
        self.gram = {}
        self.rto_drm = solver_rto_drm(b.dims, cfg, self.device) if cfg.rounding == "rto" else None

    def _round(self, v, spec):
        if self.cfg.rounding == "svd":
            return tt_round(v, spec, zero_rel=self.cfg.zero_rel)
        return tt_truncate_left_orth(rto_sweeps(v, self.rto_drm), spec)

    def _rounded_norm(self, v):
        """||v|| of a rounded vector from the core carrying the norm: the last
        core after tt_round (left-orthogonal), core 0 after the right-to-left
        truncation of the rto mode (right-orthogonal)."""
        core = 0 if (self.cfg.rounding == "rto" and self.cfg.combine_mode == "explicit") else -1
        return tt_norm_orthogonal(v, core)

    def run(self):
        cfg = self.cfg
        t_start = time.perf_counter()
        tm = self.timer
        tm.mark("sketch")
        nb_sketch = float(np.linalg.norm(kr_apply(self.sketch, self.b)))
        if self.x0 is None:
            r0 = self.b.copy()
        else:
            r0 = tt_combine([self.b, tt_matvec(self.a, self.x0)], [1.0, -1.0])
        beta = tt_norm(r0)
        if beta == 0 or nb_sketch == 0:
            self.report.converged = True
            return (self.x0.copy() if self.x0 is not None else self.b.copy()), self.report
        v1 = tt_scale(r0, 1.0 / beta)
        sr0 = kr_apply(self.sketch, r0)
        self.pairs.append(stream_sketch(v1, self.frame))
        self.x0_pair = stream_sketch(self.x0, self.frame) if self.x0 is not None else None
        self.window = [(0, v1)]
        spec_basis = RoundSpec(cfg.eta * cfg.tol, cfg.max_rank)
        y = np.zeros(1)
        k_done = 0
        converged = False
        for k in range(1, cfg.maxit + 1):
            kk = k - 1
            tm.mark("matvec")
            vt = self.window[-1][1]
            if self.precond is not None:  # right preconditioning: A P^{-1} v (solvers.py:315-320)
                vt = self.precond.apply_inverse(vt)
            vt = tt_matvec(self.a, vt)
            tm.mark("orth")
            # one dot sweep: <vt, vt> and <vt, v_i> for the window (MGS
            # coefficients follow from the cached window Gram matrix)
            dv = tt_dots(vt, [vt] + [v for _, v in self.window]).cpu().numpy()
            norm_av = float(np.sqrt(max(dv[0], 0.0)))
            tm.mark("sketch")
            self.w_cols.append(kr_apply(self.sketch, vt))
            tm.mark("orth")
            if cfg.combine_mode == "explicit":
                hs = []
                for i, (gi, _) in enumerate(self.window):
                    h = dv[1 + i]
                    for j in range(i):
                        h -= hs[j] * self.gram[(self.window[j][0], gi)]
                    hs.append(float(h))
                vt = tt_combine([vt] + [v for _, v in self.window], [1.0] + [-h for h in hs])
                tm.mark("round")
                vt = self._round(vt, spec_basis)
            else:
                hs = [float(dv[1 + i]) for i in range(len(self.window))]
                pv = stream_sketch(vt, self.frame)
                tm.mark("round")
                comb = combine_pairs([pv] + [self.pairs[gi] for gi, _ in self.window],
                                     [1.0] + [-h for h in hs])
                vt = stream_recover(comb, spec_basis, zero_rel=cfg.zero_rel)
            hnew = self._rounded_norm(vt)
            lucky = hnew <= _BREAKDOWN_FACTOR * norm_av
            if not lucky:
                vnew = tt_scale(vt, 1.0 / hnew)
                tm.mark("sketch")
                self.pairs.append(stream_sketch(vnew, self.frame))
                tm.mark("orth")
                self.report.max_resident_basis = max(self.report.max_resident_basis, len(self.window) + 1)
                if len(self.window) >= 1 and cfg.combine_mode == "explicit":
                    g = tt_dots(vnew, [v for _, v in self.window]).cpu().numpy()
                    for (gi, _), val in zip(self.window, g):
                        self.gram[(gi, k)] = float(val)
                self.window.append((k, vnew))
                if len(self.window) > cfg.ell:
                    old = self.window.pop(0)[0]
                    self.gram = {key: v for key, v in self.gram.items() if old not in key}
            tm.mark("lsq")
            w = np.stack(self.w_cols, axis=1)
            y, res, sv = _lsq_svd(w, sr0)
            if sv.size and sv[-1] < _CONDITION_WATERMARK * sv[0]:
                msg = f"iteration {k}: sketched basis nearly rank-deficient"
                if not self.report.warnings or self.report.warnings[-1][:9] != msg[:9]:
                    self.report.warnings.append(msg)
            rel = res / nb_sketch
            self.report.res_sketched.append(rel)
            self.report.basis_rank.append(max((max(v.ranks) for _, v in self.window), default=1))
            for thr in (1e-6,):
                if rel <= thr and thr not in self.report.time_to_tol:
                    self.report.time_to_tol[thr] = time.perf_counter() - t_start
            k_done = k
            if cfg.track_true_residual:
                tm.mark("recovery")
                x_k = self.assemble(y)
                if self.report.res_true is None:
                    self.report.res_true = []
                self.report.res_true.append(true_residual(self.a, self.b, x_k, cfg.zero_rel))
            tm.mark(None)
            tm.flush()
            hit = res <= nb_sketch * cfg.tol
            if hit:
                converged = True
            if (hit and not cfg.force_iterations) or lucky:
                if lucky:
                    converged = True
                break
        tm.mark("recovery")
        x = self.assemble(y)
        tm.mark(None)
        tm.flush()
        tm.resolve()
        _trim_timer_tail(self.report, k_done)
        self.report.converged = converged
        self.report.iterations = k_done
        self.report.wall_time = time.perf_counter() - t_start
        return x, self.report

    def assemble(self, y):
        """Combine the per-basis-vector sketch pairs with y and recover (solvers.py:450-465)."""
        pairs = [self.pairs[i] for i in range(len(y))]
        coeffs = [float(c) for c in y]
        if self.x0 is not None:
            pairs.append(self.x0_pair)
            coeffs.append(1.0)
        spec = RoundSpec(self.cfg.tol, default_solution_rank(self.b, self.cfg))
        u = stream_recover(combine_pairs(pairs, coeffs), spec, zero_rel=self.cfg.zero_rel)
        if self.precond is not None:  # x = P^{-1} u (solvers.py:462-463)
            u = self.precond.apply_inverse(u)
        return u


def _trim_timer_tail(report, k_done):
    """Fold the post-loop assemble row into the last iteration (solvers.py:278-285)."""
    for p in PHASES:
        lst = report.times[p]
        while len(lst) > k_done and len(lst) > 1:
            extra = lst.pop()
            lst[-1] += extra


def tt_sgmres(a: TTOperator, b: TTVector, x0, cfg: SolverConfig, sketch: KhatriRaoSketch,
              frame: StreamFrame | None = None):
    """Sketch-only-memory TT-sGMRES with a window of ell basis vectors (solvers.py:474-480)."""
    if frame is None:
        frame = make_solver_frame(b, cfg, seed=cfg.seed + 1)
    return _SketchedRun(a, b, x0, cfg, sketch, frame).run()


def tt_spgmres(a: TTOperator, precond, b: TTVector, x0, cfg: SolverConfig, sketch: KhatriRaoSketch,
               frame: StreamFrame | None = None):
    """Right-preconditioned TT-sGMRES (solvers.py:483-490): the Krylov space is
    built for A P^{-1} with P^{-1} an ExpSumPreconditioner (precond.py) applied
    on the device; the returned solution is x = P^{-1} u."""
    if frame is None:
        frame = make_solver_frame(b, cfg, seed=cfg.seed + 1)
    return _SketchedRun(a, b, x0, cfg, sketch, frame, precond=precond).run()
