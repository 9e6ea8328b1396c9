"""Exponential-sum approximate inverse of a Kronecker sum (mirrors ttkrylov/precond.py).

1/z ~= sum_j alpha_j exp(-beta_j z) on the operator's spectral interval turns
(sum_i (+) A_i)^{-1} v into zeta rank-preserving mode multiplications
x_i exp(-beta_j A_i) (precond.py:203-278).  Split as in the reference:

* construction (host, once): the spectral interval, the exp-sum nodes and
  minimax weights (a small LP), and the zeta*d factor exponentials -- then
  uploaded to the device as fp64 matrices;
* apply (device): all zeta terms in ONE grouped DMMA launch
  (``ttk_mode_multiply``, precond.py:189-200 + the alpha scaling :270-272),
  accumulated either by rounded TT additions (TT-SVD rounding on the device)
  or in sketch space (device stream sketch / combine / recover).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import ShapeMismatch
from .streaming import StreamFrame, combine_pairs, stream_recover, stream_sketch
from .tt import ZERO_REL, RoundSpec, TTVector, _check_cuda_vec, tt_add, tt_round

_REPORT_POINTS = 1000  # precond.py:17


# ---------------------------------------------------------------------------
# host-side construction


def matrix_exp(m) -> np.ndarray:
    """exp(m) for a finite square matrix (precond.py:20-27; SciPy's
    scaling-and-squaring Pade, the routine the reference calls)."""
    import scipy.linalg

    a = np.asarray(m, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ShapeMismatch(f"matrix_exp needs a square matrix, got {a.shape}")
    if not np.isfinite(a).all():
        raise ValueError("matrix_exp needs finite entries")
    return scipy.linalg.expm(a)


def _exp_basis(z, beta):
    """exp(-z_p beta_j) with the exponent clipped to [0, 700] (precond.py:30-33)."""
    with np.errstate(over="ignore", under="ignore"):
        return np.exp(-np.clip(np.multiply.outer(z, beta), 0.0, 700.0))


def _max_rel_error(z, alpha, beta) -> float:
    """max_p |z_p E(z_p) - 1| for E(z) = sum_j alpha_j exp(-beta_j z)."""
    return float(np.max(np.abs(z * (_exp_basis(z, beta) @ alpha) - 1.0)))


def _lp_weights(z, beta):
    """Nonnegative weights minimising max_p |z_p E(z_p) - 1| for fixed nodes:
    the LP  min t  s.t.  -t <= B w - 1 <= t,  w, t >= 0  over column-scaled
    basis B (precond.py:36-62).  Returns (None, inf) if HiGHS fails."""
    from scipy.optimize import linprog

    basis = z[:, None] * _exp_basis(z, beta)
    colmax = np.abs(basis).max(axis=0)
    colmax[colmax == 0] = 1.0
    bn = basis / colmax[None, :]
    npts, nn = bn.shape
    ones = np.ones((npts, 1))
    a_ub = np.concatenate([np.concatenate([bn, -ones], axis=1),
                           np.concatenate([-bn, -ones], axis=1)], axis=0)
    b_ub = np.concatenate([np.ones(npts), -np.ones(npts)])
    c = np.zeros(nn + 1)
    c[nn] = 1.0
    sol = linprog(c, A_ub=a_ub, b_ub=b_ub, bounds=[(0, None)] * (nn + 1), method="highs")
    if sol.status != 0:
        return None, np.inf
    return sol.x[:nn] / colmax, float(sol.x[nn])


class _NodeSearch:
    """The exp-sum node window search of expsum_coeffs (precond.py:70-135):
    geometric nodes between e^u/hi and e^v/lo, weights from the LP (trapezoid
    weights h*beta if the LP fails), a 6x6 grid over (u, v) followed by a
    compass search with halving steps."""

    def __init__(self, lo, hi, zeta):
        self.lo, self.hi, self.zeta = lo, hi, zeta
        self.z = np.logspace(np.log10(lo), np.log10(hi), max(1200, 20 * zeta))

    def nodes(self, u, v):
        b0, b1 = np.exp(u) / self.hi, np.exp(v) / self.lo
        if not b1 > b0:
            return None
        if self.zeta == 1:
            return np.array([np.sqrt(b0 * b1)])
        return np.geomspace(b0, b1, self.zeta)

    def evaluate(self, u, v):
        beta = self.nodes(u, v)
        if beta is None:
            return np.inf, None, None
        alpha, err = _lp_weights(self.z, beta)
        if alpha is None:
            h = (v - u + np.log(self.hi / self.lo)) / max(self.zeta - 1, 1)
            alpha = h * beta
            err = _max_rel_error(self.z, alpha, beta)
        return err, alpha, beta

    def run(self):
        best_err, best_a, best_b, at = np.inf, None, None, (0.0, 0.0)
        for u in np.linspace(-1.5, 2.0, 6):
            for v in np.linspace(-1.0, 2.5, 6):
                err, a, b = self.evaluate(u, v)
                if err < best_err:
                    best_err, best_a, best_b, at = err, a, b, (u, v)
        u, v = at
        step = 0.4
        while step > 0.02:
            for du, dv in ((1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (-1, -1)):
                cu, cv = u + du * step, v + dv * step
                err, a, b = self.evaluate(cu, cv)
                if err < best_err:
                    best_err, best_a, best_b = err, a, b
                    u, v = cu, cv
                    break
            else:
                step /= 2.0
        return best_a, best_b


def expsum_coeffs(lambda_min: float, lambda_max: float, zeta: int):
    """(alpha, beta, bound) of an exp-sum for 1/z on [lambda_min, lambda_max]
    (precond.py:70-135); bound = max |z E(z) - 1| over 1000 log-spaced z."""
    if lambda_min <= 0:
        raise ValueError("lambda_min must be positive")
    if lambda_max < lambda_min:
        raise ValueError("lambda_max must be >= lambda_min")
    if zeta < 1:
        raise ValueError("zeta must be >= 1")
    lo, hi = float(lambda_min), float(lambda_max)
    if hi / lo < 1.0 + 1e-9:  # degenerate interval: widen by 1e-9 relative
        lo, hi = lo * (1.0 - 1e-9), hi * (1.0 + 1e-9)
    alpha, beta = _NodeSearch(lo, hi, zeta).run()
    zr = np.logspace(np.log10(lo), np.log10(hi), _REPORT_POINTS)
    return alpha, beta, _max_rel_error(zr, alpha, beta)


def _lowest_eig_lower_bound(sym, shift) -> float:
    """Lower estimate of the smallest eigenvalue of a symmetric matrix: power
    iteration on shift*I - sym, Rayleigh quotient minus residual norm
    (precond.py:162-186)."""
    n = sym.shape[0]
    if n == 1:
        return float(sym[0, 0])
    x = np.ones(n) + 1e-3 * np.cos(np.arange(n))
    x /= np.linalg.norm(x)
    prev = np.inf
    for it in range(20 * n + 200):
        y = shift * x - sym @ x
        ny = np.linalg.norm(y)
        if ny == 0:
            return float(shift)
        x = y / ny
        if it % 8 == 0:
            rq = float(x @ (sym @ x))
            if abs(rq - prev) <= 1e-12 * max(abs(shift), 1.0):
                break
            prev = rq
    rq = float(x @ (sym @ x))
    return max(rq - float(np.linalg.norm(sym @ x - rq * x)), 0.0)


def spectral_interval(factors):
    """[lambda_min, lambda_max] of the symmetric part of sum_i (+) A_i:
    Gershgorin upper bounds and power-iteration lower estimates summed over
    factors, lambda_min floored at 1e-8 lambda_max (precond.py:138-159)."""
    lo = hi = 0.0
    for i, f in enumerate(factors):
        a = np.asarray(f, dtype=np.float64)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ShapeMismatch(f"factor {i} is not square")
        sym = 0.5 * (a + a.T)
        diag = np.diag(sym)
        radius = np.abs(sym).sum(axis=1) - np.abs(diag)  # Gershgorin radii
        top = float(np.max(diag + radius))
        hi += top
        lo += _lowest_eig_lower_bound(sym, top)
    return max(lo, 1e-8 * hi), hi


# ---------------------------------------------------------------------------
# device apply


def _mode_multiply_many(v: TTVector, mat_lists, alphas=None):
    """One ttk_mode_multiply launch for several matrix lists (device fp64
    tensors) applied to the same TT; returns one TTVector per list."""
    _check_cuda_vec(v)
    lib = _lib.load()
    d, dev = v.d, v.device
    nt = len(mat_lists)
    r = list(v.ranks)
    n = list(v.dims)
    m = [int(mk.shape[0]) for mk in mat_lists[0]]
    outs = [[torch.empty((r[k], m[k], r[k + 1]), dtype=torch.float64, device=dev) for k in range(d)]
            for _ in range(nt)]
    mats = [mk for ml in mat_lists for mk in ml]
    _lib.check(lib.ttk_mode_multiply(
        nt, d, _lib.int_array(n), _lib.int_array(m), _lib.int_array(r),
        _lib.double_array(alphas) if alphas is not None else None,
        _lib.ptr_array(mats), _lib.ptr_array(v.cores), _lib.ptr_array([c for o in outs for c in o]),
        _lib.stream_ptr(dev)))
    return [TTVector(o) for o in outs]


def _device_mats(matrices, v: TTVector):
    if len(matrices) != v.d:
        raise ShapeMismatch("need one matrix per mode")
    out = []
    for mk, c in zip(matrices, v.cores):
        t = torch.as_tensor(np.asarray(mk, dtype=np.float64) if not torch.is_tensor(mk) else mk)
        t = t.to(device=v.device, dtype=torch.float64).contiguous()
        if t.ndim != 2 or t.shape[1] != c.shape[1]:
            raise ShapeMismatch("matrix columns must match mode size")
        out.append(t)
    return out


def mode_multiply(v: TTVector, matrices) -> TTVector:
    """Multiply mode k of the tensor by matrices[k]; ranks unchanged (precond.py:189-200)."""
    return _mode_multiply_many(v, [_device_mats(matrices, v)])[0]


class ExpSumPreconditioner:
    """Approximate inverse of a Kronecker sum via exponential sums (precond.py:203-278).

    ``zero_rel``: the rounding zero test of the accumulation roundings (the
    reference's tt_round rule by default; None bypasses it, quirk Q1)."""

    def __init__(self, factors, alpha, beta, spec: RoundSpec, accumulate: str = "sequential",
                 quad_bound: float | None = None, stream_seed: int = 0,
                 zero_rel: float | None = ZERO_REL):
        self.factors = [np.asarray(f, dtype=np.float64) for f in factors]
        self.alpha = np.asarray(alpha, dtype=np.float64)
        self.beta = np.asarray(beta, dtype=np.float64)
        if self.alpha.ndim != 1 or self.alpha.shape != self.beta.shape:
            raise ValueError("alpha and beta must be equal-length vectors")
        if np.any(self.beta < 0):
            raise ValueError("beta coefficients must be nonnegative")
        if accumulate not in ("sequential", "stream"):
            raise ValueError("accumulate must be 'sequential' or 'stream'")
        self.spec = spec
        self.accumulate = accumulate
        self.quad_bound = quad_bound
        self.stream_seed = stream_seed
        self.zero_rel = zero_rel
        # cached factor exponentials exp(-beta_j A_i), host copies + device copies
        self.exps = [[matrix_exp(-bj * f) for f in self.factors] for bj in self.beta]
        self._dev_exps = None  # (device, zeta x d device matrices), uploaded on first apply

    @property
    def zeta(self) -> int:
        return len(self.beta)

    @property
    def dims(self) -> tuple:
        return tuple(f.shape[0] for f in self.factors)

    @classmethod
    def from_kron_sum(cls, factors, zeta: int, spec: RoundSpec, accumulate: str = "sequential",
                      interval=None, stream_seed: int = 0,
                      zero_rel: float | None = ZERO_REL) -> "ExpSumPreconditioner":
        """Coefficients for the spectral interval of sum_i (+) A_i (precond.py:235-244)."""
        if interval is None:
            interval = spectral_interval(factors)
        alpha, beta, bound = expsum_coeffs(interval[0], interval[1], zeta)
        return cls(factors, alpha, beta, spec, accumulate=accumulate, quad_bound=bound,
                   stream_seed=stream_seed, zero_rel=zero_rel)

    def _device_exps(self, device):
        if self._dev_exps is None or self._dev_exps[0] != device:
            mats = [[torch.as_tensor(e).to(device=device, dtype=torch.float64).contiguous() for e in row]
                    for row in self.exps]
            self._dev_exps = (device, mats)
        return self._dev_exps[1]

    def terms(self, v: TTVector):
        """alpha_j * (x_i exp(-beta_j A_i)) v for every j, one grouped launch (precond.py:246-254)."""
        if v.dims != self.dims:
            raise ShapeMismatch(f"vector dims {v.dims} do not match {self.dims}")
        return _mode_multiply_many(v, self._device_exps(v.device), [float(a) for a in self.alpha])

    def apply_inverse(self, v: TTVector) -> TTVector:
        """Approximate (sum_i (+) A_i)^{-1} v (precond.py:256-278)."""
        terms = self.terms(v)
        if self.accumulate == "sequential":
            acc = terms[0]
            inner = RoundSpec(self.spec.rel_tol, None)
            for t in terms[1:]:
                acc = tt_round(tt_add(acc, t), inner, zero_rel=self.zero_rel)
            return tt_round(acc, self.spec, zero_rel=self.zero_rel)
        cap = self.spec.max_rank
        target = cap if cap is not None else 2 * max(max(t.ranks) for t in terms)
        frame = StreamFrame.create(self.dims, [target] * (v.d - 1), seed=self.stream_seed, device=v.device)
        comb = combine_pairs([stream_sketch(t, frame) for t in terms], [1.0] * len(terms))
        return stream_recover(comb, self.spec, zero_rel=self.zero_rel)


def precond_apply(p: ExpSumPreconditioner, v: TTVector) -> TTVector:
    """Apply the exponential-sum approximate inverse to a TT vector (precond.py:281-283)."""
    return p.apply_inverse(v)
