"""Exponential-sum approximate inverse of a Kronecker sum (mirrors ttkrylov/precond.py).

1/z ~= sum_j alpha_j exp(-beta_j z) on the operator's spectral interval turns
(sum_i (+) A_i)^{-1} v into zeta rank-preserving mode multiplications
x_i exp(-beta_j A_i) (precond.py:203-278).  Split as in the reference:

* setup (once): the caller supplies the exp-sum coefficients alpha, beta
  (the reference derives them on the host, precond.py:70-159 -- out of scope);
  the zeta*d factor exponentials are formed once and uploaded as fp64 matrices;
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

# ---------------------------------------------------------------------------
# factor exponentials (setup, once per preconditioner)
#
# The exp-sum coefficients (alpha_j, beta_j) and the spectral interval are
# inputs: the reference computes them on the host once per operator
# (precond.py:70-159, an LP and a power iteration -- out of scope here, SURVEY
# section 2); a user passes the reference's own values, e.g.
# ExpSumPreconditioner(factors, *ttkrylov.precond.expsum_coeffs(lo, hi, zeta)[:2], spec).


def matrix_exp(m) -> np.ndarray:
    """exp(m) of a finite square fp64 matrix (the routine precond.py:20-27
    delegates to: SciPy's scaling-and-squaring Pade approximant)."""
    import scipy.linalg

    a = np.asarray(m, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ShapeMismatch(f"matrix_exp needs a square matrix, got {a.shape}")
    if not np.isfinite(a).all():
        raise ValueError("matrix_exp needs finite entries")
    return scipy.linalg.expm(a)


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
