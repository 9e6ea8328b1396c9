"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (needs /root/reference):
    python tests/golden/make_golden.py
Writes small .npz fixtures next to this script.  The GPU box never runs this
script; tests load the committed fixtures.  Shapes and seeds follow the
reference's own tests (pkg/tests/test_tt.py, test_sketch.py,
test_streaming.py, test_solvers.py) plus one BASELINE-size solver history
(config 1, with the reference's tt_round zero test bypassed -- quirk Q1).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import ttkrylov  # noqa: E402
import ttkrylov.solvers as rsolvers  # noqa: E402
import ttkrylov.streaming as rstreaming  # noqa: E402
from ttkrylov import tt as rtt  # noqa: E402
from ttkrylov.problems import ConvectionDiffusionSpec, convection_diffusion  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cores_dict(prefix, cores, out):
    out[f"{prefix}__d"] = np.array(len(cores))
    for k, c in enumerate(cores):
        out[f"{prefix}__{k}"] = np.ascontiguousarray(c)


def random_operator(row_dims, col_dims, ranks, seed):
    # same construction as pkg/tests/test_tt.py:48-55
    rng = np.random.default_rng(seed)
    full = [1] + list(ranks) + [1]
    return [rng.standard_normal((full[k], row_dims[k], col_dims[k], full[k + 1]))
            for k in range(len(row_dims))]


def gen_tt_ops():
    out = {}
    # matvec (test_tt.py:193-220)
    cases = [
        ("mv_identity", [np.eye(n).reshape(1, n, n, 1) for n in (3, 4, 5)],
         ttkrylov.tt_random([3, 4, 5], [2, 3], seed=11)),
        ("mv_rankprod", random_operator([3, 3, 3], [3, 3, 3], [2, 2], 12),
         ttkrylov.tt_random([3, 3, 3], [3, 3], seed=13)),
        ("mv_dense", random_operator([4, 4, 4], [4, 4, 4], [2, 3], 14),
         ttkrylov.tt_random([4, 4, 4], [2, 2], seed=15)),
        ("mv_rect", random_operator([2, 3], [4, 5], [2], 16),
         ttkrylov.tt_random([4, 5], [3], seed=17)),
        ("mv_mixed", random_operator([5, 3, 6, 2], [4, 7, 3, 5], [3, 1, 2], 18),
         ttkrylov.tt_random([4, 7, 3, 5], [4, 5, 2], seed=19)),
    ]
    names = []
    for name, op, v in cases:
        res = ttkrylov.tt_matvec(ttkrylov.TTOperator(op), v)
        cores_dict(name + "_op", op, out)
        cores_dict(name + "_x", v.cores, out)
        cores_dict(name + "_y", res.cores, out)
        names.append(name)
    out["mv_names"] = np.array(names)

    # add / scale (test_tt.py:112-160)
    a = ttkrylov.tt_random([3, 3, 3], [2, 3], seed=0)
    b = ttkrylov.tt_random([3, 3, 3], [1, 2], seed=1)
    cores_dict("add_a", a.cores, out)
    cores_dict("add_b", b.cores, out)
    cores_dict("add_y", ttkrylov.tt_add(a, b).cores, out)
    a1 = ttkrylov.TTVector([np.array([[[1.0], [2.0]]])])
    b1 = ttkrylov.TTVector([np.array([[[5.0], [7.0]]])])
    cores_dict("add1_a", a1.cores, out)
    cores_dict("add1_b", b1.cores, out)
    cores_dict("add1_y", ttkrylov.tt_add(a1, b1).cores, out)
    s = ttkrylov.tt_random([3, 4, 3], [2, 2], seed=6)
    cores_dict("scale_a", s.cores, out)
    cores_dict("scale_y", ttkrylov.tt_scale(s, -2.5).cores, out)
    # a multi-term explicit Arnoldi update: vt - h1 v1 - h2 v2 (solvers.py:361-366)
    vt = ttkrylov.tt_random([4, 5, 3, 4], [3, 4, 2], seed=40)
    v1 = ttkrylov.tt_random([4, 5, 3, 4], [2, 2, 2], seed=41)
    v2 = ttkrylov.tt_random([4, 5, 3, 4], [1, 3, 2], seed=42)
    acc = vt
    hs = [0.37, -1.25]
    for h, vi in zip(hs, (v1, v2)):
        acc = ttkrylov.tt_add(acc, ttkrylov.tt_scale(vi, -h))
    for nm, v in (("axpy_vt", vt), ("axpy_v1", v1), ("axpy_v2", v2), ("axpy_y", acc)):
        cores_dict(nm, v.cores, out)
    out["axpy_h"] = np.array(hs)

    # dot / norm (test_tt.py:163-190)
    da = ttkrylov.tt_random([5, 5, 5], [3, 3], seed=8)
    db = ttkrylov.tt_random([5, 5, 5], [2, 4], seed=9)
    cores_dict("dot_a", da.cores, out)
    cores_dict("dot_b", db.cores, out)
    out["dot_ab"] = np.array(ttkrylov.tt_dot(da, db))
    nn = ttkrylov.tt_random([4, 6, 3], [2, 5], seed=10)
    cores_dict("norm_a", nn.cores, out)
    out["norm_a_val"] = np.array(ttkrylov.tt_norm(nn))

    # rounding (test_tt.py:228-275), reference tt_round as-is
    rcases = []
    a = ttkrylov.tt_random([4, 4, 4], [2, 2], seed=18)
    rcases.append(("rd_minimal", a, 1e-14, None))
    a = ttkrylov.tt_random([4, 4, 4], [2, 2], seed=19)
    rcases.append(("rd_doubled", ttkrylov.tt_add(a, a), 1e-12, None))
    for tol in (1e-2, 1e-6, 1e-10):
        for seed in (0, 3, 7):
            rcases.append((f"rd_contract_{tol:g}_{seed}",
                           ttkrylov.tt_random([5, 6, 4, 5], [4, 6, 4], seed=seed), tol, None))
    rcases.append(("rd_cap", ttkrylov.tt_random([6, 6, 6], [5, 5], seed=21), 0.0, 2))
    a = ttkrylov.tt_random([3, 4, 3], [2, 2], seed=2)
    rcases.append(("rd_cancel", ttkrylov.tt_add(a, ttkrylov.tt_scale(a, -1.0)), 1e-12, None))
    a = ttkrylov.tt_add(ttkrylov.tt_random([4, 5, 4], [3, 3], seed=22),
                        ttkrylov.tt_random([4, 5, 4], [2, 2], seed=23))
    rcases.append(("rd_idem", a, 1e-3, None))
    names = []
    for name, v, tol, cap in rcases:
        r = ttkrylov.tt_round(v, ttkrylov.RoundSpec(tol, cap))
        cores_dict(name + "_x", v.cores, out)
        out[name + "_dense"] = ttkrylov.tt_to_dense(r)
        out[name + "_ranks"] = np.array(r.ranks)
        out[name + "_spec"] = np.array([tol, -1 if cap is None else cap])
        names.append(name)
    out["rd_names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "tt_ops.npz"), **out)


def gen_sketch():
    out = {}
    cases = [
        ("kr_d1", ttkrylov.kr_sketch_new([6], 4, seed=7), ttkrylov.tt_random([6], [], seed=8)),
        ("kr_dense", ttkrylov.kr_sketch_new([3, 4, 4], 7, seed=9),
         ttkrylov.tt_random([3, 4, 4], [3, 2], seed=10)),
        ("kr_lin", ttkrylov.kr_sketch_new([3, 3, 3], 9, seed=11),
         ttkrylov.tt_random([3, 3, 3], [2, 2], seed=12)),
        ("kr_chunk", ttkrylov.kr_sketch_new([3, 4], 50, seed=18),
         ttkrylov.tt_random([3, 4], [3], seed=19)),
        ("kr_wide", ttkrylov.kr_sketch_new([5, 8, 6, 7, 4], 33, seed=20),
         ttkrylov.tt_random([5, 8, 6, 7, 4], [5, 17, 9, 3], seed=21)),
    ]
    names = []
    for name, s, v in cases:
        y = ttkrylov.kr_apply(s, v)
        for k, f in enumerate(s.factors):
            out[f"{name}_F__{k}"] = f
        cores_dict(name + "_x", v.cores, out)
        out[name + "_y"] = y
        names.append(name)
    out["kr_names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "sketch.npz"), **out)


def gen_streaming():
    out = {}
    frame = rstreaming.StreamFrame.create([3, 4, 3], [2, 2], oversampling=3, seed=6)
    t = ttkrylov.tt_random([3, 4, 3], [2, 3], seed=7)
    pair = rstreaming.stream_sketch(t, frame)
    cores_dict("ss_left", frame.left.cores, out)
    cores_dict("ss_right", frame.right.cores, out)
    cores_dict("ss_x", t.cores, out)
    for k, p in enumerate(pair.psi):
        out[f"ss_psi__{k}"] = p
    for k, o in enumerate(pair.omega):
        out[f"ss_omega__{k}"] = o
    # 5-term combination + recovery (test_streaming.py:85-98)
    dims = [4, 4, 4, 4]
    frame = rstreaming.StreamFrame.create(dims, [4, 10, 4], oversampling=8, seed=22)
    vs = [ttkrylov.tt_random(dims, [2, 2, 2], seed=200 + i) for i in range(5)]
    ys = np.array([0.3, -1.1, 2.0, 0.7, -0.4])
    comb = rstreaming.combine_pairs([rstreaming.stream_sketch(v, frame) for v in vs], ys)
    got = rstreaming.stream_recover(comb, ttkrylov.RoundSpec(1e-12))
    cores_dict("rc_left", frame.left.cores, out)
    cores_dict("rc_right", frame.right.cores, out)
    for i, v in enumerate(vs):
        cores_dict(f"rc_v{i}", v.cores, out)
    out["rc_y"] = ys
    out["rc_dense"] = ttkrylov.tt_to_dense(got)
    out["rc_ranks"] = np.array(got.ranks)
    np.savez_compressed(os.path.join(HERE, "streaming.npz"), **out)


def nozero_round(v, spec):
    """Reference tt_round minus its zero test (tt.py:350-356), built from the
    reference's own _right_orthogonalize/_truncation_rank (quirk Q1 bypass)."""
    d = v.d
    if d == 1:
        return v.copy()
    cores = rtt._right_orthogonalize([c.copy() for c in v.cores])
    nrm = np.linalg.norm(cores[0])
    if nrm == 0:
        return rtt.tt_zero(v.dims)
    budget = spec.rel_tol * nrm / np.sqrt(d - 1)
    for k in range(d - 1):
        c = cores[k]
        r0, n, r1 = c.shape
        u, sv, vt = np.linalg.svd(c.reshape(r0 * n, r1), full_matrices=False)
        r = rtt._truncation_rank(sv, budget)
        if spec.max_rank is not None:
            r = min(r, spec.max_rank)
        cores[k] = u[:, :r].reshape(r0, n, r)
        cores[k + 1] = np.tensordot(sv[:r, None] * vt[:r], cores[k + 1], axes=([1], [0]))
    return ttkrylov.TTVector(cores)


def probe_sketch(x, nprobe=24, seed=777):
    s = ttkrylov.kr_sketch_new(list(x.dims), nprobe, seed=seed)
    return ttkrylov.kr_apply(s, x)


def solver_case(name, op, b, cfg, sketch, out, frame=None):
    x, rep = rsolvers.tt_sgmres(op, b, None, cfg, sketch, frame)
    cores_dict(name + "_op", op.op_cores, out)
    cores_dict(name + "_b", b.cores, out)
    for k, f in enumerate(sketch.factors):
        out[f"{name}_F__{k}"] = f
    out[name + "_res"] = np.array(rep.res_sketched)
    out[name + "_ranks"] = np.array(rep.basis_rank)
    out[name + "_iters"] = np.array(rep.iterations)
    out[name + "_conv"] = np.array(rep.converged)
    out[name + "_xprobe"] = probe_sketch(x)
    out[name + "_xnorm"] = np.array(ttkrylov.tt_norm(x))
    out[name + "_cfg"] = np.array([cfg.maxit, cfg.tol, cfg.ell, cfg.eta,
                                   -1 if cfg.max_rank is None else cfg.max_rank,
                                   cfg.sketch_rows, cfg.oversampling,
                                   -1 if cfg.solution_rank is None else cfg.solution_rank,
                                   cfg.seed, 1 if cfg.combine_mode == "stta" else 0])
    if frame is not None:
        cores_dict(name + "_left", frame.left.cores, out)
        cores_dict(name + "_right", frame.right.cores, out)
    return x, rep


def gen_solver_small():
    out = {}
    op, rhs = convection_diffusion(ConvectionDiffusionSpec(d=3, n=5))
    cfg = rsolvers.SolverConfig(maxit=100, tol=1e-8, ell=1, eta=0.3, seed=6, solution_rank=10)
    s = ttkrylov.kr_sketch_new(rhs.dims, cfg.sketch_rows, seed=7)
    solver_case("sv_pde", op, rhs, cfg, s, out)
    cfg = rsolvers.SolverConfig(maxit=60, tol=1e-8, ell=2, eta=0.3, seed=3, solution_rank=10)
    s = ttkrylov.kr_sketch_new(rhs.dims, cfg.sketch_rows, seed=4)
    solver_case("sv_ell2", op, rhs, cfg, s, out)
    cfg = rsolvers.SolverConfig(maxit=100, tol=1e-7, ell=2, seed=14, combine_mode="stta",
                                solution_rank=10)
    s = ttkrylov.kr_sketch_new(rhs.dims, cfg.sketch_rows, seed=15)
    solver_case("sv_stta", op, rhs, cfg, s, out)
    out["sv_names"] = np.array(["sv_pde", "sv_ell2", "sv_stta"])
    np.savez_compressed(os.path.join(HERE, "solver_small.npz"), **out)


def gen_solver_cfg1():
    """BASELINE config 1 with the Q1 zero test bypassed."""
    out = {}
    n, d = 32, 8
    lap = (n + 1) ** 2 * (2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1))
    op = ttkrylov.kron_sum_operator([lap] * d)
    rng = np.random.default_rng(0)
    b = ttkrylov.tt_rank_one([rng.standard_normal(n) for _ in range(d)])
    b = ttkrylov.tt_scale(b, 1.0 / ttkrylov.tt_norm(b))
    cfg = rsolvers.SolverConfig(maxit=40, tol=1e-8, ell=2, eta=1.0, max_rank=30,
                                sketch_rows=80, seed=0)
    s = ttkrylov.kr_sketch_new(b.dims, 80, seed=0)
    # StreamFrame.create overflows nowhere at d=8, n=32 (8*5 bits), so it is usable here
    frame = rsolvers.make_solver_frame(b, cfg, seed=1)
    saved = (rsolvers.tt_round, rstreaming.tt_round)
    rsolvers.tt_round = nozero_round
    rstreaming.tt_round = nozero_round
    try:
        t0 = time.perf_counter()
        solver_case("cfg1", op, b, cfg, s, out, frame=frame)
        # the frame is regenerated from its seed (SeedSequence(1).spawn(2)) by the tests
        for key in [k for k in out if k.startswith("cfg1_left") or k.startswith("cfg1_right")]:
            del out[key]
        out["cfg1_wall"] = np.array(time.perf_counter() - t0)
    finally:
        rsolvers.tt_round, rstreaming.tt_round = saved
    np.savez_compressed(os.path.join(HERE, "solver_cfg1.npz"), **out)


def gen_serial():
    """TT containers written by the reference's save_vector / save_operator
    (tt.py:451-520) on the shapes of its own round-trip tests
    (test_tt.py:363-380), plus the cores for a bit-exact comparison."""
    out = {}
    v = rtt.tt_random([3, 5, 2], [2, 3], seed=30)
    a = ttkrylov.TTOperator(random_operator([3, 4], [2, 5], [3], seed=31))
    rtt.save_vector(os.path.join(HERE, "serial_vec.ttk"), v)
    rtt.save_operator(os.path.join(HERE, "serial_op.ttk"), a)
    cores_dict("vec", v.cores, out)
    cores_dict("op", a.op_cores, out)
    np.savez_compressed(os.path.join(HERE, "serial.npz"), **out)


def _lap(n):
    # pkg/tests/test_precond.py:39-41 (positive definite orientation)
    return -(-2.0 * np.eye(n) + np.diag(np.ones(n - 1), 1) + np.diag(np.ones(n - 1), -1))


def _spgmres_case(name, op, b, p, cfg, sketch, out, frame=None):
    x, rep = rsolvers.tt_spgmres(op, p, b, None, cfg, sketch, frame)
    cores_dict(name + "_op", op.op_cores, out)
    cores_dict(name + "_b", b.cores, out)
    for k, f in enumerate(sketch.factors):
        out[f"{name}_F__{k}"] = f
    out[name + "_alpha"] = p.alpha
    out[name + "_beta"] = p.beta
    out[name + "_spec"] = np.array([p.spec.rel_tol, -1 if p.spec.max_rank is None else p.spec.max_rank])
    out[name + "_res"] = np.array(rep.res_sketched)
    out[name + "_ranks"] = np.array(rep.basis_rank)
    out[name + "_iters"] = np.array(rep.iterations)
    out[name + "_conv"] = np.array(rep.converged)
    out[name + "_x"] = rtt.tt_to_dense(x)
    out[name + "_true_res"] = np.array(rsolvers.true_residual(op, b, x))
    out[name + "_cfg"] = np.array([cfg.maxit, cfg.tol, cfg.ell, cfg.eta,
                                   -1 if cfg.max_rank is None else cfg.max_rank,
                                   cfg.sketch_rows, cfg.oversampling,
                                   -1 if cfg.solution_rank is None else cfg.solution_rank, cfg.seed])
    if frame is not None:
        cores_dict(name + "_left", frame.left.cores, out)
        cores_dict(name + "_right", frame.right.cores, out)


def gen_precond():
    """Exp-sum preconditioner (precond.py) on the cases of pkg/tests/test_precond.py
    and the preconditioned solver cases of test_solvers.py:255-285."""
    from ttkrylov import precond as rp
    from ttkrylov.problems import cd_factor_matrices
    out = {}
    # exp-sum coefficients (test_precond.py:83-112 intervals)
    cases = [(0.5, 60.0, 12), (0.2, 30.0, 9), (3.0, 3.0, 1), (0.1, 10.0, 2)]
    out["coef_cases"] = np.array(cases)
    for i, c in enumerate(cases):
        a, b, bound = rp.expsum_coeffs(*c)
        out[f"coef{i}_alpha"], out[f"coef{i}_beta"], out[f"coef{i}_bound"] = a, b, np.array(bound)
    # spectral intervals (test_precond.py:115-133) + a nonsymmetric set
    rng = np.random.default_rng(42)
    sets = [[np.eye(4)] * 3, [np.diag([1.0, 2.0, 3.0])], [_lap(8)] * 3,
            [rng.standard_normal((6, 6)) + 6 * np.eye(6) for _ in range(3)]]
    for i, fs in enumerate(sets):
        out[f"int{i}_n"] = np.array(len(fs))
        for k, f in enumerate(fs):
            out[f"int{i}_f{k}"] = f
        out[f"int{i}_val"] = np.array(rp.spectral_interval(fs))
    out["int_count"] = np.array(len(sets))
    # mode_multiply with rectangular matrices (mode sizes change)
    v = rtt.tt_random([3, 4, 5], [2, 3], seed=40)
    mats = [rng.standard_normal((5, 3)), rng.standard_normal((4, 4)), rng.standard_normal((2, 5))]
    w = rp.mode_multiply(v, mats)
    cores_dict("mm_in", v.cores, out)
    cores_dict("mm_out", w.cores, out)
    for k, m in enumerate(mats):
        out[f"mm_mat{k}"] = m
    # approximate inverse, sequential accumulation (test_precond.py:145-156)
    factors = [_lap(6) for _ in range(3)]
    p = rp.ExpSumPreconditioner.from_kron_sum(factors, 24, rtt.RoundSpec(1e-12))
    x = rtt.tt_random([6, 6, 6], [2, 2], seed=5)
    x = rtt.tt_scale(x, 1.0 / rtt.tt_norm(x))
    qx = rtt.tt_matvec(ttkrylov.kron_sum_operator(factors), x)
    got = rp.precond_apply(p, qx)
    cores_dict("inv_x", x.cores, out)
    cores_dict("inv_qx", qx.cores, out)
    out["inv_alpha"], out["inv_beta"], out["inv_bound"] = p.alpha, p.beta, np.array(p.quad_bound)
    out["inv_out"] = rtt.tt_to_dense(got)
    out["inv_ranks"] = np.array(got.ranks)
    # sequential vs stream accumulation (test_precond.py:182-191)
    factors = [_lap(5) for _ in range(3)]
    spec = rtt.RoundSpec(1e-10, max_rank=12)
    seq = rp.ExpSumPreconditioner.from_kron_sum(factors, 10, spec, accumulate="sequential")
    st = rp.ExpSumPreconditioner(factors, seq.alpha, seq.beta, spec, accumulate="stream")
    v = rtt.tt_random([5, 5, 5], [2, 2], seed=10)
    cores_dict("acc_v", v.cores, out)
    out["acc_alpha"], out["acc_beta"] = seq.alpha, seq.beta
    out["acc_seq"] = rtt.tt_to_dense(rp.precond_apply(seq, v))
    out["acc_stream"] = rtt.tt_to_dense(rp.precond_apply(st, v))
    # preconditioned solver: identity preconditioner (test_solvers.py:256-266)
    op, rhs = convection_diffusion(ConvectionDiffusionSpec(d=3, n=5))
    pid = rp.ExpSumPreconditioner([np.zeros((5, 5))] * 3, [1.0], [0.0], rtt.RoundSpec(1e-14))
    cfg = rsolvers.SolverConfig(maxit=60, tol=1e-6, ell=1, seed=31, solution_rank=10)
    s = ttkrylov.kr_sketch_new(rhs.dims, cfg.sketch_rows, seed=32)
    frame = rstreaming.StreamFrame.create(rhs.dims, [10, 10], seed=33)
    _spgmres_case("sp_id", op, rhs, pid, cfg, s, out, frame=frame)
    x_u, rep_u = rsolvers.tt_sgmres(op, rhs, None, cfg, s, frame)
    out["sp_id_plain_res"] = np.array(rep_u.res_sketched)
    # exp-sum preconditioned convection-diffusion (test_solvers.py:268-285)
    spec = ConvectionDiffusionSpec(d=3, n=16)
    op, rhs = convection_diffusion(spec)
    fac = cd_factor_matrices(spec)
    p = rp.ExpSumPreconditioner.from_kron_sum(fac, 17, rtt.RoundSpec(1e-9, max_rank=30))
    cfg = rsolvers.SolverConfig(maxit=20, tol=1e-9, ell=1, eta=0.1, seed=34, max_rank=30, solution_rank=15)
    s = ttkrylov.kr_sketch_new(rhs.dims, cfg.sketch_rows, seed=35)
    for k, f in enumerate(fac):
        out[f"sp_pde_fac{k}"] = f
    _spgmres_case("sp_pde", op, rhs, p, cfg, s, out)
    np.savez_compressed(os.path.join(HERE, "precond.npz"), **out)


def _cfg5_problem(j):
    """BASELINE config 5: c_k = rng(0).uniform(0.1, 1, 50), A =
    kron_sum_operator([c_k L]) with L = (n+1)^2 tridiag(-1, 2, -1), n = 256;
    RHS j = rank-1 TT of 50 rng(j) Gaussian vectors scaled to ||b|| = 1."""
    n, d = 256, 50
    c = np.random.default_rng(0).uniform(0.1, 1.0, d)
    lap = (n + 1) ** 2 * (2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1))
    op = ttkrylov.kron_sum_operator([ck * lap for ck in c])
    rng = np.random.default_rng(j)
    b = ttkrylov.tt_rank_one([rng.standard_normal(n) for _ in range(d)])
    b = ttkrylov.tt_scale(b, 1.0 / ttkrylov.tt_norm(b))
    cfg = rsolvers.SolverConfig(maxit=60, tol=1e-8, ell=3, eta=1.0, max_rank=100, sketch_rows=120, seed=j)
    s = ttkrylov.kr_sketch_new(b.dims, 120, seed=j)
    # StreamFrame.create overflows its cumprod clipping at d=50, n=256 (quirk Q2):
    # build the frame exactly as make_solver_frame + StreamFrame.create would
    # (solution rank max(2*1, 20) = 20 -> recovery ranks 40, left ranks 60,
    # seeds SeedSequence(j+1).spawn(2)), without the overflowing clip.
    s_right, s_left = np.random.SeedSequence(j + 1).spawn(2)
    frame = rstreaming.StreamFrame(right=rstreaming.tt_drm_new(b.dims, [40] * (d - 1), seed=s_right),
                                   left=rstreaming.tt_drm_new(b.dims, [60] * (d - 1), seed=s_left))
    return c, op, b, cfg, s, frame


def gen_solver_cfg5(rhs=(0, 1)):
    """BASELINE config 5 (d=50, n=256, ell=3, s=120, maxit 60, cap 100) solved
    by the reference tt_sgmres with the Q1 zero test bypassed, one RHS at a
    time (~60 s each on 8 cores).  Stored: iteration count, rank and residual
    histories, a 24-row Khatri-Rao probe of x and ||x||, per-iteration phase
    times and the wall time; the inputs are regenerated from their seeds by
    the tests (configs.config5), checked against the stored c_k and b."""
    out = {}
    saved = (rsolvers.tt_round, rstreaming.tt_round)
    rsolvers.tt_round = nozero_round
    rstreaming.tt_round = nozero_round
    try:
        for j in rhs:
            c, op, b, cfg, s, frame = _cfg5_problem(j)
            name = f"cfg5_{j}"
            t0 = time.perf_counter()
            x, rep = rsolvers.tt_sgmres(op, b, None, cfg, s, frame)
            wall = time.perf_counter() - t0
            out[name + "_c"] = c
            cores_dict(name + "_b", b.cores, out)
            out[name + "_res"] = np.array(rep.res_sketched)
            out[name + "_ranks"] = np.array(rep.basis_rank)
            out[name + "_iters"] = np.array(rep.iterations)
            out[name + "_conv"] = np.array(rep.converged)
            out[name + "_xprobe"] = probe_sketch(x)
            out[name + "_xnorm"] = np.array(ttkrylov.tt_norm(x))
            out[name + "_xranks"] = np.array(x.ranks)
            out[name + "_wall"] = np.array(wall)
            out[name + "_iter_s"] = np.array([sum(rep.times[p][i] for p in rep.times)
                                              for i in range(len(rep.times["round"]))])
            out[name + "_sketch0"] = s.factors[0][:4].copy()
            print(f"{name}: {rep.iterations} it, res {rep.res_sketched[-1]:.3e}, wall {wall:.1f} s",
                  flush=True)
    finally:
        rsolvers.tt_round, rstreaming.tt_round = saved
    out["cfg5_rhs"] = np.array(list(rhs))
    np.savez_compressed(os.path.join(HERE, "solver_cfg5.npz"), **out)


def gen_kr_cfg4(which=(0, 1, 63)):
    """BASELINE config 4: reference kr_apply with KhatriRaoSketch(F) (quirk Q4:
    F_k ~ N(0, 1/n) drawn from rng(0), k = 0..19, s = 512) on vectors 0, 1 and
    63 of the 64-vector batch (rng(1), d=20, n=64, r=100, scale 1/sqrt(n r));
    the batch is redrawn in order and only the kept vectors are sketched."""
    d, n, r, s = 20, 64, 100, 512
    rng = np.random.default_rng(0)
    fac = [rng.normal(0.0, 1.0 / np.sqrt(n), size=(s, n)) for _ in range(d)]
    sk = ttkrylov.KhatriRaoSketch(fac)
    rng = np.random.default_rng(1)
    full = [1] + [r] * (d - 1) + [1]
    out = {}
    for i in range(max(which) + 1):
        cores = [rng.standard_normal((full[k], n, full[k + 1])) * (1.0 / np.sqrt(n * r)) for k in range(d)]
        if i in which:
            t0 = time.perf_counter()
            out[f"kr4_y{i}"] = ttkrylov.kr_apply(sk, ttkrylov.TTVector(cores))
            out[f"kr4_wall{i}"] = np.array(time.perf_counter() - t0)
            out[f"kr4_x{i}_probe"] = np.array([cores[0][0, :4, 0], cores[-1][:4, 0, 0]])
    out["kr4_which"] = np.array(list(which))
    out["kr4_F0"] = fac[0][:4, :4].copy()
    np.savez_compressed(os.path.join(HERE, "kr_cfg4.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["tt_ops", "sketch", "streaming", "solver_small", "solver_cfg1", "serial", "precond"]
    for name in which:
        globals()["gen_" + name]()
    print("golden fixtures written to", HERE)
