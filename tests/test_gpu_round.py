"""GPU parity of the factorisations (TSQR, Jacobi SVD), TT-SVD rounding,
randomize-then-orthogonalize rounding and the streaming sketches."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import _lib
from golden_io import cores, load

pytestmark = pytest.mark.gpu


def tt_np(v):
    return [c.cpu().numpy() for c in v.cores]


def run_qr(A, cuda, transposed=False, auto=False):
    lib = _lib.load()
    m, l = A.shape
    k = min(m, l)
    if transposed:
        At = torch.as_tensor(np.ascontiguousarray(A.T), device=cuda)
        a_rs, a_cs = 1, m
    else:
        At = torch.as_tensor(A, device=cuda)
        a_rs, a_cs = l, 1
    Q = torch.empty((m, k), dtype=torch.float64, device=cuda)
    R = torch.empty((k, l), dtype=torch.float64, device=cuda)
    ws = _lib.workspace(lib.ttk_qr_ws_bytes(m, l), cuda)
    fn = lib.ttk_qr_auto if auto else lib.ttk_qr
    _lib.check(fn(m, l, At.data_ptr(), a_rs, a_cs, Q.data_ptr(), k, 1, R.data_ptr(), ws.data_ptr(),
                  ws.numel(), _lib.stream_ptr(cuda)))
    return Q.cpu().numpy(), R.cpu().numpy()


@pytest.mark.parametrize("m,l", [(10240, 80), (3200, 50), (100000, 16), (500, 112), (7, 3), (3, 7),
                                 (64, 64), (25600, 100), (1, 1), (300, 1), (3584, 119), (30720, 120),
                                 (5000, 128), (2000, 160), (150, 160)])
def test_tsqr_orthonormal_and_exact(cuda, m, l):
    rng = np.random.default_rng(m + l)
    A = rng.standard_normal((m, l))
    Q, R = run_qr(A, cuda)
    k = min(m, l)
    assert np.abs(Q.T @ Q - np.eye(k)).max() <= 1e-13 * max(l, 1) ** 0.5 * 10
    assert np.linalg.norm(Q @ R - A) <= 1e-13 * np.linalg.norm(A) * max(1, np.log2(m))
    assert np.allclose(np.tril(R, -1), 0.0)


def test_tsqr_rank_deficient_and_zero(cuda):
    rng = np.random.default_rng(1)
    B = rng.standard_normal((5000, 5))
    A = np.concatenate([B, B @ rng.standard_normal((5, 35)), np.zeros((5000, 10))], axis=1)  # rank 5 of 50
    Q, R = run_qr(A, cuda)
    assert np.abs(Q.T @ Q - np.eye(50)).max() <= 1e-12
    assert np.linalg.norm(Q @ R - A) <= 1e-13 * np.linalg.norm(A) * 10
    Z = np.zeros((900, 20))
    Q, R = run_qr(Z, cuda)
    assert np.abs(Q.T @ Q - np.eye(20)).max() <= 1e-14
    assert np.all(R == 0)


def test_tsqr_tree_rank_deficient(cuda):
    rng = np.random.default_rng(3)
    B = rng.standard_normal((6000, 30))
    A = np.concatenate([B, B, np.zeros((6000, 40)), B @ rng.standard_normal((30, 20))], axis=1)  # 120 cols
    Q, R = run_qr(A, cuda)
    assert np.abs(Q.T @ Q - np.eye(120)).max() <= 1e-12
    assert np.linalg.norm(Q @ R - A) <= 1e-13 * np.linalg.norm(A) * 10


@pytest.mark.parametrize("kind", ["gauss", "graded1e6", "graded1e12", "graded1e15", "dup", "zero"])
@pytest.mark.parametrize("trans", [False, True])
def test_qr_auto_cholqr_paths(cuda, kind, trans):
    """Shifted CholeskyQR2/3 fast path and its Householder fallback: Q orthonormal,
    A = QR to working precision, for well-, ill- and exactly-deficient inputs."""
    rng = np.random.default_rng(11)
    m, l = 12800, 80
    if kind == "gauss":
        A = rng.standard_normal((m, l))
    elif kind.startswith("graded"):
        kap = float(kind[len("graded"):])
        U, _ = np.linalg.qr(rng.standard_normal((m, l)))
        V, _ = np.linalg.qr(rng.standard_normal((l, l)))
        A = (U * np.logspace(0, -np.log10(kap), l)) @ V.T
    elif kind == "dup":
        B = rng.standard_normal((m, 40))
        A = np.concatenate([B, B], axis=1)
    else:
        A = np.zeros((m, l))
    Q, R = run_qr(A, cuda, transposed=trans, auto=True)
    # every path (CholeskyQR2, rank-robust shifted CholeskyQR3 with completion,
    # Householder) must be a backward-stable QR: orthonormal Q and A = QR to a
    # few ulps -- the solver's Arnoldi combinations cancel ~1e6x, so a 1e-12
    # factorisation error shows up as 1e-6 in the residual history
    assert np.abs(Q.T @ Q - np.eye(l)).max() <= 5e-14
    assert np.linalg.norm(Q @ R - A) <= 1e-14 * np.linalg.norm(A) + 1e-300


@pytest.mark.parametrize("m,l", [(128, 80), (80, 80), (256, 40), (512, 100), (100, 64), (1000, 96)])
@pytest.mark.parametrize("kind", ["gauss", "graded1e12", "dup"])
def test_qr_auto_squarish(cuda, m, l, kind):
    """Square-ish panels (m < 4 l) now take the CholeskyQR2 route with its
    rank-robust / Householder fallbacks (qr_auto); same backward-stability bar."""
    rng = np.random.default_rng(m + l)
    if kind == "gauss":
        A = rng.standard_normal((m, l))
    elif kind == "graded1e12":
        U, _ = np.linalg.qr(rng.standard_normal((m, l)))
        V, _ = np.linalg.qr(rng.standard_normal((l, l)))
        A = (U * np.logspace(0, -12, l)) @ V.T
    else:
        B = rng.standard_normal((m, l // 2))
        A = np.concatenate([B, B[:, : l - l // 2]], axis=1)
    Q, R = run_qr(A, cuda, auto=True)
    assert np.abs(Q.T @ Q - np.eye(l)).max() <= 5e-14
    assert np.linalg.norm(Q @ R - A) <= 1e-14 * np.linalg.norm(A)


def test_tsqr_transposed_input(cuda):
    rng = np.random.default_rng(2)
    A = rng.standard_normal((4096, 37))
    Q, R = run_qr(A, cuda, transposed=True)
    assert np.linalg.norm(Q @ R - A) <= 1e-13 * np.linalg.norm(A) * 12


@pytest.mark.parametrize("k,l", [(80, 80), (50, 50), (128, 128), (10, 30), (60, 40), (1, 5), (7, 1),
                                 (150, 150), (120, 160)])
def test_jacobi_svd(cuda, k, l):
    lib = _lib.load()
    rng = np.random.default_rng(k * 7 + l)
    # graded singular values down to 1e-13: one-sided Jacobi keeps relative accuracy
    U0, _ = np.linalg.qr(rng.standard_normal((k, k)))
    V0, _ = np.linalg.qr(rng.standard_normal((l, l)))
    kn = min(k, l)
    s0 = np.logspace(0, -13, kn)
    B = (U0[:, :kn] * s0) @ V0[:, :kn].T
    Bt = torch.as_tensor(B, device=cuda)
    U = torch.empty((k, kn), dtype=torch.float64, device=cuda)
    S = torch.empty(kn, dtype=torch.float64, device=cuda)
    want_v = k * l + l * l <= 26000
    V = torch.empty((l, kn), dtype=torch.float64, device=cuda) if want_v else None
    _lib.check(lib.ttk_svd_small(k, l, Bt.data_ptr(), U.data_ptr(), S.data_ptr(),
                                 V.data_ptr() if V is not None else None, _lib.stream_ptr(cuda)))
    S, U = S.cpu().numpy(), U.cpu().numpy()
    np.testing.assert_allclose(S, np.linalg.svd(B, compute_uv=False)[:kn], rtol=1e-9, atol=1e-15)
    assert np.all(np.diff(S) <= 0)
    if V is not None:
        V = V.cpu().numpy()
        assert np.linalg.norm((U * S) @ V.T - B) <= 1e-13 * np.linalg.norm(B) * 10


@pytest.mark.parametrize("l", [42, 50, 64, 80, 96, 100, 128])
def test_jacobi_orthogonality_gaussian(cuda, l):
    """The early-stop rule (stop after a sweep whose pairs were all within
    1e-7) must leave U and V orthonormal to working precision on the
    truncation's R^T inputs, for every kernel form (warp / block / cluster)."""
    lib = _lib.load()
    rng = np.random.default_rng(l)
    R = np.linalg.qr(rng.standard_normal((4 * l, l)))[1]
    B = np.ascontiguousarray(R.T)
    Bt = torch.as_tensor(B, device=cuda)
    U = torch.empty((l, l), dtype=torch.float64, device=cuda)
    S = torch.empty(l, dtype=torch.float64, device=cuda)
    V = torch.empty((l, l), dtype=torch.float64, device=cuda)
    _lib.check(lib.ttk_svd_small(l, l, Bt.data_ptr(), U.data_ptr(), S.data_ptr(), V.data_ptr(),
                                 _lib.stream_ptr(cuda)))
    u, s, v = U.cpu().numpy(), S.cpu().numpy(), V.cpu().numpy()
    assert np.abs(u.T @ u - np.eye(l)).max() <= 1e-13
    assert np.abs(v.T @ v - np.eye(l)).max() <= 1e-13
    assert np.abs(s - np.linalg.svd(B, compute_uv=False)).max() <= 1e-13 * s[0]
    assert np.linalg.norm(B @ v - u * s[None, :]) <= 1e-13 * np.linalg.norm(B)


def test_tt_round_golden(cuda):
    z = load("tt_ops.npz")
    for name in z["rd_names"]:
        tol, cap = z[f"{name}_spec"]
        cap = None if cap < 0 else int(cap)
        v = T.TTVector(cores(z, f"{name}_x"), device=cuda)
        r = T.tt_round(v, T.RoundSpec(float(tol), cap))
        assert r.ranks == tuple(z[f"{name}_ranks"]), name
        want = z[f"{name}_dense"]
        got = T.tt_to_dense(r).cpu().numpy()
        assert np.linalg.norm(got - want) <= 1e-12 * max(np.linalg.norm(want), 1.0), name


@pytest.mark.parametrize("tol,cap", [(1e-8, None), (1e-3, None), (0.0, 12), (1e-10, 25)])
def test_tt_round_vs_oracle(cuda, tol, cap):
    dims = [12, 9, 16, 7, 11, 10]
    a = O.tt_random(dims, [8, 14, 10, 9, 6], seed=3)
    b = O.tt_random(dims, [5, 6, 12, 7, 4], seed=4)
    x = O.add(a, O.scale(O.add(a, b), 0.5))  # redundant ranks
    want = O.tt_round(x, tol, cap, zero_rel=None)
    got = T.tt_round(T.TTVector(x, device=cuda), T.RoundSpec(tol, cap), zero_rel=None)
    assert got.ranks == tuple([1] + [c.shape[2] for c in want])
    assert O.rel_diff(tt_np(got), want) <= 1e-10


def test_rto_exactness_kat(cuda):
    """l >= true rank => RTO is exact (the RTO known-answer test)."""
    dims = [6, 6, 6, 6, 6]
    x = O.tt_random(dims, [3, 5, 4, 2], seed=11)
    big = O.add(x, O.scale(x, 0.25))  # rank doubled, true rank unchanged
    drm = O.drm_new(dims, [7, 7, 7, 7], seed=5)
    ls = O.rto_ranks(dims, [1] + [c.shape[2] for c in big], [7, 7, 7, 7])
    got = T.rto_sweeps(T.TTVector(big, device=cuda), [torch.as_tensor(g, device=cuda) for g in drm])
    assert got.ranks == tuple([1] + ls + [1])
    assert O.rel_diff(tt_np(got), O.scale(x, 1.25)) <= 1e-12
    # left-orthonormal cores
    for c in tt_np(got)[:-1]:
        q = c.reshape(-1, c.shape[2])
        assert np.abs(q.T @ q - np.eye(q.shape[1])).max() <= 1e-13


def test_rto_vs_oracle(cuda):
    dims = [16, 12, 20, 16, 10, 14]
    x = O.tt_random(dims, [30, 40, 40, 30, 14], seed=21)
    drm = O.drm_new(dims, [18, 25, 25, 18, 10], seed=9)
    ls = O.rto_ranks(dims, [1] + [c.shape[2] for c in x], [18, 25, 25, 18, 10])
    want = O.rto_sweeps(x, O.slice_drm(drm, ls))
    got = T.rto_sweeps(T.TTVector(x, device=cuda), [torch.as_tensor(g, device=cuda) for g in drm])
    assert got.ranks == tuple([1] + [c.shape[2] for c in want])
    assert O.rel_diff(tt_np(got), want) <= 1e-10
    # full randomized rounding (sweeps + truncation)
    want_r = O.rto_round(x, O.slice_drm(drm, ls), 1e-6, 15)
    got_r = T.tt_truncate_left_orth(got, T.RoundSpec(1e-6, 15))
    assert got_r.ranks == tuple([1] + [c.shape[2] for c in want_r])
    assert O.rel_diff(tt_np(got_r), want_r) <= 1e-10


@pytest.mark.parametrize("tol,cap", [(1e-8, None), (1e-3, None), (0.0, 12), (1e-10, 25)])
def test_truncate_left_orth_vs_oracle(cuda, tol, cap):
    dims = [12, 9, 16, 7, 11, 10]
    x = O.tt_random(dims, [8, 14, 10, 9, 6], seed=3)
    lo = O.rto_sweeps(O.add(x, O.scale(x, 0.5)), O.drm_new(dims, [12, 20, 20, 12, 10], seed=4))
    want = O.truncate_left_orth(lo, tol, cap)
    got = T.tt_truncate_left_orth(T.TTVector(lo, device=cuda), T.RoundSpec(tol, cap))
    assert got.ranks == tuple([1] + [c.shape[2] for c in want])
    assert O.rel_diff(tt_np(got), want) <= 1e-10


def test_rto_config2_shape(cuda):
    """BASELINE config 2 structure at d=6 (rank-200 sum of 10 rank-20 TTs, l=50, cap 40)."""
    d, n = 6, 64
    rng = np.random.default_rng(0)
    terms = [O.gaussian_tt([n] * d, [20] * (d - 1), rng, 1 / np.sqrt(n * 20)) for _ in range(10)]
    x = terms[0]
    for t in terms[1:]:
        x = O.add(x, t)
    drm = O.drm_new([n] * d, [50] * (d - 1), seed=1)
    want = O.rto_round(x, drm, 0.0, 40)
    got = T.tt_round_rto(T.TTVector(x, device=cuda), T.RoundSpec(0.0, 40),
                         drm=[torch.as_tensor(g, device=cuda) for g in drm])
    assert got.ranks == tuple([1] + [c.shape[2] for c in want])
    assert O.rel_diff(tt_np(got), want) <= 1e-10


def test_stream_sketch_and_recover_golden(cuda):
    z = load("streaming.npz")
    to = lambda cs: [torch.as_tensor(c, device=cuda) for c in cs]  # noqa: E731
    left = T.TTDRM([3, 4, 3], [1, 5, 5, 1], to(cores(z, "ss_left")))
    right = T.TTDRM([3, 4, 3], [1, 2, 2, 1], to(cores(z, "ss_right")))
    frame = T.StreamFrame(right, left)
    pair = T.stream_sketch(T.TTVector(cores(z, "ss_x"), device=cuda), frame)
    for k, p in enumerate(pair.psi):
        np.testing.assert_allclose(p.cpu().numpy(), z[f"ss_psi__{k}"], rtol=0, atol=1e-13)
    for k, o in enumerate(pair.omega):
        np.testing.assert_allclose(o.cpu().numpy(), z[f"ss_omega__{k}"], rtol=0, atol=1e-13)
    lc, rc = cores(z, "rc_left"), cores(z, "rc_right")
    frame = T.StreamFrame(T.TTDRM([4] * 4, [1] + [c.shape[2] for c in rc], to(rc)),
                          T.TTDRM([4] * 4, [1] + [c.shape[2] for c in lc], to(lc)))
    pairs = [T.stream_sketch(T.TTVector(cores(z, f"rc_v{i}"), device=cuda), frame) for i in range(5)]
    got = T.stream_recover(T.combine_pairs(pairs, list(z["rc_y"])), T.RoundSpec(1e-12))
    assert got.ranks == tuple(z["rc_ranks"])
    want = z["rc_dense"]
    assert np.linalg.norm(T.tt_to_dense(got).cpu().numpy() - want) <= 1e-10 * np.linalg.norm(want)


def test_frame_create_matches_reference_draws(cuda):
    z = load("streaming.npz")
    f = T.StreamFrame.create([3, 4, 3], [2, 2], oversampling=3, seed=6, device=cuda)
    for a, b in zip(f.left.cores + f.right.cores, cores(z, "ss_left") + cores(z, "ss_right")):
        assert np.array_equal(a.cpu().numpy(), b)


def test_counter_drm_blocks_and_moments(cuda):
    """Device TT-DRM: every leading block equals the same block of the full
    map (the solver grows its sketch ranks without redrawing), entries are
    N(0, 1/(R_{k-1} n R_k)) of the full ranks, and the map is deterministic."""
    import math
    dims = [6, 5, 7, 4]
    full = T.CounterDRM(dims, [9, 11, 8], seed=123, device=cuda)
    F = full.cores
    blk = full.block([3, 5, 2])
    L = [1, 3, 5, 2, 1]
    for k in range(4):
        assert torch.equal(blk[k], F[k][: L[k], :, : L[k + 1]].contiguous())
    again = T.CounterDRM(dims, [9, 11, 8], seed=123, device=cuda).cores
    assert all(torch.equal(a, b) for a, b in zip(F, again))
    other = T.CounterDRM(dims, [9, 11, 8], seed=124, device=cuda).cores
    assert not torch.equal(F[1], other[1])
    big = T.CounterDRM([64, 64], [256], seed=7, device=cuda).cores[1]  # 256 x 64 x 1
    z = (big * math.sqrt(256 * 64)).flatten().cpu().numpy()
    assert abs(z.mean()) < 0.05 and abs(z.std() - 1.0) < 0.05


@pytest.mark.parametrize("host,chunk", [(False, 1), (False, 4), (True, 3), (True, 100)])
def test_matvec_round_rto_pipeline(cuda, host, chunk):
    """tt_matvec_round_rto (per-core uploads, chunked matvec, event-gated RTO
    sweeps, host-streamed truncation) == tt_matvec -> rto_sweeps ->
    tt_truncate_left_orth (bit for bit on device inputs), and == the oracle."""
    rng = np.random.default_rng(5)
    dims = [12, 10, 16, 9, 14, 11, 8]
    d = len(dims)
    opc = [rng.standard_normal((1 if k == 0 else 3, n, n, 1 if k == d - 1 else 3)) for k, n in enumerate(dims)]
    x = O.tt_random(dims, [6, 9, 12, 10, 8, 5], seed=8)
    drm = O.drm_new(dims, [14, 20, 24, 20, 16, 10], seed=2)
    spec = T.RoundSpec(1e-9, 11)
    dev_op, dev_x = T.TTOperator(opc, device=cuda), T.TTVector(x, device=cuda)
    G = [torch.as_tensor(g, device=cuda) for g in drm]
    ref = T.tt_truncate_left_orth(T.rto_sweeps(T.tt_matvec(dev_op, dev_x), G), spec)
    if host:
        a = T.TTOperator([torch.as_tensor(c).pin_memory() for c in opc])
        v = T.TTVector([torch.as_tensor(c).pin_memory() for c in x])
    else:
        a, v = dev_op, dev_x
    got = T.tt_matvec_round_rto(a, v, spec, G, chunk=chunk, device=cuda)
    torch.cuda.synchronize()
    assert got.device.type == ("cpu" if host else "cuda")
    assert got.ranks == ref.ranks
    # a right sweep that runs beside matvec chunks keeps its contractions off the TMA-staged
    # GEMM (DESIGN 6.2): same arithmetic, another kernel's summation order
    assert O.rel_diff([c.cpu().numpy() for c in got.cores], [c.cpu().numpy() for c in ref.cores]) <= 1e-12
    y = O.matvec(opc, x)
    ls = O.rto_ranks(dims, [1] + [c.shape[2] for c in y], [14, 20, 24, 20, 16, 10])
    want = O.rto_round(y, O.slice_drm(drm, ls), 1e-9, 11)
    assert got.ranks == tuple([1] + [c.shape[2] for c in want])
    assert O.rel_diff([c.cpu().numpy() for c in got.cores], want) <= 1e-10


@pytest.mark.parametrize("host", [False, True])
@pytest.mark.parametrize("dims", [[9], [7, 11], [5, 6, 4]])
def test_matvec_round_rto_pipeline_small(cuda, host, dims):
    """Edge sizes of the pipelined call (d = 1 takes the copy branches)."""
    rng = np.random.default_rng(len(dims))
    d = len(dims)
    opc = [rng.standard_normal((1 if k == 0 else 2, n, n, 1 if k == d - 1 else 2)) for k, n in enumerate(dims)]
    x = O.tt_random(dims, [3] * (d - 1), seed=4) if d > 1 else [rng.standard_normal((1, dims[0], 1))]
    drm = O.drm_new(dims, [4] * (d - 1), seed=6) if d > 1 else [rng.standard_normal((1, dims[0], 1))]
    spec = T.RoundSpec(1e-10, 5)
    G = [torch.as_tensor(g, device=cuda) for g in drm]
    dev_op, dev_x = T.TTOperator(opc, device=cuda), T.TTVector(x, device=cuda)
    ref = T.tt_truncate_left_orth(T.rto_sweeps(T.tt_matvec(dev_op, dev_x), G), spec)
    if host:
        a = T.TTOperator([torch.as_tensor(c).pin_memory() for c in opc])
        v = T.TTVector([torch.as_tensor(c).pin_memory() for c in x])
    else:
        a, v = dev_op, dev_x
    got = T.tt_matvec_round_rto(a, v, spec, G, device=cuda)
    torch.cuda.synchronize()
    assert got.ranks == ref.ranks
    if host and len(dims) > 1:
        assert O.rel_diff([c.cpu().numpy() for c in got.cores], [c.cpu().numpy() for c in ref.cores]) <= 1e-12
    else:
        for g_, w in zip(got.cores, ref.cores):
            assert torch.equal(g_.cpu(), w.cpu())


# ---------------------------------------------------------------------------
# ranks above the register-resident kernels (kQrMaxCols = 160): column-blocked
# QR (BCGS2 panels) and the grid-cooperative Jacobi (csrc/qr_wide.cu)

@pytest.mark.parametrize("m,l,kind", [(12800, 200, "gauss"), (4000, 300, "gauss"), (12800, 192, "graded1e12"),
                                      (6000, 200, "dup"), (64, 200, "gauss"), (192, 200, "gauss"),
                                      (200, 200, "gauss"), (900, 161, "zero")])
def test_qr_wide_blocked(cuda, m, l, kind):
    rng = np.random.default_rng(m + l)
    if kind == "gauss":
        A = rng.standard_normal((m, l))
    elif kind == "graded1e12":
        U, _ = np.linalg.qr(rng.standard_normal((m, l)))
        V, _ = np.linalg.qr(rng.standard_normal((l, l)))
        A = (U * np.logspace(0, -12, l)) @ V.T
    elif kind == "dup":
        B = rng.standard_normal((m, 100))
        A = np.concatenate([B, B], axis=1)
    else:
        A = np.zeros((m, l))
    for trans in (False, True):
        Q, R = run_qr(A, cuda, transposed=trans, auto=True)
        k = min(m, l)
        assert np.abs(Q.T @ Q - np.eye(k)).max() <= 5e-14
        assert np.linalg.norm(Q @ R - A) <= 1e-14 * np.linalg.norm(A) + 1e-300
        if kind == "gauss":  # full-rank panels take the triangular fast path
            assert np.all(np.tril(R, -1) == 0)


@pytest.mark.parametrize("k,l", [(200, 200), (192, 192), (300, 250), (80, 200), (200, 64), (161, 161)])
def test_jacobi_svd_wide(cuda, k, l):
    lib = _lib.load()
    rng = np.random.default_rng(k * 7 + l)
    U0, _ = np.linalg.qr(rng.standard_normal((k, k)))
    V0, _ = np.linalg.qr(rng.standard_normal((l, l)))
    kn = min(k, l)
    s0 = np.logspace(0, -13, kn)
    B = (U0[:, :kn] * s0) @ V0[:, :kn].T
    Bt = torch.as_tensor(B, device=cuda)
    U = torch.empty((k, kn), dtype=torch.float64, device=cuda)
    S = torch.empty(kn, dtype=torch.float64, device=cuda)
    V = torch.empty((l, kn), dtype=torch.float64, device=cuda)
    _lib.check(lib.ttk_svd_small(k, l, Bt.data_ptr(), U.data_ptr(), S.data_ptr(), V.data_ptr(),
                                 _lib.stream_ptr(cuda)))
    S, U, V = S.cpu().numpy(), U.cpu().numpy(), V.cpu().numpy()
    np.testing.assert_allclose(S, np.linalg.svd(B, compute_uv=False)[:kn], rtol=1e-9, atol=1e-15)
    assert np.all(np.diff(S) <= 0)
    # accumulated V: one rounding error per rotation, ~sweeps x l rotations per column
    assert np.abs(V.T @ V - np.eye(kn)).max() <= 2e-15 * l
    assert np.linalg.norm((U * S) @ V.T - B) <= 1e-13 * np.linalg.norm(B) * 10


def test_tt_round_rank200_vs_oracle(cuda):
    """TT-SVD at ranks above 160 (tt.py:330,361 at any rank): d=5, rank 200 -> tol/cap."""
    rng = np.random.default_rng(5)
    dims, ranks = [8, 30, 30, 30, 8], [1, 8, 200, 200, 8, 1]
    x = [rng.standard_normal((ranks[k], dims[k], ranks[k + 1])) for k in range(5)]
    for tol, cap in ((1e-10, None), (0.0, 170), (1e-3, None)):
        got = T.tt_round(T.TTVector(x, device=cuda), T.RoundSpec(tol, cap), zero_rel=None)
        want = O.tt_round(x, tol, cap, zero_rel=None)
        assert list(got.ranks) == [1] + [c.shape[2] for c in want]
        assert O.rel_diff(tt_np(got), want) <= 1e-10


# ---------------------------------------------------------------------------
# race detection by determinism (compute-sanitizer is closed on the GPU pool,
# profiles/r02_sanitizer_refused.log): the kernels with cross-CTA hand-offs --
# DSMEM st.async + mbarrier block moves (Jacobi cluster kernels), cooperative
# grid barriers (fused CholeskyQR2) -- must give bit-identical results on every
# run and when several run concurrently on separate streams; a missing
# barrier / stale DSMEM read would show up as run-to-run differences.

@pytest.mark.parametrize("l", [80, 50, 112])
def test_jacobi_cluster_kernels_deterministic(cuda, l):
    lib = _lib.load()
    rng = np.random.default_rng(l)
    B = torch.as_tensor(np.ascontiguousarray(np.linalg.qr(rng.standard_normal((10 * l, l)))[1].T), device=cuda)
    outs = []
    streams = [torch.cuda.Stream(cuda) for _ in range(4)]
    for it in range(24):
        st = streams[it % 4]
        U = torch.empty((l, l), dtype=torch.float64, device=cuda)
        S = torch.empty(l, dtype=torch.float64, device=cuda)
        V = torch.empty((l, l), dtype=torch.float64, device=cuda)
        with torch.cuda.stream(st):
            _lib.check(lib.ttk_svd_small(l, l, B.data_ptr(), U.data_ptr(), S.data_ptr(), V.data_ptr(), st.cuda_stream))
        outs.append((U, S, V))
    torch.cuda.synchronize()
    for U, S, V in outs[1:]:
        assert torch.equal(U, outs[0][0]) and torch.equal(S, outs[0][1]) and torch.equal(V, outs[0][2])


def test_fused_cholqr2_deterministic(cuda):
    lib = _lib.load()
    m, l = 10240, 80
    A = torch.as_tensor(np.random.default_rng(0).standard_normal((m, l)), device=cuda)
    res = []
    for it in range(16):
        Q = torch.empty_like(A)
        R = torch.empty((l, l), dtype=torch.float64, device=cuda)
        ws = _lib.workspace(lib.ttk_qr_ws_bytes(m, l), cuda)
        _lib.check(lib.ttk_qr_auto(m, l, A.data_ptr(), l, 1, Q.data_ptr(), l, 1, R.data_ptr(), ws.data_ptr(),
                                   ws.numel(), _lib.stream_ptr(cuda)))
        res.append((Q, R))
    torch.cuda.synchronize()
    for Q, R in res[1:]:
        assert torch.equal(Q, res[0][0]) and torch.equal(R, res[0][1])


def _trunc_paths():
    import ctypes
    from paper_2409_09471_b200 import _lib
    c = (ctypes.c_longlong * 3)()
    _lib.load().ttk_debug_truncate_paths(ctypes.addressof(c))
    return c[0], c[1], c[2]


def test_truncate_gram_path_certified(cuda):
    """Exact-rank truncation (rel_tol = 0, cap) of a generic left-orthogonal TT goes
    through the Gram + Cholesky path on every core and matches the oracle's SVD path."""
    dims = [12, 9, 16, 7, 11, 10]
    x = O.tt_random(dims, [8, 14, 10, 9, 6], seed=5)
    lo = O.rto_sweeps(x, O.drm_new(dims, [8, 14, 10, 9, 6], seed=6))  # sketch ranks = TT ranks: full rank
    want = O.truncate_left_orth(lo, 0.0, 6)
    g0, q0, x0 = _trunc_paths()
    got = T.tt_truncate_left_orth(T.TTVector(lo, device=cuda), T.RoundSpec(0.0, 6))
    g1, q1, x1 = _trunc_paths()
    assert (g1 - g0, q1 - q0, x1 - x0) == (len(dims) - 1, 0, 0)
    assert got.ranks == tuple([1] + [c.shape[2] for c in want])
    assert O.rel_diff(tt_np(got), want) <= 1e-10
    for c in got.cores[1:]:  # right-orthonormal cores, as the SVD path leaves them
        u = c.cpu().numpy().reshape(c.shape[0], -1)
        assert np.abs(u @ u.T - np.eye(u.shape[0])).max() <= 1e-12


def _trunc_paths_ex(n=5):
    import ctypes
    from paper_2409_09471_b200 import _lib
    c = (ctypes.c_longlong * n)()
    _lib.load().ttk_debug_truncate_paths_ex(ctypes.addressof(c), n)
    return np.array(list(c))


def test_rto_sweeps_deferred_acceptance(cuda):
    """The left sweep of a shape whose last sweep stayed on the fused CholeskyQR2 fast path
    accepts its factorisations on the device and checks the flags once per sweep (no per-core
    host wait); a deferred sweep that meets exactly rank-deficient sketches is redone with the
    per-core check (rank-robust path) and takes the shape out of the deferral again.  Every
    result represents its input exactly."""
    dims = [40, 36, 44, 40, 41]  # a shape no other test uses
    x = O.tt_random(dims, [40, 48, 48, 40], seed=21)
    drm = [torch.as_tensor(g, device=cuda) for g in O.drm_new(dims, [34, 40, 40, 34], seed=22)]
    xv = T.TTVector(x, device=cuda)
    c0 = _trunc_paths_ex(7)
    first = T.rto_sweeps(xv, drm)
    d1 = _trunc_paths_ex(7) - c0
    assert (d1[5], d1[6]) == (0, 0)  # unknown shape: per-core check
    got = T.rto_sweeps(xv, drm)
    d2 = _trunc_paths_ex(7) - c0 - d1
    assert (d2[5], d2[6]) == (1, 0)  # proven shape: deferred
    for a, b in zip(first.cores, got.cores):
        assert torch.equal(a, b)
    assert O.rel_diff(tt_np(got), O.rto_sweeps(x, O.drm_new(dims, [34, 40, 40, 34], seed=22))) <= 1e-10
    # same nominal shape, true ranks halved: every sketch Gram is singular
    y = O.tt_random(dims, [20, 24, 24, 20], seed=23)
    z = O.add(y, O.scale(y, 0.5))
    zv = T.TTVector(z, device=cuda)
    c0 = _trunc_paths_ex(7)
    got = T.rto_sweeps(zv, drm)
    d3 = _trunc_paths_ex(7) - c0
    assert (d3[5], d3[6]) == (0, 1)  # refused, redone
    assert O.rel_diff(tt_np(got), z) <= 1e-10
    got2 = T.rto_sweeps(zv, drm)
    d4 = _trunc_paths_ex(7) - c0 - d3
    assert (d4[5], d4[6]) == (0, 0)  # back to the per-core check
    for a, b in zip(got.cores, got2.cores):
        assert torch.equal(a, b)


def _gapped_left_orth(dims, r, s, eps, seed):
    """Left-orthogonal TT (RTO output with exact range) whose unfoldings have a
    gap ~1/eps after the first r singular values: A + eps B, rank r + s."""
    a = O.tt_random(dims, [r] * (len(dims) - 1), seed=seed)
    b = O.tt_random(dims, [s] * (len(dims) - 1), seed=seed + 1)
    x = O.add(a, O.scale(b, eps))
    return O.rto_sweeps(x, O.drm_new(dims, [r + s] * (len(dims) - 1), seed=seed + 2))


@pytest.mark.parametrize("r,s,eps", [(6, 4, 1e-3), (20, 12, 1e-2), (64, 16, 1e-2)])
def test_truncate_subspace_path_gapped(cuda, r, s, eps):
    """Exact-rank truncation of a TT with a clear gap at the cap: every core takes
    the gap-certified subspace kernel (no Jacobi SVD), the rounded TT matches the
    oracle's SVD truncation to 1e-12 with equal ranks and right-orthonormal cores."""
    dims = [10, 12, 9, 11, 8, 10] if r < 64 else [24, 16, 20, 16]
    lo = _gapped_left_orth(dims, r, s, eps, seed=11)
    want = O.truncate_left_orth(lo, 0.0, r)
    c0 = _trunc_paths_ex()
    got = T.tt_truncate_left_orth(T.TTVector(lo, device=cuda), T.RoundSpec(0.0, r))
    d = _trunc_paths_ex() - c0
    # cores with n_k r_k < r_{k-1} (a rank-deficient Gram) take the QR path
    assert d[3] >= 2 and d[3] + d[1] == len(dims) - 1 and d[4] == 0 and d[0] == 0
    assert got.ranks == tuple([1] + [c.shape[2] for c in want])
    assert O.rel_diff(tt_np(got), want) <= 1e-12
    # right-orthonormal cores: M G M^T = I to the Cholesky's rounding; the kernel
    # looks at D = M F - I (and removes it to second order) unless its condition
    # bound already keeps it below ~5e-12 (DESIGN 2.2); the represented tensor
    # above is what parity is stated on
    for c in got.cores[1:]:
        u = c.cpu().numpy().reshape(c.shape[0], -1)
        assert np.abs(u @ u.T - np.eye(u.shape[0])).max() <= 2e-11


def test_truncate_subspace_certificate_rejects_flat_spectrum(cuda):
    """No gap at the cap: the subspace certificate fails, the sweep is redone with the
    Jacobi SVD (same result as the oracle), and the next call of the same shape goes
    straight to the Jacobi path."""
    dims = [12, 9, 16, 7, 11, 13]
    x = O.tt_random(dims, [8, 14, 10, 9, 6], seed=5)
    lo = O.rto_sweeps(x, O.drm_new(dims, [8, 14, 10, 9, 6], seed=6))
    want = O.truncate_left_orth(lo, 0.0, 6)
    # a shape no other test uses, so the skip hint starts clean
    c0 = _trunc_paths_ex()
    got = T.tt_truncate_left_orth(T.TTVector(lo, device=cuda), T.RoundSpec(0.0, 6))
    d1 = _trunc_paths_ex() - c0
    assert d1[4] == 1 and d1[0] == len(dims) - 1 and d1[2] == 0
    assert O.rel_diff(tt_np(got), want) <= 1e-10
    got2 = T.tt_truncate_left_orth(T.TTVector(lo, device=cuda), T.RoundSpec(0.0, 6))
    d2 = _trunc_paths_ex() - c0 - d1
    assert d2[4] == 0 and d2[3] == 0 and d2[0] == len(dims) - 1
    for a, b in zip(got.cores, got2.cores):
        assert torch.equal(a, b)


def test_truncate_gram_path_falls_back_on_rank_deficiency(cuda):
    """rel_tol = 0 on a TT whose unfoldings are exactly rank deficient: the kept
    singular values include ~1e-16 ones, a certificate fails and the truncation
    is redone through the QR path (the reference's behaviour: keep min(cap, l))."""
    dims = [10, 12, 9, 11, 8]
    y = O.tt_random(dims, [3, 4, 4, 3], seed=7)
    x = O.add(y, O.scale(y, 0.5))  # nominal ranks 6, 8, 8, 6; true ranks 3, 4, 4, 3
    lo = O.rto_sweeps(x, O.drm_new(dims, [8, 10, 10, 8], seed=8))
    want = O.truncate_left_orth(lo, 0.0, 6)
    g0, q0, x0 = _trunc_paths()
    got = T.tt_truncate_left_orth(T.TTVector(lo, device=cuda), T.RoundSpec(0.0, 6))
    g1, q1, x1 = _trunc_paths()
    assert x1 - x0 == 1 and q1 - q0 == len(dims) - 1
    assert got.ranks == tuple([1] + [c.shape[2] for c in want])
    assert O.diff_norm(tt_np(got), want) <= 1e-10 * O.norm(want)
