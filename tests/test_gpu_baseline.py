"""Parity at the full BASELINE.json sizes (configs 2-5), on the device, against
the reference's own outputs (golden fixtures made by make_golden.py, which
runs the reference package) or the CPU oracle where the reference has no
implementation (randomize-then-orthogonalize).

North-star bars (BASELINE.json): rounded TTs <= 1e-10 relative via the
orthogonalize-then-norm metric with equal ranks; sketched vectors <= 1e-12
relative; solver: identical iteration counts and rank histories, final
residual within 1e-8 relative.
"""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2409_09471_b200 as T
from golden_io import cores, load
from paper_2409_09471_b200 import configs

pytestmark = pytest.mark.gpu

# absolute roundoff floor of a sketched residual (relative to ||S b||, ~45 ulp):
# the reference's own final residual moves by ~1e-16 absolute under 1e-16
# noise in its roundings (profiles/r02_solver_sensitivity_small.txt)
RES_FLOOR = 1e-14


def _probe(x):
    """24-row Khatri-Rao probe of a TT (make_golden.probe_sketch: kr_sketch_new(dims, 24, seed=777))."""
    f = O.kr_factors_new(list(x.dims), 24, seed=777)
    return O.kr_apply(f, [c.cpu().numpy() for c in x.cores])


# ---------------------------------------------------------------------------
# config 3: matvec (rho=3, r=64 -> 192) + RTO l=80 -> 64, d=32, n=128

def test_config3_full_size_vs_oracle(cuda):
    """The headline step at full size, device-resident and through the host
    pipeline, against oracle.matvec + oracle.rto_round on the same seeded inputs."""
    import ctypes
    from paper_2409_09471_b200 import _lib
    C = configs.config3()
    spec = T.RoundSpec(C["rel_tol"], C["max_rank"])
    drm = [torch.as_tensor(g, device=cuda) for g in C["drm"]]
    c0 = (ctypes.c_longlong * 5)()
    _lib.load().ttk_debug_truncate_paths_ex(ctypes.addressof(c0), 5)
    got = T.tt_matvec_round_rto(T.TTOperator(C["op"], device=cuda), T.TTVector(C["x"], device=cuda), spec, drm,
                                device=cuda)
    y = O.matvec(C["op"], C["x"])
    want = O.rto_round(y, C["drm"], C["rel_tol"], C["max_rank"])
    assert list(got.ranks) == [1] + [c.shape[2] for c in want] == [1] + [64] * 31 + [1]
    assert O.rel_diff([c.cpu().numpy() for c in got.cores], want) <= 1e-10
    # every core went through the gap-certified subspace kernel (sigma_64 / sigma_65 = 41..440)
    c1 = (ctypes.c_longlong * 5)()
    _lib.load().ttk_debug_truncate_paths_ex(ctypes.addressof(c1), 5)
    assert (c1[3] - c0[3], c1[4] - c0[4], c1[0] - c0[0]) == (31, 0, 0)
    for c in got.cores[1:]:  # right-orthonormal, as the reference's SVD leaves them
        u = c.cpu().numpy().reshape(c.shape[0], -1)
        assert np.abs(u @ u.T - np.eye(u.shape[0])).max() <= 1e-12
    # host (pinned) cores in and out: the same tensor (the pipelined right sweep uses the cp.async GEMM)
    host = T.tt_matvec_round_rto(T.TTOperator([torch.as_tensor(g).pin_memory() for g in C["op"]]),
                                 T.TTVector([torch.as_tensor(c).pin_memory() for c in C["x"]]), spec, drm,
                                 device=cuda)
    assert list(host.ranks) == list(got.ranks)
    assert O.rel_diff([c.cpu().numpy() for c in host.cores], [c.cpu().numpy() for c in got.cores]) <= 1e-12
    # the unrounded matvec cores elementwise (<= 1e-13 of the core norm)
    ym = T.tt_matvec(T.TTOperator(C["op"], device=cuda), T.TTVector(C["x"], device=cuda))
    for k in (0, 1, 15, 31):
        g = ym.cores[k].cpu().numpy()
        assert np.abs(g - y[k]).max() <= 1e-13 * np.abs(y[k]).max()


def test_config3_two_problems_in_flight(cuda):
    """Two host threads, each driving the headline step on its own stream inside
    _lib.concurrent_problems() (how bench.py's in-flight mode and
    parallel.solve_rhs_sharded run): every result is the same tensor as a lone run.
    DESIGN 6.2: with the TMA-staged GEMM left on, overlapping problems returned
    corrupted cores in ~1 of 3 runs."""
    import threading
    from paper_2409_09471_b200 import _lib
    C = configs.config3()
    spec = T.RoundSpec(C["rel_tol"], C["max_rank"])
    drm = [torch.as_tensor(g, device=cuda) for g in C["drm"]]
    op, x = T.TTOperator(C["op"], device=cuda), T.TTVector(C["x"], device=cuda)
    ref = T.tt_matvec_round_rto(op, x, spec, drm, device=cuda)
    nref = float(T.tt_norm(ref))
    torch.cuda.synchronize()
    out = {}

    def worker(i):
        torch.cuda.set_device(cuda)
        s = torch.cuda.Stream(cuda)
        with torch.cuda.stream(s):
            worst = 0.0
            for _ in range(4):
                y = T.tt_matvec_round_rto(op, x, spec, drm, device=cuda)
                assert y.ranks == ref.ranks
                worst = max(worst, float(T.tt_norm(T.tt_add(y, T.tt_scale(ref, -1.0)))) / nref)
            s.synchronize()
        out[i] = worst

    with _lib.concurrent_problems():
        ths = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
        [t.start() for t in ths]
        [t.join() for t in ths]
    # ||a - b|| through dot products: cancellation floor ~1e-8; a corrupted core gives >= 1e-4
    assert sorted(out) == [0, 1] and max(out.values()) <= 1e-6, out


# ---------------------------------------------------------------------------
# config 2: sum of 10 rank-20 TTs (d=16, n=64) -> rank 200; RTO l=50 -> 40

def test_config2_full_size_rto_vs_oracle(cuda):
    C = configs.config2()
    x = T.TTVector(C["x"], device=cuda)
    assert list(x.ranks) == [1] + [200] * 15 + [1]
    drm = [torch.as_tensor(g, device=cuda) for g in C["drm"]]
    sw = T.rto_sweeps(x, drm)
    got = T.tt_truncate_left_orth(sw, T.RoundSpec(C["rel_tol"], C["max_rank"]))
    want_sw = O.rto_sweeps(C["x"], C["drm"])
    assert list(sw.ranks) == [1] + [c.shape[2] for c in want_sw] == [1] + [50] * 15 + [1]
    assert O.rel_diff([c.cpu().numpy() for c in sw.cores], want_sw) <= 1e-10
    want = O.truncate_left_orth(want_sw, C["rel_tol"], C["max_rank"])
    assert list(got.ranks) == [1] + [c.shape[2] for c in want] == [1] + [40] * 15 + [1]
    assert O.rel_diff([c.cpu().numpy() for c in got.cores], want) <= 1e-10


def test_config2_full_size_tt_svd_vs_oracle(cuda):
    """Reference tt_round (TT-SVD, Q1 bypassed) at rank 200 -> cap 40: QR of
    (64*200) x 200 unfoldings and 200 x 200 SVDs on the device."""
    C = configs.config2()
    got = T.tt_round(T.TTVector(C["x"], device=cuda), T.RoundSpec(0.0, 40), zero_rel=None)
    want = O.tt_round(C["x"], 0.0, 40, zero_rel=None)
    assert list(got.ranks) == [1] + [c.shape[2] for c in want]
    assert O.rel_diff([c.cpu().numpy() for c in got.cores], want) <= 1e-10


# ---------------------------------------------------------------------------
# config 4: Khatri-Rao sketch, s=512, 64 TTs d=20 n=64 r=100

@pytest.fixture(scope="module")
def cfg4(cuda):
    C = configs.config4()
    sk = T.KhatriRaoSketch(C["factors"], device=cuda)
    vs = [T.TTVector(v, device=cuda) for v in C["vecs"]]
    return C, sk, vs


def test_config4_full_batch_vs_reference(cuda, cfg4):
    """The full 64-vector batch in one launch; vectors 0, 1, 63 against the
    reference kr_apply(KhatriRaoSketch(F), v) outputs (sketch.py:50-70)."""
    C, sk, vs = cfg4
    z = load("kr_cfg4.npz")
    assert np.array_equal(C["factors"][0][:4, :4], z["kr4_F0"])
    y = T.kr_apply_batch(sk, vs).cpu().numpy()
    assert y.shape == (64, 512)
    for i in z["kr4_which"]:
        i = int(i)
        assert np.array_equal(np.array([C["vecs"][i][0][0, :4, 0], C["vecs"][i][-1][:4, 0, 0]]), z[f"kr4_x{i}_probe"])
        want = z[f"kr4_y{i}"]
        assert np.linalg.norm(y[i] - want) <= 1e-12 * np.linalg.norm(want), i


def test_config4_row_shards_match_full(cuda, cfg4):
    """Row-sharded sketches (the 1/2/4/8-GPU partition) reassemble the full batch in fixed row order."""
    from paper_2409_09471_b200.parallel import row_partition
    C, sk, vs = cfg4
    full = T.kr_apply_batch(sk, vs)
    for world in (2, 8):
        parts = [T.kr_apply_rows(sk, vs, lo, hi) for lo, hi in row_partition(512, world)]
        got = torch.cat(parts, dim=1)
        # fixed row positions; a shard may take the two-phase path (different
        # summation order), so equal to the full batch to roundoff, per vector
        err = torch.linalg.norm(got - full, dim=1) / torch.linalg.norm(full, dim=1)
        assert float(err.max()) <= 1e-13, world


# ---------------------------------------------------------------------------
# config 5: TT-sGMRES, d=50, n=256, ell=3, s=120, maxit 60, cap 100

def _cfg5_inputs(j, cuda, **extra):
    C = configs.config5(j)
    z = load("solver_cfg5.npz")
    # the committed reference run used the same seeded inputs
    assert np.array_equal(np.random.default_rng(0).uniform(0.1, 1.0, 50), z[f"cfg5_{j}_c"])
    for a, b in zip(C["b"], cores(z, f"cfg5_{j}_b")):
        assert np.allclose(a, b, rtol=1e-15, atol=0)
    cfg = T.SolverConfig(**C["cfg"], zero_rel=None, **extra)
    a = T.TTOperator(C["op"], device=cuda)
    b = T.TTVector(C["b"], device=cuda)
    s = T.kr_sketch_new(C["dims"], cfg.sketch_rows, seed=C["sketch_seed"], device=cuda)
    assert np.array_equal(s.factors[0][:4].cpu().numpy(), z[f"cfg5_{j}_sketch0"])
    frame = T.make_solver_frame(b, cfg, seed=C["frame_seed"])
    return C, z, cfg, a, b, s, frame


@pytest.mark.parametrize("j", [0, 1])
def test_config5_tt_svd_vs_reference(cuda, j):
    """Reference tt_sgmres (TT-SVD rounding, Q1 bypassed) at the full config-5 size."""
    C, z, cfg, a, b, s, frame = _cfg5_inputs(j, cuda)
    x, rep = T.tt_sgmres(a, b, None, cfg, s, frame)
    name = f"cfg5_{j}"
    assert rep.iterations == int(z[name + "_iters"])
    assert rep.converged == bool(z[name + "_conv"])
    assert rep.basis_rank == [int(r) for r in z[name + "_ranks"]]
    want = z[name + "_res"]
    assert abs(rep.res_sketched[-1] - want[-1]) <= 1e-8 * want[-1] + RES_FLOOR
    np.testing.assert_allclose(rep.res_sketched, want, rtol=1e-8, atol=RES_FLOOR)
    assert list(x.ranks) == [int(r) for r in z[name + "_xranks"]]
    wp = z[name + "_xprobe"]
    assert np.linalg.norm(_probe(x) - wp) <= 1e-8 * np.linalg.norm(wp)
    assert abs(T.tt_norm(x) - float(z[name + "_xnorm"])) <= 1e-8 * float(z[name + "_xnorm"])


def test_config5_rto_vs_oracle(cuda):
    """Randomized-rounding mode at full config-5 size against oracle.sgmres(rounding="rto")
    with the device counter-based DRM materialised for the oracle."""
    C, z, cfg, a, b, s, frame = _cfg5_inputs(0, cuda, rounding="rto")
    x, rep = T.tt_sgmres(a, b, None, cfg, s, frame)
    ocfg = {"maxit": cfg.maxit, "tol": cfg.tol, "ell": cfg.ell, "eta": cfg.eta, "max_rank": cfg.max_rank,
            "oversampling": cfg.oversampling, "seed": cfg.seed, "zero_rel": None}
    drm = [g.cpu().numpy() for g in T.solver_rto_drm(b.dims, cfg, device=cuda).cores]
    f_np = [f.cpu().numpy() for f in s.factors]
    ox, orep = O.sgmres(C["op"], C["b"], ocfg, f_np, frame=O.solver_frame(C["b"], ocfg, seed=C["frame_seed"]),
                        rounding="rto", rto_drm=drm)
    assert rep.iterations == orep["iterations"]
    assert rep.converged == orep["converged"]
    assert rep.basis_rank == orep["basis_rank"]
    assert abs(rep.res_sketched[-1] - orep["res_sketched"][-1]) <= 1e-8 * orep["res_sketched"][-1] + RES_FLOOR
    np.testing.assert_allclose(rep.res_sketched, orep["res_sketched"], rtol=1e-8, atol=RES_FLOOR)
    assert O.rel_diff([c.cpu().numpy() for c in x.cores], ox) <= 1e-8
