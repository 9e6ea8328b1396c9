"""Pin the CPU oracle (oracle/) to golden vectors produced by the reference itself."""

import numpy as np
import pytest

import oracle as O
from golden_io import cores, factors, load


def assert_cores_close(got, want, rtol=1e-13):
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g.shape == w.shape
        scale = max(np.abs(w).max(), 1e-300)
        assert np.abs(g - w).max() <= rtol * scale


@pytest.fixture(scope="module")
def ops():
    return load("tt_ops.npz")


def test_matvec_golden(ops):
    for name in ops["mv_names"]:
        y = O.matvec(cores(ops, f"{name}_op"), cores(ops, f"{name}_x"))
        assert_cores_close(y, cores(ops, f"{name}_y"), 1e-14)


def test_add_scale_axpy_golden(ops):
    assert_cores_close(O.add(cores(ops, "add_a"), cores(ops, "add_b")), cores(ops, "add_y"), 0)
    assert_cores_close(O.add(cores(ops, "add1_a"), cores(ops, "add1_b")), cores(ops, "add1_y"), 0)
    assert_cores_close(O.scale(cores(ops, "scale_a"), -2.5), cores(ops, "scale_y"), 0)
    h = ops["axpy_h"]
    y = O.concat_axpy([cores(ops, "axpy_vt"), cores(ops, "axpy_v1"), cores(ops, "axpy_v2")],
                      [1.0, -h[0], -h[1]])
    assert_cores_close(y, cores(ops, "axpy_y"), 0)


def test_dot_norm_golden(ops):
    assert O.dot(cores(ops, "dot_a"), cores(ops, "dot_b")) == pytest.approx(float(ops["dot_ab"]), rel=1e-14)
    assert O.norm(cores(ops, "norm_a")) == pytest.approx(float(ops["norm_a_val"]), rel=1e-14)


def test_round_golden(ops):
    for name in ops["rd_names"]:
        tol, cap = ops[f"{name}_spec"]
        cap = None if cap < 0 else int(cap)
        r = O.tt_round(cores(ops, f"{name}_x"), tol, cap)
        assert tuple([1] + [c.shape[2] for c in r]) == tuple(ops[f"{name}_ranks"])
        want = ops[f"{name}_dense"]
        scale = max(np.linalg.norm(want), 1.0)
        assert np.linalg.norm(O.to_dense(r) - want) <= 1e-12 * scale


def test_kr_golden():
    z = load("sketch.npz")
    for name in z["kr_names"]:
        y = O.kr_apply(factors(z, name), cores(z, f"{name}_x"))
        want = z[f"{name}_y"]
        assert np.abs(y - want).max() <= 1e-13 * max(np.abs(want).max(), 1.0)


def test_streaming_golden():
    z = load("streaming.npz")
    left, right = cores(z, "ss_left"), cores(z, "ss_right")
    # the frame generator reproduces StreamFrame.create(dims, [2,2], oversampling=3, seed=6)
    l2, r2 = O.frame_new([3, 4, 3], [2, 2], oversampling=3, seed=6)
    for a, b in zip(l2 + r2, left + right):
        assert np.array_equal(a, b)
    psi, omega = O.stream_sketch(cores(z, "ss_x"), left, right)
    for k, p in enumerate(psi):
        np.testing.assert_allclose(p, z[f"ss_psi__{k}"], rtol=0, atol=1e-13)
    for k, o in enumerate(omega):
        np.testing.assert_allclose(o, z[f"ss_omega__{k}"], rtol=0, atol=1e-13)
    left, right = cores(z, "rc_left"), cores(z, "rc_right")
    vs = [cores(z, f"rc_v{i}") for i in range(5)]
    comb = O.combine_pairs([O.stream_sketch(v, left, right) for v in vs], list(z["rc_y"]))
    got = O.stream_recover(comb[0], comb[1], [4, 4, 4, 4], 1e-12)
    assert tuple([1] + [c.shape[2] for c in got]) == tuple(z["rc_ranks"])
    want = z["rc_dense"]
    assert np.linalg.norm(O.to_dense(got) - want) <= 1e-10 * np.linalg.norm(want)


def _cfg_from(z, name):
    c = z[f"{name}_cfg"]
    return {"maxit": int(c[0]), "tol": float(c[1]), "ell": int(c[2]), "eta": float(c[3]),
            "max_rank": None if c[4] < 0 else int(c[4]), "sketch_rows": int(c[5]),
            "oversampling": int(c[6]), "solution_rank": None if c[7] < 0 else int(c[7]),
            "seed": int(c[8]), "combine_mode": "stta" if c[9] else "explicit"}


def test_solver_small_golden():
    z = load("solver_small.npz")
    for name in z["sv_names"]:
        cfg = _cfg_from(z, name)
        x, rep = O.sgmres(cores(z, f"{name}_op"), cores(z, f"{name}_b"), cfg, factors(z, name))
        assert rep["iterations"] == int(z[f"{name}_iters"])
        assert rep["basis_rank"] == list(z[f"{name}_ranks"])
        np.testing.assert_allclose(rep["res_sketched"], z[f"{name}_res"], rtol=1e-8)
        assert abs(rep["res_sketched"][-1] - z[f"{name}_res"][-1]) <= 1e-8 * z[f"{name}_res"][-1]
        probe = O.kr_apply(O.kr_factors_new([c.shape[1] for c in x], 24, seed=777), x)
        want = z[f"{name}_xprobe"]
        assert np.linalg.norm(probe - want) <= 1e-8 * np.linalg.norm(want)


def test_solver_cfg1_golden():
    """BASELINE config 1 (d=8, n=32, 40 iterations) with the Q1 zero test bypassed."""
    z = load("solver_cfg1.npz")
    cfg = _cfg_from(z, "cfg1")
    cfg["zero_rel"] = None
    b = cores(z, "cfg1_b")
    frame = O.solver_frame(b, cfg, seed=1)
    x, rep = O.sgmres(cores(z, "cfg1_op"), b, cfg, factors(z, "cfg1"), frame=frame)
    assert rep["iterations"] == int(z["cfg1_iters"])
    assert rep["basis_rank"] == list(z["cfg1_ranks"])
    np.testing.assert_allclose(rep["res_sketched"], z["cfg1_res"], rtol=1e-8)
    probe = O.kr_apply(O.kr_factors_new([c.shape[1] for c in x], 24, seed=777), x)
    want = z["cfg1_xprobe"]
    assert np.linalg.norm(probe - want) <= 1e-8 * np.linalg.norm(want)


def test_kr_config4_golden():
    """BASELINE config 4 vectors 0 and 1 (s=512, d=20, n=64, r=100) against the
    reference kr_apply(KhatriRaoSketch(F), v) (sketch.py:50-70)."""
    from paper_2409_09471_b200 import configs
    z = load("kr_cfg4.npz")
    C = configs.config4(nvec=2)
    for i in (0, 1):
        want = z[f"kr4_y{i}"]
        got = O.kr_apply(C["factors"], C["vecs"][i])
        assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)


def test_solver_cfg5_rhs1_golden():
    """BASELINE config 5 (d=50, n=256, maxit 60, ell 3, cap 100), RHS 1 (16
    iterations, ~30 s): the oracle TT-SVD solve against the reference's run."""
    from paper_2409_09471_b200 import configs
    z = load("solver_cfg5.npz")
    C = configs.config5(1)
    cfg = dict(C["cfg"], zero_rel=None, oversampling=20)
    f = O.kr_factors_new(C["dims"], cfg["sketch_rows"], seed=C["sketch_seed"])
    x, rep = O.sgmres(C["op"], C["b"], cfg, f, frame=O.solver_frame(C["b"], cfg, seed=C["frame_seed"]))
    assert rep["iterations"] == int(z["cfg5_1_iters"])
    assert rep["basis_rank"] == [int(r) for r in z["cfg5_1_ranks"]]
    np.testing.assert_allclose(rep["res_sketched"], z["cfg5_1_res"], rtol=1e-8)
    probe = O.kr_apply(O.kr_factors_new(C["dims"], 24, seed=777), x)
    want = z["cfg5_1_xprobe"]
    assert np.linalg.norm(probe - want) <= 1e-8 * np.linalg.norm(want)


def test_oracle_rto_exactness_kat():
    """Pins the RTO restatement (no reference implementation exists): with
    sketch rank >= true rank the randomized rounding is exact."""
    dims = [6, 6, 6, 6, 6]
    x = O.tt_random(dims, [3, 5, 4, 2], seed=11)
    big = O.add(x, O.scale(x, 0.25))
    drm = O.drm_new(dims, [7, 7, 7, 7], seed=5)
    ls = O.rto_ranks(dims, [1] + [c.shape[2] for c in big], [7, 7, 7, 7])
    out = O.rto_sweeps(big, O.slice_drm(drm, ls))
    assert O.rel_diff(out, O.scale(x, 1.25)) <= 1e-12
    r = O.rto_round(big, O.slice_drm(drm, ls), 1e-12)
    assert [c.shape[2] for c in r][:-1] == [c.shape[2] for c in x][:-1]
    assert O.rel_diff(r, O.scale(x, 1.25)) <= 1e-12


def test_oracle_truncate_left_orth_matches_tt_round_when_exact():
    """On a left-orthogonal input the right-to-left truncation and the
    reference-order TT-SVD agree whenever the discarded mass is ~0, and both
    honour the rel_tol contract otherwise."""
    dims = [5, 6, 4, 5]
    a = O.tt_random(dims, [4, 6, 4], seed=1)
    x = O.add(a, O.scale(a, 2.0))
    lo = O.rto_sweeps(x, O.drm_new(dims, [5, 12, 5], seed=2))  # left-orthogonal, exact (rank 4,6,4 <= 5,12,5)
    t1 = O.truncate_left_orth(lo, 1e-12)
    t2 = O.tt_round(lo, 1e-12, zero_rel=None)
    assert [c.shape for c in t1] == [c.shape for c in t2]
    assert O.rel_diff(t1, t2) <= 1e-12
    for tol in (1e-1, 1e-2):
        t = O.truncate_left_orth(lo, tol)
        assert O.rel_diff(t, lo) <= tol


def test_oracle_rto_dense_randomized_svd():
    """At the first cut RTO's core spans range(X_(1) G_(1)^T): the randomized
    range finder on the dense unfolding with the DRM's right interface."""
    dims = [5, 6, 4]
    x = O.tt_random(dims, [5, 4], seed=3)
    drm = O.slice_drm(O.drm_new(dims, [3, 2], seed=4), O.rto_ranks(dims, [1, 5, 4, 1], [3, 2]))
    out = O.rto_sweeps(x, drm)
    full = O.to_dense(x).reshape(5, -1)
    gr = np.tensordot(drm[1], drm[2], axes=([2], [0]))[:, :, :, 0]  # (l1, n1, n2)
    y = full @ gr.reshape(gr.shape[0], -1).T
    q = out[0].reshape(5, -1)
    assert np.abs(q.T @ q - np.eye(q.shape[1])).max() <= 1e-14
    assert np.linalg.norm(y - q @ (q.T @ y)) <= 1e-13 * np.linalg.norm(y)
