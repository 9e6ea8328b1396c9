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
        np.testing.assert_allclose(rep["res_sketched"], z[f"{name}_res"], rtol=1e-6)
        probe = O.kr_apply(O.kr_factors_new([c.shape[1] for c in x], 24, seed=777), x)
        want = z[f"{name}_xprobe"]
        assert np.linalg.norm(probe - want) <= 1e-7 * np.linalg.norm(want)


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
