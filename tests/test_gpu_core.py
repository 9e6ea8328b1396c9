"""GPU parity of the exact-arithmetic kernels (matvec, axpy/concat, dot/norm,
Khatri-Rao sketch) against the golden fixtures and the CPU oracle."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2409_09471_b200 as T
from golden_io import cores, factors, load

pytestmark = pytest.mark.gpu


def to_np(v):
    return [c.cpu().numpy() for c in (v.cores if hasattr(v, "cores") else v)]


def assert_cores_close(got, want, rtol):
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g.shape == w.shape, (g.shape, w.shape)
        scale = max(np.abs(w).max(), 1e-300)
        err = np.abs(g - w).max()
        assert err <= rtol * scale, (err, scale)


@pytest.fixture(scope="module")
def ops():
    return load("tt_ops.npz")


def test_matvec_golden(cuda, ops):
    for name in ops["mv_names"]:
        a = T.TTOperator(cores(ops, f"{name}_op"), device=cuda)
        x = T.TTVector(cores(ops, f"{name}_x"), device=cuda)
        y = T.tt_matvec(a, x)
        assert_cores_close(to_np(y), cores(ops, f"{name}_y"), 1e-13)


@pytest.mark.parametrize("rho,r,n,m,d", [(3, 64, 128, 128, 4), (2, 20, 256, 256, 3), (1, 7, 5, 9, 5),
                                         (3, 100, 17, 13, 3), (2, 130, 33, 33, 3)])
def test_matvec_shapes_vs_oracle(cuda, rho, r, n, m, d):
    rng = np.random.default_rng(rho * 1000 + r)
    op = O.gaussian_tt  # noqa: F841
    full = [1] + [rho] * (d - 1) + [1]
    opc = [rng.standard_normal((full[k], m, n, full[k + 1])) for k in range(d)]
    xc = O.gaussian_tt([n] * d, [r] * (d - 1), rng, 1.0 / np.sqrt(n * r))
    y = T.tt_matvec(T.TTOperator(opc, device=cuda), T.TTVector(xc, device=cuda))
    assert_cores_close(to_np(y), O.matvec(opc, xc), 1e-13)


def test_matvec_config3_cores(cuda):
    """BASELINE config 3 shape: rho=3, r=64, n=128 (two interior cores checked against the oracle)."""
    rng = np.random.default_rng(0)
    opc = [rng.standard_normal((3, 128, 128, 3)) for _ in range(2)]
    xc = [rng.standard_normal((64, 128, 64)) / np.sqrt(128 * 64) for _ in range(2)]
    lib_out = []
    for k in range(2):
        # embed each interior core in a d=3 chain with trivial boundaries
        a = T.TTOperator([np.ones((1, 1, 1, 3)), opc[k], np.ones((3, 1, 1, 1))], device=cuda)
        x = T.TTVector([np.ones((1, 1, 64)), xc[k], np.ones((64, 1, 1))], device=cuda)
        lib_out.append(T.tt_matvec(a, x).cores[1].cpu().numpy())
    want = O.matvec(opc, xc)
    assert_cores_close(lib_out, want, 1e-13)


def _banded_op(rng, d, n, rho, w, kinds):
    """Operator cores whose blocks are zero / scaled identity / random band-w matrices."""
    full = [1] + [rho] * (d - 1) + [1]
    out = []
    for k in range(d):
        c = np.zeros((full[k], n, n, full[k + 1]))
        for al in range(full[k]):
            for be in range(full[k + 1]):
                kind = kinds[(k + al + be) % len(kinds)]
                if kind == "eye":
                    c[al, :, :, be] = rng.standard_normal() * np.eye(n)
                elif kind == "band":
                    m = rng.standard_normal((n, n))
                    c[al, :, :, be] = np.triu(np.tril(m, w), -w)
        out.append(c)
    return out


@pytest.mark.parametrize("d,n,rho,r,w", [(5, 16, 3, 12, 1), (4, 33, 2, 40, 2), (6, 8, 1, 5, 0),
                                         (3, 128, 3, 64, 1), (4, 7, 2, 9, 2)])
def test_matvec_structured_vs_dense_and_oracle(cuda, d, n, rho, r, w):
    """Banded-block operators: the structure-aware kernel equals
    the dense DMMA path and the oracle; config-3's explicit operator is banded."""
    rng = np.random.default_rng(d * 100 + n + w)
    opc = _banded_op(rng, d, n, rho, w, ["eye", "band", "zero", "band"])
    xc = O.gaussian_tt([n] * d, [r] * (d - 1), rng, 1.0 / np.sqrt(n * r))
    a, x = T.TTOperator(opc, device=cuda), T.TTVector(xc, device=cuda)
    bt = a.band_tables()
    assert bt is not None and bt[0] <= w
    ys = T.tt_matvec(a, x, structured=True)
    assert_cores_close(to_np(ys), O.matvec(opc, xc), 1e-13)
    assert_cores_close(to_np(ys), to_np(T.tt_matvec(a, x)), 1e-13)


def test_matvec_structured_config3_operator_and_fallback(cuda):
    from paper_2409_09471_b200 import configs
    opc = configs.config3_operator(d=6, n=32, seed=0)
    rng = np.random.default_rng(1)
    xc = O.gaussian_tt([32] * 6, [10] * 5, rng, 0.1)
    a, x = T.TTOperator(opc, device=cuda), T.TTVector(xc, device=cuda)
    assert a.band_tables()[0] == 1
    assert_cores_close(to_np(T.tt_matvec(a, x, structured=True)), O.matvec(opc, xc), 1e-13)
    # a dense block: band_tables() is None and structured=True takes the DMMA path
    opc[2][0, :, :, 1] = rng.standard_normal((32, 32))
    a2 = T.TTOperator(opc, device=cuda)
    assert a2.band_tables() is None
    assert_cores_close(to_np(T.tt_matvec(a2, x, structured=True)), O.matvec(opc, xc), 1e-13)
    # rectangular cores are never banded
    a3 = T.TTOperator([np.ones((1, 3, 4, 1))], device=cuda)
    assert a3.band_tables() is None


@pytest.mark.parametrize("d,n,m,rho,r,S", [(4, 16, 12, 2, 5, 40), (5, 32, 32, 3, 20, 120), (3, 7, 9, 1, 3, 11),
                                            (6, 64, 64, 2, 40, 80)])
def test_kr_apply_matvec_fused_vs_unfused(cuda, d, n, m, rho, r, S):
    """Fused matvec -> sketch equals sketching the materialised
    matvec output, and the oracle's sketch of the oracle matvec."""
    rng = np.random.default_rng(d * 31 + n + S)
    full = [1] + [rho] * (d - 1) + [1]
    opc = [rng.standard_normal((full[k], m, n, full[k + 1])) for k in range(d)]
    xc = O.gaussian_tt([n] * d, [r] * (d - 1), rng, 1.0 / np.sqrt(n * r))
    fs = [rng.standard_normal((S, m)) / np.sqrt(m) for _ in range(d)]
    a, x = T.TTOperator(opc, device=cuda), T.TTVector(xc, device=cuda)
    sk = T.KhatriRaoSketch(fs, device=cuda)
    got = T.kr_apply_matvec(sk, a, x)
    want = T.kr_apply(sk, T.tt_matvec(a, x))
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= 1e-12 * scale
    assert np.abs(got - O.kr_apply(fs, O.matvec(opc, xc))).max() <= 1e-12 * scale
    # the cached premultiplied factors are reused for a second vector
    x2 = T.TTVector(O.gaussian_tt([n] * d, [r] * (d - 1), rng, 1.0), device=cuda)
    w2 = T.kr_apply(sk, T.tt_matvec(a, x2))
    assert np.abs(T.kr_apply_matvec(sk, a, x2) - w2).max() <= 1e-12 * np.abs(w2).max()
    with pytest.raises(T.ShapeMismatch):
        T.kr_apply_matvec(T.KhatriRaoSketch([f[:, :5] for f in fs], device=cuda), a, x)


def test_add_scale_combine_golden(cuda, ops):
    a = T.TTVector(cores(ops, "add_a"), device=cuda)
    b = T.TTVector(cores(ops, "add_b"), device=cuda)
    assert_cores_close(to_np(T.tt_add(a, b)), cores(ops, "add_y"), 0)
    a1 = T.TTVector(cores(ops, "add1_a"), device=cuda)
    b1 = T.TTVector(cores(ops, "add1_b"), device=cuda)
    assert_cores_close(to_np(T.tt_add(a1, b1)), cores(ops, "add1_y"), 0)
    s = T.TTVector(cores(ops, "scale_a"), device=cuda)
    assert_cores_close(to_np(T.tt_scale(s, -2.5)), cores(ops, "scale_y"), 0)
    h = ops["axpy_h"]
    terms = [T.TTVector(cores(ops, n), device=cuda) for n in ("axpy_vt", "axpy_v1", "axpy_v2")]
    y = T.tt_combine(terms, [1.0, -h[0], -h[1]])
    # bit-exact with the reference's chained tt_add(tt_scale(.)) (same single multiply per entry)
    assert_cores_close(to_np(y), cores(ops, "axpy_y"), 0)


def test_combine_many_terms_vs_oracle(cuda):
    rng = np.random.default_rng(5)
    dims = [6, 7, 5, 8, 4]
    terms = [O.tt_random(dims, list(rng.integers(1, 9, size=4)), seed=50 + t) for t in range(20)]
    coeffs = [1.0] + list(rng.standard_normal(19))
    y = T.tt_combine([T.TTVector(t, device=cuda) for t in terms], coeffs)
    want = O.concat_axpy(terms, coeffs)
    assert_cores_close(to_np(y), want, 1e-15)


def test_dot_norm_golden(cuda, ops):
    a = T.TTVector(cores(ops, "dot_a"), device=cuda)
    b = T.TTVector(cores(ops, "dot_b"), device=cuda)
    assert T.tt_dot(a, b) == pytest.approx(float(ops["dot_ab"]), rel=1e-13)
    n = T.TTVector(cores(ops, "norm_a"), device=cuda)
    assert T.tt_norm(n) == pytest.approx(float(ops["norm_a_val"]), rel=1e-13)
    assert T.tt_norm(T.tt_zero([3, 3, 3], device=cuda)) == 0.0


def test_dots_batched_vs_oracle(cuda):
    dims = [32, 16, 40, 24, 32, 8]
    x = O.tt_random(dims, [30, 60, 45, 50, 7], seed=1)
    ys = [O.tt_random(dims, [r] * 5, seed=10 + r) for r in (1, 5, 20, 33)]
    got = T.tt_dots(T.TTVector(x, device=cuda), [T.TTVector(y, device=cuda) for y in ys]).cpu().numpy()
    want = np.array([O.dot(x, y) for y in ys])
    nx = O.norm(x)
    for g, w, y in zip(got, want, ys):
        assert abs(g - w) <= 1e-12 * nx * O.norm(y)


def test_kr_golden(cuda):
    z = load("sketch.npz")
    for name in z["kr_names"]:
        s = T.KhatriRaoSketch(factors(z, name), device=cuda)
        v = T.TTVector(cores(z, f"{name}_x"), device=cuda)
        y = T.kr_apply(s, v)
        want = z[f"{name}_y"]
        assert np.linalg.norm(y - want) <= 1e-12 * max(np.linalg.norm(want), 1.0)


@pytest.mark.parametrize("path", [0, 1])
def test_kr_paths_vs_oracle(cuda, path):
    """Fused and two-phase kernels agree with the oracle (rows split and odd sizes)."""
    from paper_2409_09471_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(3)
    dims = [7, 64, 13, 32, 5]
    fs = [rng.normal(0, 1 / np.sqrt(n), size=(300, n)) for n in dims]
    vs = [O.tt_random(dims, [5, 60, 100, 3], seed=70 + i) for i in range(3)]
    s = T.KhatriRaoSketch(fs, device=cuda)
    tv = [T.TTVector(v, device=cuda) for v in vs]
    lo, hi = 37, 291
    out = torch.empty((3, hi - lo), dtype=torch.float64, device=cuda)
    ranks = _lib.int_array([r for v in tv for r in v.ranks])
    n = _lib.int_array(dims)
    nbytes = lib.ttk_kr_sketch_ws_bytes(len(dims), n, 0, 300, 3, ranks) + (1 << 26)
    ws = _lib.workspace(nbytes, cuda)
    _lib.check(lib.ttk_kr_sketch_path(path, len(dims), n, lo, hi, _lib.ptr_array(s.factors), 3, ranks,
                                      _lib.ptr_array([c for v in tv for c in v.cores]), out.data_ptr(),
                                      ws.data_ptr(), ws.numel(), _lib.stream_ptr(cuda)))
    got = out.cpu().numpy()
    for i, v in enumerate(vs):
        want = O.kr_apply([f[lo:hi] for f in fs], v)
        assert np.linalg.norm(got[i] - want) <= 1e-12 * np.linalg.norm(want)


def test_kr_linearity_and_batch(cuda):
    s = T.kr_sketch_new([3, 3, 3], 9, seed=11, device=cuda)
    a = T.tt_random([3, 3, 3], [2, 2], seed=12, device=cuda)
    b = T.tt_random([3, 3, 3], [2, 3], seed=13, device=cuda)
    lhs = T.kr_apply(s, T.tt_add(a, b))
    rhs = T.kr_apply(s, a) + T.kr_apply(s, b)
    assert np.allclose(lhs, rhs, atol=1e-12 * max(1.0, np.linalg.norm(rhs)))
    batch = T.kr_apply_batch(s, [a, b]).cpu().numpy()
    assert np.array_equal(batch[0], T.kr_apply(s, a)) or np.allclose(batch[0], T.kr_apply(s, a), rtol=1e-14)
