"""Host-side logic of the product package (no GPU needed): validation,
error mapping, rank rules and constructors."""

import numpy as np
import pytest
import torch

import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import ShapeMismatch


def test_roundspec_validation():
    with pytest.raises(ValueError):
        T.RoundSpec(-1.0)
    with pytest.raises(ValueError):
        T.RoundSpec(0.1, 0)
    assert T.RoundSpec(0.1, 3).max_rank == 3


def test_ttvector_validation_cpu():
    with pytest.raises(ShapeMismatch):
        T.TTVector([np.zeros((2, 3, 1))], device="cpu")
    with pytest.raises(ShapeMismatch):
        T.TTVector([np.zeros((1, 3, 2)), np.zeros((3, 3, 1))], device="cpu")
    with pytest.raises(ShapeMismatch):
        T.TTVector([np.zeros((1, 3))], device="cpu")
    with pytest.raises(ValueError):
        T.TTVector([], device="cpu")
    v = T.TTVector([np.zeros((1, 3, 2)), np.zeros((2, 4, 1))], device="cpu")
    assert v.dims == (3, 4) and v.ranks == (1, 2, 1) and v.d == 2


def test_ttoperator_validation_cpu():
    with pytest.raises(ShapeMismatch):
        T.TTOperator([np.zeros((1, 2, 2, 2))], device="cpu")
    a = T.kron_sum_operator([np.eye(3)] * 4, device="cpu")
    assert a.ranks == (1, 2, 2, 2, 1)
    with pytest.raises(ShapeMismatch):
        T.kron_sum_operator([np.zeros((2, 3))], device="cpu")


def test_shape_errors_raise_before_any_launch():
    a = T.identity_operator([2, 2], device="cpu")
    with pytest.raises(ShapeMismatch):
        T.tt_matvec(a, T.TTVector([np.zeros((1, 2, 1)), np.zeros((1, 3, 1))], device="cpu"))
    with pytest.raises(ShapeMismatch):
        T.tt_add(T.TTVector([np.zeros((1, 2, 1))] * 2, device="cpu"),
                 T.TTVector([np.zeros((1, 2, 1)), np.zeros((1, 3, 1))], device="cpu"))


def test_no_cpu_fallback():
    """Compute entry points refuse CPU tensors instead of silently falling back."""
    v = T.tt_random([3, 3], [2], seed=0, device="cpu")
    with pytest.raises(RuntimeError):
        T.tt_matvec(T.identity_operator([3, 3], device="cpu"), v)
    with pytest.raises(RuntimeError):
        T.tt_dot(v, v)


def test_tt_random_matches_reference_draws():
    import oracle as O
    v = T.tt_random([4, 5, 3], [3, 9], seed=7, device="cpu")
    ref = O.tt_random([4, 5, 3], [3, 9], seed=7)
    assert v.ranks == (1, 3, 3, 1)  # 9 clipped to the right unfolding size 3
    for a, b in zip(v.numpy(), ref):
        assert np.array_equal(a, b)


def test_attainable_ranks_no_overflow():
    # quirk Q2: the reference's int64 cumprod overflows at d=32, n=128
    r = T.attainable_ranks([128] * 32, [64] * 31)
    assert r == [64] * 31


def test_kr_sketch_factor_law():
    s = T.kr_sketch_new([50, 50], 200, seed=5, device="cpu")
    var = 200.0 ** (-1.0 / 2)
    assert abs(float(s.factors[0].var()) - var) <= 0.1 * var
    with pytest.raises(ValueError):
        T.kr_sketch_new([2], 0)
