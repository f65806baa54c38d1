"""Pins for the oracle's fixed-point measure of importance (Eq. 1; readings R1-R3, R7)."""
import numpy as np
import pytest

from oracle import sambaten as O


def test_ceil_log2_and_scale():
    assert [O.ceil_log2(v) for v in (1, 2, 3, 4, 5, 0.5, 0.75, 2 ** -10)] == [0, 1, 2, 2, 3, -1, 0, -10]
    # C1 cap 1.25e5, max |x| ~3 -> S = 62 - 17 - 2 - 8 = 35
    assert O.fixed_point_scale(125_000, 3.0) == 35
    # C4: cap 2.7e10 (ceil log2 = 35), max |x| ~10 (4) -> 15
    assert O.fixed_point_scale(3000 ** 3, 10.0) == 15
    with pytest.raises(ValueError):
        O.fixed_point_scale(10, 0.0)


def test_all_ones_example():
    """2x2x2 all-ones tensor -> (4, 4) per mode, here scaled by 2**S."""
    T = np.ones((2, 2, 2), np.float32)
    for moi in (O.MOI_ABS, O.MOI_SQ):
        x1, x2, x3 = O.marginals_dense(T, 10, moi)
        for x in (x1, x2, x3):
            assert list(x) == [4 * 2 ** 10, 4 * 2 ** 10]


def test_brute_force_triple_loop():
    rng = np.random.default_rng(0)
    T = rng.standard_normal((4, 5, 6)).astype(np.float32)
    S = 20
    x1, x2, x3 = O.marginals_dense(T, S, O.MOI_ABS)
    b1 = np.zeros(6, np.int64); b2 = np.zeros(5, np.int64); b3 = np.zeros(4, np.int64)
    for k in range(4):
        for j in range(5):
            for i in range(6):
                q = int(round(abs(float(T[k, j, i])) * 2 ** S))   # python round: half-even
                b1[i] += q; b2[j] += q; b3[k] += q
    assert np.array_equal(x1, b1) and np.array_equal(x2, b2) and np.array_equal(x3, b3)


def test_totals_equal_norms():
    """sum x_1 = sum x_2 = sum x_3 exactly; sum * 2**-S ~ ||X||_1 (|x|) or ||X||_F^2 (x^2)
    within N * 2**-(S+1)."""
    rng = np.random.default_rng(1)
    T = rng.standard_normal((7, 9, 11)).astype(np.float32)
    N = T.size
    for moi, ref in ((O.MOI_ABS, np.abs(T.astype(np.float64)).sum()),
                     (O.MOI_SQ, (T.astype(np.float64) ** 2).sum())):
        S = 30
        x1, x2, x3 = O.marginals_dense(T, S, moi)
        assert x1.sum() == x2.sum() == x3.sum()
        assert abs(x1.sum() * 2.0 ** -S - ref) <= N * 2.0 ** -(S + 1)


def test_closed_form_planted_nonnegative():
    """For X = [[lam; A, B, C]] with nonnegative factors: x_1(i) = sum_f lam_f A(i,f)
    (sum_j B(j,f)) (sum_k C(k,f)) up to quantisation (|x| = x)."""
    rng = np.random.default_rng(2)
    I, J, K, R = 8, 7, 6, 3
    A, B, C = rng.random((I, R)), rng.random((J, R)), rng.random((K, R))
    lam = np.array([1.0, 2.0, 0.5])
    T = np.einsum("f,if,jf,kf->kji", lam, A, B, C).astype(np.float32)
    S = 40
    x1, x2, x3 = O.marginals_dense(T, S, O.MOI_ABS)
    c1 = (A * lam) @ (B.sum(0) * C.sum(0))
    c2 = (B * lam) @ (A.sum(0) * C.sum(0))
    c3 = (C * lam) @ (A.sum(0) * B.sum(0))
    # float32 rounding of the entries dominates: each entry within 2**-24 relative
    for x, c, n in ((x1, c1, J * K), (x2, c2, I * K), (x3, c3, I * J)):
        assert np.allclose(x * 2.0 ** -S, c, rtol=2e-7 * 4, atol=n * 2.0 ** -S)


def test_coo_equals_dense_and_append_is_additive():
    rng = np.random.default_rng(3)
    T = rng.standard_normal((5, 6, 7)).astype(np.float32)
    T[rng.random(T.shape) < 0.6] = 0
    I, J, K = 7, 6, 5
    kk, jj, ii = np.nonzero(T)
    X = O.coo_canonical(ii, jj, kk, T[kk, jj, ii], (I, J, K))
    S = 25
    d = O.marginals_dense(T, S)
    c = O.marginals_coo(X, S)
    for a, b in zip(d, c):
        assert np.array_equal(a, b)
    # incremental = full recompute (integer associativity), modes 1 and 2
    a1, a2, a3 = O.marginals_dense(T[:3], S)
    b1, b2, b3 = O.marginals_dense(T[3:], S)
    assert np.array_equal(a1 + b1, d[0]) and np.array_equal(a2 + b2, d[1])
    assert np.array_equal(np.concatenate([a3, b3]), d[2])


def test_half_even_rounding():
    # 0.5 * 2**0 -> 0, 1.5 -> 2, 2.5 -> 2 (round half to even)
    T = np.array([[[0.5, 1.5, 2.5]]], np.float32)
    x1, _, _ = O.marginals_dense(T, 0)
    assert list(x1) == [0, 2, 2]
