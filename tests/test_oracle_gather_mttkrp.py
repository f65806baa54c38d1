"""Pins for the oracle's summary gather and MTTKRP."""
import numpy as np

from oracle import sambaten as O


def _rand_dense(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape).astype(np.float32)


def test_gather_coordinate_lookup():
    T = _rand_dense((9, 8, 7), 0)          # K, J, I
    Is, Js, Ks = np.array([0, 3, 6]), np.array([1, 2, 7]), np.array([0, 4])
    Kp = O.k_prime(Ks, 6, 3)
    assert list(Kp) == [0, 4, 6, 7, 8]
    Y = O.gather_dense(T, Is, Js, Kp)
    assert Y.shape == (3, 3, 5) and Y.dtype == np.float32
    for p, i in enumerate(Is):
        for q, j in enumerate(Js):
            for u, k in enumerate(Kp):
                assert Y[p, q, u] == T[k, j, i]


def test_gather_full_sets_identity_and_coo_agrees():
    T = _rand_dense((5, 4, 3), 1)
    T[np.random.default_rng(2).random(T.shape) < 0.5] = 0
    Y = O.gather_dense(T, np.arange(3), np.arange(4), np.arange(5))
    assert np.array_equal(Y, O.view_ijk(T))
    kk, jj, ii = np.nonzero(T)
    X = O.coo_canonical(ii, jj, kk, T[kk, jj, ii], (3, 4, 5))
    Is, Js, Kp = np.array([0, 2]), np.array([1, 3]), np.array([0, 3, 4])
    Yc = O.gather_coo(X, Is, Js, Kp)
    Yd = O.gather_dense(T, Is, Js, Kp)
    D = np.zeros(Yd.shape, np.float32)
    D[Yc.i, Yc.j, Yc.k] = Yc.v
    assert np.array_equal(D, Yd)
    lin = (Yc.k * 2 + Yc.j) * 2 + Yc.i
    assert np.all(np.diff(lin) > 0)          # canonical (k, j, i)


def test_mttkrp_all_ones_and_zero():
    """2x2x2 all ones with all-ones 2x1 factors -> column (4, 4); S:52 zero tensor."""
    Y = np.ones((2, 2, 2))
    U = [np.ones((2, 1))] * 3
    for m in range(3):
        assert np.array_equal(O.mttkrp(Y, U, m), [[4.0], [4.0]])
        assert np.array_equal(O.mttkrp(np.zeros((2, 2, 2)), U, m), np.zeros((2, 1)))


def test_mttkrp_cp_closed_form():
    """For Y = [[lam; A, B, C]]: M_0(Y; B', C') = A diag(lam) ((B^T B') * (C^T C')), etc."""
    rng = np.random.default_rng(3)
    I, J, K, R, R2 = 7, 6, 5, 3, 4
    A, B, C = rng.standard_normal((I, R)), rng.standard_normal((J, R)), rng.standard_normal((K, R))
    lam = rng.random(R) + 0.5
    Y = np.einsum("f,if,jf,kf->ijk", lam, A, B, C)
    P = [rng.standard_normal((n, R2)) for n in (I, J, K)]
    exp0 = (A * lam) @ ((B.T @ P[1]) * (C.T @ P[2]))
    exp1 = (B * lam) @ ((A.T @ P[0]) * (C.T @ P[2]))
    exp2 = (C * lam) @ ((A.T @ P[0]) * (B.T @ P[1]))
    for m, e in enumerate((exp0, exp1, exp2)):
        assert np.allclose(O.mttkrp(Y, P, m), e, rtol=1e-12, atol=1e-12)


def test_mttkrp_modes_consistent_inner_product():
    """sum_{i,f} M_m(i,f) U_m(i,f) = <Y, [[U_0, U_1, U_2]]> for every mode (a transposed or
    mis-ordered operand in any mode breaks the equality)."""
    rng = np.random.default_rng(4)
    Y = rng.standard_normal((5, 4, 6))
    U = [rng.standard_normal((n, 3)) for n in Y.shape]
    vals = [float(np.sum(O.mttkrp(Y, U, m) * U[m])) for m in range(3)]
    assert np.allclose(vals, vals[0], rtol=1e-12)


def test_mttkrp_unfolding_khatri_rao():
    """Khatri-Rao Gram identity; MTTKRP equals a loop over stored entries."""
    rng = np.random.default_rng(5)
    a, b = rng.standard_normal((3, 2)), rng.standard_normal((4, 2))
    kr = O.khatri_rao(a, b)
    assert np.allclose(kr.T @ kr, (a.T @ a) * (b.T @ b), rtol=1e-12)
    assert np.array_equal(O.khatri_rao(np.eye(2), np.eye(2)), [[1, 0], [0, 0], [0, 0], [0, 1]])
    assert np.array_equal(O.khatri_rao(np.array([[1.0], [2.0]]), np.array([[3.0], [4.0]])).ravel(), [3, 4, 6, 8])
    Y = rng.standard_normal((3, 4, 5))
    U = [rng.standard_normal((n, 2)) for n in Y.shape]
    M = np.zeros((4, 2))
    for i in range(3):
        for j in range(4):
            for k in range(5):
                M[j] += Y[i, j, k] * U[0][i] * U[2][k]
    assert np.allclose(O.mttkrp(Y, U, 1), M, rtol=1e-12)


def test_mttkrp_coo_equals_dense():
    rng = np.random.default_rng(6)
    T = rng.standard_normal((6, 5, 4)).astype(np.float32)
    T[rng.random(T.shape) < 0.7] = 0
    kk, jj, ii = np.nonzero(T)
    X = O.coo_canonical(ii, jj, kk, T[kk, jj, ii], (4, 5, 6))
    U = [rng.standard_normal((n, 3)) for n in (4, 5, 6)]
    for m in range(3):
        assert np.allclose(O.mttkrp(X, U, m), O.mttkrp(O.view_ijk(T), U, m), rtol=1e-12, atol=1e-12)
