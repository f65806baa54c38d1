"""Pins of the GetRank oracle (Alg. 2; readings R29-R31 in DESIGN.md).

* CorConDia of an exact CP tensor with its own (scaled, permuted) factors is 100 (closed form:
  the least-squares core is the superdiagonal unit core).
* The mode-product core equals the brute-force Kronecker solution vec(G) = pinv(C (x) B (x) A') vec(X)
  (a different computation of the same least-squares problem).
* A perturbed core lowers the rating by exactly sum (dG)^2 / F (the definition's quadratic form).
* A converged rank-1 ALS model rates 100 (R31's reason for the threshold rule).
* GetRank recovers the planted rank of noiseless rank-2 / rank-3 tensors (threshold 90).
"""
import numpy as np
import pytest

from oracle import getrank as GR
from oracle import sambaten as O


def _cp(A, B, C, lam=None):
    lam = np.ones(A.shape[1]) if lam is None else lam
    return np.einsum("if,jf,kf,f->ijk", A, B, C, lam)


def test_corcondia_exact_model_is_100():
    rng = np.random.default_rng(0)
    for F in (1, 2, 3, 5):
        A, B, C = rng.random((9, F)), rng.random((8, F)), rng.random((7, F))
        lam = rng.random(F) + 0.5
        Y = _cp(A, B, C, lam)
        assert abs(GR.corcondia(Y, lam, A, B, C) - 100.0) < 1e-8
        # column scaling moved between the factors and a column permutation do not change it
        p = rng.permutation(F)
        s = rng.random(F) + 0.5
        assert abs(GR.corcondia(Y, lam[p] * s[p], A[:, p] / s[p], B[:, p], C[:, p]) - 100.0) < 1e-8


def test_core_equals_kronecker_least_squares():
    rng = np.random.default_rng(1)
    F = 3
    Y = rng.standard_normal((6, 5, 4))
    A, B, C = rng.standard_normal((6, F)), rng.standard_normal((5, F)), rng.standard_normal((4, F))
    lam = rng.random(F) + 0.5
    G = GR.tucker_core(Y, lam, A, B, C)
    A1 = A * lam[None, :]
    # vec with i fastest: X[i, j, k] -> index i + 6 (j + 5 k); the Kronecker C (x) B (x) A' matches
    K = np.kron(C, np.kron(B, A1))
    g = np.linalg.lstsq(K, Y.reshape(-1, order="F"), rcond=None)[0]
    assert np.allclose(G.reshape(-1, order="F"), g, atol=1e-10)


def test_corcondia_is_the_core_deviation_quadratic_form():
    rng = np.random.default_rng(2)
    F = 3
    A, B, C = rng.random((7, F)), rng.random((6, F)), rng.random((5, F))
    dG = 0.05 * rng.standard_normal((F, F, F))
    core = GR.superdiagonal(F) + dG
    Y = np.einsum("fgh,if,jg,kh->ijk", core, A, B, C)
    assert abs(GR.corcondia(Y, np.ones(F), A, B, C) - 100.0 * (1 - np.sum(dG ** 2) / F)) < 1e-8


def test_rank1_als_model_rates_100():
    rng = np.random.default_rng(3)
    Y = rng.random((8, 7, 6))
    U0 = O.als_init(Y.shape, 1, 5, GR.GETRANK_ID + 1, 0)
    lam, U, _, _, _ = O.cp_als(Y, U0, 200, 1e-14)
    assert abs(GR.corcondia(Y, lam, *U) - 100.0) < 1e-6


@pytest.mark.parametrize("F,seed", [(2, 0), (3, 1)])
def test_getrank_recovers_planted_rank(F, seed):
    rng = np.random.default_rng(seed)
    A, B, C = rng.random((12, F)), rng.random((11, F)), rng.random((10, F))
    Y = _cp(A, B, C)
    R_new, cc = GR.getrank(Y, 4, 2, 7, 300, 1e-12)
    assert R_new == F, cc
    assert cc[F - 1].max() > 99.0
