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


def _stream(F_true, R, seed, I=40, J=36, K=30, K0=24, noise=0.0):
    """Planted tensor of rank F_true; the model carries R >= F_true components (the extra ones
    with all-zero time factors, i.e. absent from the data)."""
    rng = np.random.default_rng(seed)
    A, B, C = rng.random((I, R)), rng.random((J, R)), rng.random((K, R))
    C[:, F_true:] = 0.0
    X = np.einsum("if,jf,kf->ijk", A, B, C)
    T = np.ascontiguousarray(np.transpose(X, (2, 1, 0))).astype(np.float32)
    return T[:K0], T[K0:], (np.ones(R), A, B, C[:K0])


def test_update_with_getrank_equals_plain_update_when_full_rank():
    """GetRank finds the universal rank -> the update is the plain Alg. 1 update, bit for bit."""
    T0, batch, model = _stream(3, 3, 0)
    outs = []
    for gr in (False, True):
        cfg = O.Config(R=3, s=(2, 2, 2), r=3, seed=4, maxit=300, tol=1e-12, tau=0.0, getrank=gr)
        st = O.init_factors(T0, cfg, *model, T0.size * 2)
        last = O.update(st, batch)
        if gr:
            assert all(rp["rank"] == 3 for rp in last["reps"])
        outs.append((st.lam.copy(), st.A.copy(), st.B.copy(), st.C.copy()))
    for x, y in zip(*outs):
        assert np.array_equal(x, y)


def test_update_with_getrank_matches_only_the_present_components():
    """Rank-deficient update: the data has 2 of the model's 3 components; GetRank picks 2,
    only 2 candidate columns are matched, the third component keeps its lambda and gets zero
    time rows for the new slices."""
    T0, batch, model = _stream(2, 3, 1)
    cfg = O.Config(R=3, s=(2, 2, 2), r=3, seed=6, maxit=400, tol=1e-12, tau=0.0, getrank=True)
    st = O.init_factors(T0, cfg, *model, T0.size * 2)
    lam0 = st.lam.copy()
    last = O.update(st, batch)
    assert all(rp["rank"] == 2 for rp in last["reps"])
    for rp in last["reps"]:
        assert rp["match"].valid.sum() == 2 and not rp["match"].valid[2]
    assert st.lam[2] == lam0[2]
    Kn = batch.shape[0]
    assert np.all(st.C[-Kn:, 2] == 0.0)
    # the present components are recovered in the old frame (noiseless, model = truth with
    # lambda = 1): the new time rows equal the planted ones
    rng = np.random.default_rng(1)
    _, _, Ct = rng.random((40, 3)), rng.random((36, 3)), rng.random((30, 3))
    assert np.allclose(st.C[-Kn:, :2], Ct[-Kn:, :2], rtol=1e-3, atol=1e-6)


def test_corcondia_of_a_coo_tensor_is_that_of_its_densification():
    """The oracle rates a Coo through its densification: equal to the dense call on the same
    entries (pins the Coo branch), and an exact CP tensor stored as COO rates 100."""
    from oracle import sambaten as O
    rng = np.random.default_rng(5)
    A, B, C = rng.random((9, 2)), rng.random((8, 2)), rng.random((7, 2))
    Y = np.einsum("if,jf,kf->ijk", A, B, C).astype(np.float32).astype(np.float64)
    ii, jj, kk = np.nonzero(Y > -1)
    X = O.coo_canonical(ii, jj, kk, Y[ii, jj, kk].astype(np.float32), Y.shape)
    lam = np.ones(2)
    assert GR.corcondia(X, lam, A, B, C) == GR.corcondia(Y, lam, A, B, C)
    assert abs(GR.corcondia(X, lam, A, B, C) - 100.0) < 1e-4


def test_coo_update_with_getrank_equals_the_dense_one():
    """The same stream stored as a COO tensor (every entry): GetRank on the sparse summaries
    (cp_als on the Coo, CorConDia of the densified summary) gives the dense update's per-rep
    ranks and, to rounding, its merged model -- the COO handle's parity target (R33)."""
    T0, batch, model = _stream(2, 3, 1)

    def coo(T):
        kk, jj, ii = np.nonzero(T != 0.0)
        return O.coo_canonical(ii, jj, kk, T[kk, jj, ii], (T.shape[2], T.shape[1], T.shape[0]))

    cfg = O.Config(R=3, s=(2, 2, 2), r=3, seed=6, maxit=200, tol=1e-12, tau=0.0, getrank=True)
    sd = O.init_factors(T0, cfg, *model, T0.size * 2)
    ld = O.update(sd, batch)
    X0, Xb = coo(T0), coo(batch)
    sc = O.init_factors(X0, cfg, *model, (X0.nnz + Xb.nnz) * 2)
    lc = O.update(sc, Xb)
    assert [rp["rank"] for rp in lc["reps"]] == [rp["rank"] for rp in ld["reps"]] == [2, 2, 2]
    for a, b in zip((sc.lam, sc.A, sc.B, sc.C), (sd.lam, sd.A, sd.B, sd.C)):
        assert np.allclose(a, b, rtol=1e-8, atol=1e-10)
