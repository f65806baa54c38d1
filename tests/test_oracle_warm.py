"""Pins of the warm-started summary ALS (reading R34 in DESIGN.md).

A noiseless planted tensor whose new slices are zero has an exact CP model on every summary:
U_0 = A(I_s), U_1 = B(J_s), U_2 = [C(K_s) diag(lambda); 0].  Started from the model's rows (new
rows of U_2 at zero), that point is a fixed point of the ALS sweep, so the summary fit is 1 to
rounding of the fp32 data after ONE iteration; a cold start is far from it.  A wrong row set, a transposed factor or a missing lambda breaks this.
"""
import numpy as np
import pytest

from oracle import sambaten as O


def _stream(seed, I=30, J=28, K0=20, Kn=4, R=3):
    rng = np.random.default_rng(seed)
    A, B, C = rng.random((I, R)), rng.random((J, R)), rng.random((K0, R))
    lam = rng.random(R) + 0.5
    A, B, C, lam = (np.asarray(x, np.float32).astype(np.float64) for x in (A, B, C, lam))
    X0 = np.einsum("if,jf,kf,f->kji", A, B, C, lam).astype(np.float32)
    batch = np.zeros((Kn, J, I), np.float32)
    return X0, batch, (lam, A, B, C)


@pytest.mark.parametrize("seed", [0, 1])
def test_warm_start_is_exact_after_one_sweep(seed):
    X0, batch, model = _stream(seed)
    fits = {}
    for warm in (False, True):
        cfg = O.Config(R=3, s=(2, 2, 2), r=2, seed=seed + 5, maxit=1, tol=0.0, tau=0.0, warm_start=warm)
        st = O.init_factors(X0, cfg, *model, X0.size * 2)
        last = O.update(st, batch)
        fits[warm] = [rp["fit"] for rp in last["reps"]]
    assert min(fits[True]) > 1.0 - 1e-6, fits   # the data is the exact model rounded to fp32 (<= 6e-8 relative)
    assert max(fits[False]) < 0.99, fits


def test_warm_init_rows():
    """The initial point itself: model rows of the sampled indices, lambda on U_2's old rows,
    zero rows for the new slices."""
    X0, batch, model = _stream(3)
    cfg = O.Config(R=3, s=(2, 2, 2), r=1, seed=9, maxit=1, tol=0.0, tau=0.0, warm_start=True)
    st = O.init_factors(X0, cfg, *model, X0.size * 2)
    Is, Js, Ks = np.array([1, 4, 7]), np.array([0, 2]), np.array([3, 5])
    cold = O.als_init((3, 2, 2 + 4), 3, 9, 1, 0)
    U = O.warm_init(cold, st, Is, Js, Ks)
    lam, A, B, C = model
    assert np.array_equal(U[0], A[Is]) and np.array_equal(U[1], B[Js])
    assert np.allclose(U[2][:2], C[Ks] * lam[None, :], rtol=1e-7)
    assert np.all(U[2][2:] == 0.0)
