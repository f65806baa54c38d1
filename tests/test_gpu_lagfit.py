"""The lag-1 fused fit (opts.full_fit = 2, SURVEY 8(f) NEXT #1 second half): update t+1's
marginal pass over the old slices also computes the relative error of the model
update t committed.  Checks, through the C-ABI, against the oracle and against the separate
a7 pass (full_fit = 1):
* the marginals, samples and committed models are bit-identical to full_fit = 1 (the fused
  kernel's integer sums equal the plain pass's);
* info.fit_full_prev of update t+1 equals the oracle's relative error of the GPU model of
  update t over X_t (and update 0's that of the initial model over X0) within 1e-6;
* both row layouts of the fused kernel (one column quad per thread, I <= 2048; two, I > 2048)
  and both measures of importance (|x|, x^2)."""
import numpy as np
import pytest

from oracle import sambaten as O
from synth import planted_dense, split_dense
from tests._helpers import dev

pytestmark = pytest.mark.gpu


def L():
    from paper_1709_00668_b200 import _lib
    return _lib


def _model_out(h, I, J, K, R):
    A = np.empty((I, R), np.float32); B = np.empty((J, R), np.float32)
    C = np.empty((K, R), np.float32); lam = np.empty(R, np.float32)
    L().sambaten_copy_factors(h, A, B, C, lam)
    return lam, A, B, C


@pytest.mark.parametrize("I,J,K0,bs,nb,R,moi", [(120, 96, 60, 6, 3, 5, 0),
                                                 (2400, 40, 24, 4, 2, 10, 0),
                                                 (200, 64, 40, 5, 2, 4, 1)])
def test_lag1_fit_parity(I, J, K0, bs, nb, R, moi):
    K = K0 + bs * nb
    T, truth = planted_dense(I, J, K, R, noise=0.01, seed=41)
    T0, batches = split_dense(T, K0, bs)
    model = [np.ascontiguousarray(np.asarray(x, np.float32)) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    hs = []
    for ff in (1, 2):
        opts = L().default_opts(als_max_iters=10, als_tol=0.0, accept_tau=0.0, capacity=K, full_fit=ff, moi=moi)
        hs.append(L().sambaten_init_factors(L().dense(dev(T0)), R, 2, 4, 3, model[1], model[2], model[3],
                                            model[0], opts))
    try:
        X = T0
        prev = tuple(np.asarray(x, np.float64) for x in model)
        Kt = K0
        for b in batches:
            infos = [L().sambaten_update(h, L().dense(dev(b))) for h in hs]
            # the previous model's fit over the tensor it was committed on
            rel_o = O.relative_error(X, *prev)
            assert infos[1].fit_full == -1.0
            assert abs((1.0 - infos[1].fit_full_prev) - rel_o) <= 1e-6, (infos[1].fit_full_prev, 1 - rel_o)
            Kt += b.shape[0]
            X = np.concatenate([X, b])
            m = [_model_out(h, I, J, Kt, R) for h in hs]
            for x, y in zip(*m):
                assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
            n = L().sambaten_last_samples(hs[0])
            s = [np.empty(4 * n[0], np.int32) for _ in hs]
            for h, a in zip(hs, s):
                L().sambaten_last_samples(h, a)
            assert np.array_equal(s[0], s[1])
            assert infos[0].fit_full_prev == -1.0
            prev = tuple(np.asarray(x, np.float64) for x in m[0])
            # the separate pass's value for this model is what the next fused pass must report
            assert abs((1.0 - infos[0].fit_full) - O.relative_error(X, *prev)) <= 1e-6
    finally:
        for h in hs:
            L().sambaten_destroy(h)


def test_lag1_falls_back_with_incremental_marginals():
    """full_fit = 2 with incremental marginals (no full pass to ride on) behaves as full_fit = 1:
    the committed model's own fit, after the merge."""
    I, J, K0, bs, R = 64, 48, 30, 5, 3
    T, truth = planted_dense(I, J, K0 + 2 * bs, R, noise=0.01, seed=42)
    T0, batches = split_dense(T, K0, bs)
    model = [np.ascontiguousarray(np.asarray(x, np.float32)) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    opts = L().default_opts(als_max_iters=8, als_tol=0.0, accept_tau=0.0, capacity=K0 + 2 * bs, full_fit=2,
                            incremental_marginals=1)
    h = L().sambaten_init_factors(L().dense(dev(T0)), R, 2, 4, 3, model[1], model[2], model[3], model[0], opts)
    try:
        X = T0
        for b in batches:
            info = L().sambaten_update(h, L().dense(dev(b)))
            X = np.concatenate([X, b])
            m = tuple(np.asarray(x, np.float64) for x in _model_out(h, I, J, X.shape[0], R))
            if info.fit_full_prev == -1.0:
                assert abs((1.0 - info.fit_full) - O.relative_error(X, *m)) <= 1e-6
            else:   # the first update still runs the full marginal pass (nothing committed yet)
                assert info.fit_full == -1.0
    finally:
        L().sambaten_destroy(h)
