"""GPU parity of the update's edge cases and of the largest config's kernel instantiation
(VERDICT r01 "close the parity gaps"), through the C-ABI, against the oracle:

* the exact C4 summary shape (300 x 300 x 320 summaries, R = 10, r = 16) on a host-sized
  tensor (600 x 600 x 590, s = 2): the same a4 plan the full C4 config runs (asserted through
  sambaten_als_plan), paper-literal (tau = 0) and with the acceptance test (tau = 0.9);
* zeroed model rows: the zero-entry fill (R17) with the anchor exclusion (P:198,
  R14) and the old-frame rescale (R16), on the cluster and the multi-kernel ALS;
* the lambda average (R19);
* the pseudo-inverse fallback (R12): a model component with an all-zero B column drives every
  summary solve through it; reps_pinv_mask must equal the oracle's;
* R = 32 (the warp Hungarian's widest case, R15);
* the warm-started sweep on the multi-kernel path (its Grams must be those of the warm rows).
"""
import os

import numpy as np
import pytest

from oracle import sambaten as O
from synth import planted_dense, split_dense
from tests._helpers import dev

pytestmark = pytest.mark.gpu


def L():
    from paper_1709_00668_b200 import _lib
    return _lib


def _handle(T0, cfg, model, cap_k, **kw):
    lam, A, B, C = (np.ascontiguousarray(x, np.float32) for x in model)
    opts = L().default_opts(als_max_iters=cfg.maxit, als_tol=cfg.tol, accept_tau=cfg.tau, capacity=cap_k,
                            full_fit=1, merge_policy=cfg.merge_policy, warm_start=int(cfg.warm_start), **kw)
    return L().sambaten_init_factors(L().dense(dev(T0)), cfg.R, cfg.s[0], cfg.r, cfg.seed, A, B, C, lam, opts)


def _gpu_update(h, batch, I, J, K_total, R):
    A = np.empty((I, R), np.float32); B = np.empty((J, R), np.float32)
    C = np.empty((K_total, R), np.float32); lam = np.empty(R, np.float32)
    info = L().sambaten_update(h, L().dense(dev(batch)), A, B, C, lam)
    return (lam, A, B, C), info


def _rejected(info, r):
    return [i for i in range(r) if info.reps_rejected_mask >> i & 1]


class _AlsCache:
    """Memoise the oracle's summary ALS across the two acceptance settings of one stream (the
    samples and summaries do not depend on tau; only acceptance and merge do)."""

    def __init__(self):
        self.orig = O.cp_als
        self.memo = {}

    def __call__(self, Y, U, maxit, tol, stats=None):
        key = (hash(np.asarray(Y).tobytes()), hash(b"".join(np.asarray(u).tobytes() for u in U)), maxit, tol)
        if key not in self.memo:
            st = {"pinv": False}
            self.memo[key] = (self.orig(Y, U, maxit, tol, st), st["pinv"])
        out, pinv = self.memo[key]
        if stats is not None and pinv:
            stats["pinv"] = True
        return out


def test_c4_summary_shape_parity(monkeypatch):
    """The full C4 config decomposes 16 summaries of 300 x 300 x (270 + 50) at R = 10
    (3000 / s with s = 10).  The same summary shape arises from 600 x 600 x (540 + 50) with
    s = 2, small enough for the oracle: the test asserts the update runs the a4 plan the C4
    shape gets (kind, CTAs per repetition, RB, D placement) and compares with the oracle at
    tau = 0 (paper-literal, every rep merged) and tau = 0.9 (R26): identical rejected sets,
    FMS >= 0.99, |relerr_gpu - relerr_oracle| <= 1e-3 (BASELINE north_star)."""
    I = J = 600
    K0, Kn, R, r, s, it = 540, 50, 10, 16, 2, 30
    plan_c4 = L().sambaten_als_plan(300, 300, 270 + 50, R, r)
    T, truth = planted_dense(I, J, K0 + Kn, R, noise=0.01, seed=21)
    T0, batches = split_dense(T, K0, Kn)
    model = [np.asarray(x, np.float32) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    cache = _AlsCache()
    monkeypatch.setattr(O, "cp_als", cache)
    for tau in (0.0, 0.9):
        cfg = O.Config(R=R, s=(s, s, s), r=r, seed=5, maxit=it, tol=0.0, tau=tau)
        st = O.init_factors(T0, cfg, *model, T.size)
        h = _handle(T0, cfg, model, K0 + Kn)
        try:
            try:
                oinfo = O.update(st, batches[0])
            except O.BatchRejected:
                oinfo = None
            if oinfo is None:
                with pytest.raises(L().SambatenError) as e:
                    _gpu_update(h, batches[0], I, J, K0 + Kn, R)
                assert e.value.name == "E_BATCH_REJECTED"
                continue
            gm, info = _gpu_update(h, batches[0], I, J, K0 + Kn, R)
            assert list(info.als_plan) == plan_c4, (list(info.als_plan), plan_c4)
            assert _rejected(info, r) == oinfo["rejected"], (tau, _rejected(info, r), oinfo["rejected"])
            g64 = tuple(np.asarray(x, np.float64) for x in gm)
            fms = O.fms(g64, (st.lam, st.A, st.B, st.C))
            rel_g = O.relative_error(st.X, *g64)
            rel_o = O.relative_error(st.X, st.lam, st.A, st.B, st.C)
            assert fms >= 0.99, (tau, fms)
            assert abs(rel_g - rel_o) <= 1e-3, (tau, rel_g, rel_o)
            assert abs((1.0 - info.fit_full) - rel_g) <= 1e-5
            # per-rep summary fits (mean) as a finer check of the ALS itself
            assert abs(info.fit_summary - oinfo["fit_summary"]) <= 1e-4, (info.fit_summary, oinfo["fit_summary"])
        finally:
            L().sambaten_destroy(h)


def _noiseless_truth_model(seed, I=40, K0=32, Kn=8, R=3):
    T, truth = planted_dense(I, I, K0 + Kn, R, noise=0.0, seed=seed)
    T0, batches = split_dense(T, K0, Kn)
    model = [np.asarray(x, np.float32) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    return T, T0, batches, model, [np.asarray(x, np.float32).astype(np.float64) for x in truth]


@pytest.mark.parametrize("multi_kernel", [False, True])
def test_zeroed_rows_filled_like_oracle(multi_kernel, monkeypatch):
    """Model = truth with rows of A and B zeroed ("not yet computed"): the GPU refills
    exactly the rows the oracle refills, with the oracle's values (fp32 ALS vs fp64: 1e-4), the
    true rows (noiseless, converged), and leaves every other cell bit-unchanged."""
    if multi_kernel:
        monkeypatch.setenv("SAMBATEN_NO_CLUSTER_ALS", "1")
    T, T0, batches, model, truth = _noiseless_truth_model(seed=31)
    zA, zB = [0, 3, 8, 15, 22, 37], [2, 9, 10, 25, 39]
    model[1][zA] = 0.0
    model[2][zB] = 0.0
    cfg = O.Config(R=3, s=(2, 2, 2), r=4, seed=9, maxit=600, tol=0.0, tau=0.9)
    st = O.init_factors(T0, cfg, *model, T.size)
    h = _handle(T0, cfg, model, T.shape[0])
    try:
        gm, info = _gpu_update(h, batches[0], 40, 40, T.shape[0], 3)
        oinfo = O.update(st, batches[0])
        assert (info.als_plan[0] == 0) == multi_kernel
        assert _rejected(info, 4) == oinfo["rejected"] == []
        for gF, oF, F0, Ft, zs in ((gm[1], st.A, model[1], truth[1], zA), (gm[2], st.B, model[2], truth[2], zB)):
            keep = np.ones(gF.shape[0], bool); keep[zs] = False
            assert np.array_equal(gF[keep], F0[keep])            # nonzero cells bit-unchanged
            for i in zs:
                if np.all(oF[i] == 0.0):
                    assert np.all(gF[i] == 0.0), i                 # unsampled: still not computed
                else:
                    assert np.allclose(gF[i], oF[i], rtol=1e-4), (i, gF[i], oF[i])
                    assert np.allclose(gF[i], Ft[i], rtol=1e-4), (i, gF[i], Ft[i])
        assert sum(np.any(gm[1][zA] != 0, axis=1)) + sum(np.any(gm[2][zB] != 0, axis=1)) >= 6
    finally:
        L().sambaten_destroy(h)


def test_lambda_average_like_oracle():
    """Model = truth with lambda doubled (noiseless): lambda -> (2 + 1)/2 = 1.5 (R19) on
    both sides."""
    T, T0, batches, model, truth = _noiseless_truth_model(seed=32)
    model[0] = 2.0 * model[0]
    cfg = O.Config(R=3, s=(2, 2, 2), r=4, seed=10, maxit=600, tol=0.0, tau=0.9)
    st = O.init_factors(T0, cfg, *model, T.size)
    h = _handle(T0, cfg, model, T.shape[0])
    try:
        gm, info = _gpu_update(h, batches[0], 40, 40, T.shape[0], 3)
        O.update(st, batches[0])
        assert np.allclose(st.lam, 1.5, rtol=1e-5)
        assert np.allclose(gm[0], 1.5, rtol=1e-4), gm[0]
    finally:
        L().sambaten_destroy(h)


@pytest.mark.parametrize("multi_kernel", [False, True])
def test_pinv_fallback_like_oracle(multi_kernel, monkeypatch):
    """A model component whose B column is all zero, warm-started (R34): every normal matrix of
    every summary ALS has a zero row / column, Cholesky / the SPD inverse fails and the
    pseudo-inverse (R12) runs on both sides.  reps_pinv_mask equals the oracle's (all reps), the
    paper-literal merge halves lambda of that component (lambda_hat = 0) and gives it
    zero new C rows; the other components agree with the oracle."""
    if multi_kernel:
        monkeypatch.setenv("SAMBATEN_NO_CLUSTER_ALS", "1")
    T, truth = planted_dense(48, 40, 36, 3, noise=0.01, seed=33)
    T0, batches = split_dense(T, 30, 6)
    model = [np.asarray(x, np.float32) for x in (truth[0], truth[1], truth[2], truth[3][:30])]
    model[2][:, 2] = 0.0
    cfg = O.Config(R=3, s=(2, 2, 2), r=4, seed=12, maxit=12, tol=0.0, tau=0.0, warm_start=True)
    st = O.init_factors(T0, cfg, *model, T.size)
    h = _handle(T0, cfg, model, 36)
    try:
        gm, info = _gpu_update(h, batches[0], 48, 40, 36, 3)
        oinfo = O.update(st, batches[0])
        o_mask = sum(1 << i for i, rp in enumerate(oinfo["reps"]) if rp["pinv"])
        assert o_mask == 0b1111
        assert info.reps_pinv_mask == o_mask, (bin(info.reps_pinv_mask), bin(o_mask))
        assert gm[0][2] == np.float32(model[0][2] / 2)
        assert np.all(gm[3][30:, 2] == 0.0)
        g64 = [np.asarray(x, np.float64) for x in gm]
        for gF, oF in zip(g64[1:], (st.A, st.B, st.C)):
            assert np.allclose(gF[:, :2], oF[:, :2], rtol=2e-3, atol=1e-5)
        assert np.allclose(g64[0], st.lam, rtol=2e-3)
    finally:
        L().sambaten_destroy(h)


def test_rank32_update_parity():
    """R = 32, the widest rank (kMaxR): the warp Hungarian (R > 8, R15) initialises all R + 1
    potentials; the update matches the oracle (rejected sets, FMS, relative error)."""
    I, K0, Kn, R, r = 90, 80, 10, 32, 4
    T, truth = planted_dense(I, I, K0 + Kn, R, noise=0.01, seed=34)
    T0, batches = split_dense(T, K0, Kn)
    model = [np.asarray(x, np.float32) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    cfg = O.Config(R=R, s=(2, 2, 2), r=r, seed=14, maxit=25, tol=0.0, tau=0.0)
    st = O.init_factors(T0, cfg, *model, T.size)
    h = _handle(T0, cfg, model, K0 + Kn)
    try:
        gm, info = _gpu_update(h, batches[0], I, I, K0 + Kn, R)
        oinfo = O.update(st, batches[0])
        pis = [rp["match"].pi for rp in oinfo["reps"]]
        assert all(sorted(p.tolist()) == list(range(R)) for p in pis)
        assert _rejected(info, r) == oinfo["rejected"]
        g64 = tuple(np.asarray(x, np.float64) for x in gm)
        assert O.fms(g64, (st.lam, st.A, st.B, st.C)) >= 0.99
        rel_g = O.relative_error(st.X, *g64)
        rel_o = O.relative_error(st.X, st.lam, st.A, st.B, st.C)
        assert abs(rel_g - rel_o) <= 1e-3, (rel_g, rel_o)
    finally:
        L().sambaten_destroy(h)


def test_warm_start_one_sweep_multi_kernel(monkeypatch):
    """The warm-start fixed point (R34) with one ALS sweep on the multi-kernel path: its first
    solves must use the Grams of the warm rows (a Gram of the Philox point would leave the
    summary fit well below 1)."""
    monkeypatch.setenv("SAMBATEN_NO_CLUSTER_ALS", "1")
    rng = np.random.default_rng(4)
    I, J, K0, Kn, R = 64, 48, 40, 4, 3
    A, B, C = rng.random((I, R)), rng.random((J, R)), rng.random((K0, R))
    lam = rng.random(R) + 0.5
    A, B, C, lam = (np.asarray(x, np.float32) for x in (A, B, C, lam))
    X0 = np.einsum("if,jf,kf,f->kji", *(x.astype(np.float64) for x in (A, B, C, lam))).astype(np.float32)
    opts = L().default_opts(als_max_iters=1, als_tol=0.0, accept_tau=0.0, capacity=K0 + Kn, warm_start=1)
    h = L().sambaten_init_factors(L().dense(dev(X0)), R, 2, 4, 3, A, B, C, lam, opts)
    try:
        info = L().sambaten_update(h, L().dense(dev(np.zeros((Kn, J, I), np.float32))))
        assert info.als_plan[0] == 0
        assert info.fit_summary > 1.0 - 1e-3, info.fit_summary
    finally:
        L().sambaten_destroy(h)


@pytest.mark.parametrize("grid", ["0", "1"])
def test_cluster_and_grid_als_parity(grid, monkeypatch):
    """The a4 kernel with thread-block clusters (DSMEM exchange) and with CTA groups of one
    cooperative grid (global-memory exchange, more SMs per repetition): both match the oracle
    on a C2-like stream (identical rejected sets, FMS >= 0.99, |relerr diff| <= 1e-3) and report
    their plan kind (1 cluster, 2 grid)."""
    monkeypatch.setenv("SAMBATEN_ALS_GRID", grid)
    I, K0, Kn, R, r = 200, 150, 10, 10, 8
    T, truth = planted_dense(I, I, K0 + 2 * Kn, R, noise=0.01, seed=35)
    T0, batches = split_dense(T, K0, Kn)
    model = [np.asarray(x, np.float32) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    cfg = O.Config(R=R, s=(2, 2, 2), r=r, seed=16, maxit=30, tol=0.0, tau=0.9)
    st = O.init_factors(T0, cfg, *model, T.size)
    h = _handle(T0, cfg, model, K0 + 2 * Kn)
    try:
        Kt = K0
        for b in batches:
            Kt += Kn
            gm, info = _gpu_update(h, b, I, I, Kt, R)
            oinfo = O.update(st, b)
            assert info.als_plan[0] == (2 if grid == "1" else 1), list(info.als_plan)
            assert _rejected(info, r) == oinfo["rejected"]
            g64 = tuple(np.asarray(x, np.float64) for x in gm)
            assert O.fms(g64, (st.lam, st.A, st.B, st.C)) >= 0.99
            assert abs(O.relative_error(st.X, *g64) - O.relative_error(st.X, st.lam, st.A, st.B, st.C)) <= 1e-3
            assert abs(info.fit_summary - oinfo["fit_summary"]) <= 1e-4
            st.lam, st.A, st.B, st.C = g64
    finally:
        L().sambaten_destroy(h)
