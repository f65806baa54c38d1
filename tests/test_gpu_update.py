"""End-to-end GPU parity of sambaten_update against the oracle (Alg. 1), through the C-ABI.

Both sides start from the same float32 model (sambaten_init_factors / oracle init_factors),
so the zero masks and anchors agree.  Bars (BASELINE north_star):
sampled indices bit-exact; FMS >= 0.99 between the updated models after alignment;
|relative error difference| <= 1e-3."""
import numpy as np
import pytest

from oracle import sambaten as O
from synth import planted_dense, split_dense, CONFIGS
from tests._helpers import dev, host, torch_cuda

pytestmark = pytest.mark.gpu


def L():
    from paper_1709_00668_b200 import _lib
    return _lib


def _setup(I, J, K, R, K0, batch, noise, seed, s, r, maxit, tol=0.0, tau=0.9, init="als"):
    T, truth = planted_dense(I, J, K, R, noise=noise, seed=seed)
    T0, batches = split_dense(T, K0, batch)
    cfg = O.Config(R=R, s=(s, s, s), r=r, seed=seed + 11, maxit=maxit, tol=tol, tau=tau)
    if init == "als":
        st0 = O.init_als(T0, cfg, I * J * K, maxit=300, tol=1e-9)
        model = [np.asarray(x, np.float32) for x in (st0.lam, st0.A, st0.B, st0.C)]
    else:
        model = [np.asarray(x, np.float32) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    return T, T0, batches, cfg, model


def _gpu_handle(T0, cfg, model, cap_k, full_fit=1, on_device=True):
    lam, A, B, C = model
    opts = L().default_opts(als_max_iters=cfg.maxit, als_tol=cfg.tol, accept_tau=cfg.tau,
                            capacity=cap_k, full_fit=full_fit, merge_policy=cfg.merge_policy)
    X0 = L().dense(dev(T0) if on_device else np.ascontiguousarray(T0))
    return L().sambaten_init_factors(X0, cfg.R, cfg.s[0], cfg.r, cfg.seed, A, B, C, lam, opts)


def _update_both(h, st, batch, K_total):
    """Run one update on both sides; return the GPU model (host arrays) and info."""
    I, J = batch.shape[2], batch.shape[1]
    R = st.cfg.R
    A = np.empty((I, R), np.float32); B = np.empty((J, R), np.float32)
    C = np.empty((K_total, R), np.float32); lam = np.empty(R, np.float32)
    info = L().sambaten_update(h, L().dense(dev(batch)), A, B, C, lam)
    oinfo = O.update(st, batch)
    return (lam, A, B, C), info, oinfo


def _samples(h, r):
    n = L().sambaten_last_samples(h)
    Is = np.empty(r * n[0], np.int32); Js = np.empty(r * n[1], np.int32); Ks = np.empty(r * n[2], np.int32)
    L().sambaten_last_samples(h, Is, Js, Ks)
    return Is.reshape(r, -1), Js.reshape(r, -1), Ks.reshape(r, -1)


def _check(h, st, gm, info, oinfo):
    r = st.cfg.r
    Is, Js, Ks = _samples(h, r)
    for rho, rp in enumerate(oinfo["reps"]):
        assert np.array_equal(Is[rho], rp["Is"]), rho
        assert np.array_equal(Js[rho], rp["Js"]), rho
        assert np.array_equal(Ks[rho], rp["Ks"]), rho
    g64 = tuple(np.asarray(x, np.float64) for x in gm)
    fms = O.fms(g64, (st.lam, st.A, st.B, st.C))
    rel_o = O.relative_error(st.X, st.lam, st.A, st.B, st.C)
    rel_g = O.relative_error(st.X, *g64)
    gpu_rej = [i for i in range(r) if info.reps_rejected_mask >> i & 1]
    return fms, rel_g, rel_o, gpu_rej


def test_c1_config_parity():
    """BASELINE configs[0] exactly (50^3, R=3, K0=40 + 10, s=2, r=4, 50 iterations, tol 1e-6)."""
    w = CONFIGS["C1"]
    T, T0, batches, cfg, model = _setup(w.I, w.J, w.K, w.R, w.K0, w.batch, w.noise, w.seed, w.s, w.r,
                                        w.maxit, tol=w.tol)
    st = O.init_factors(T0, cfg, *model, w.I * w.J * w.K)
    h = _gpu_handle(T0, cfg, model, w.K)
    try:
        gm, info, oinfo = _update_both(h, st, batches[0], w.K)
        fms, rel_g, rel_o, gpu_rej = _check(h, st, gm, info, oinfo)
        assert gpu_rej == oinfo["rejected"]
        assert fms >= 0.99, fms
        assert abs(rel_g - rel_o) <= 1e-3, (rel_g, rel_o)
        assert abs((1 - info.fit_full) - rel_g) <= 1e-5
        assert info.k_total == 50 and info.scale_exp == st.S
    finally:
        L().sambaten_destroy(h)


@pytest.mark.parametrize("dims,R,s,r,batch,nb", [((60, 48, 40), 4, 2, 4, 5, 3),
                                                 ((120, 120, 110), 10, 5, 8, 10, 2),
                                                 ((37, 53, 29), 3, 3, 5, 3, 2)])
def test_multi_batch_parity(dims, R, s, r, batch, nb):
    """Several consecutive updates with ragged sizes; tol = 0 (fixed iterations) so both sides
    run the same number of ALS iterations."""
    I, J, K = dims
    K0 = K - batch * nb
    T, T0, batches, cfg, model = _setup(I, J, K, R, K0, batch, 0.01, 3, s, r, 30, tol=0.0)
    st = O.init_factors(T0, cfg, *model, I * J * K)
    h = _gpu_handle(T0, cfg, model, K)
    try:
        Kt = K0
        for b in batches:
            Kt += b.shape[0]
            gm, info, oinfo = _update_both(h, st, b, Kt)
            fms, rel_g, rel_o, gpu_rej = _check(h, st, gm, info, oinfo)
            assert gpu_rej == oinfo["rejected"]
            assert fms >= 0.99, fms
            assert abs(rel_g - rel_o) <= 1e-3, (rel_g, rel_o)
            # continue both from the same (GPU) model so later batches test the same state
            st.lam, st.A, st.B, st.C = (np.asarray(x, np.float64) for x in gm)
    finally:
        L().sambaten_destroy(h)


def test_noiseless_planted_pin():
    """BASELINE pin on the GPU: noiseless planted rank-R tensor, fit > 0.999 after the update
    (500 ALS iterations, reading R27)."""
    T, T0, batches, cfg, model = _setup(50, 50, 50, 3, 40, 10, 0.0, 0, 2, 4, 500, tol=1e-9, init="truth")
    h = _gpu_handle(T0, cfg, model, 50)
    try:
        info = L().sambaten_update(h, L().dense(dev(batches[0])))
        assert info.fit_full > 0.999, info.fit_full
    finally:
        L().sambaten_destroy(h)


def test_host_buffers_and_errors_leave_state_unchanged():
    torch = torch_cuda()
    T, T0, batches, cfg, model = _setup(40, 30, 30, 3, 20, 5, 0.01, 4, 2, 3, 10)
    h = _gpu_handle(T0, cfg, model, 30, on_device=False)
    try:
        L().sambaten_checkpoint(h)
        d0 = L().sambaten_get_factors(h)["dims"]
        with pytest.raises(L().SambatenError) as e:
            L().sambaten_update(h, L().dense(np.zeros((0, 30, 40), np.float32)))
        assert e.value.name == "E_EMPTY_BATCH"
        with pytest.raises(L().SambatenError) as e:
            L().sambaten_update(h, L().dense(np.zeros((2, 31, 40), np.float32)))
        assert e.value.name == "E_SHAPE"
        big = batches[0].copy()
        big[0, 0, 0] = 1e30
        with pytest.raises(L().SambatenError) as e:
            L().sambaten_update(h, L().dense(big))
        assert e.value.name == "E_FIXEDPOINT_RANGE"
        assert L().sambaten_get_factors(h)["dims"] == d0
        # host batch (H2D inside the call) gives the same model as a device batch
        A1 = np.empty((40, 3), np.float32)
        L().sambaten_update(h, L().dense(np.ascontiguousarray(batches[0])), A1)
        L().sambaten_restore(h)
        A2 = np.empty((40, 3), np.float32)
        L().sambaten_update(h, L().dense(dev(batches[0])), A2)
        assert np.array_equal(A1, A2)           # determinism + checkpoint/restore
        assert torch.cuda.is_available()
    finally:
        L().sambaten_destroy(h)


def test_all_reps_rejected():
    T, T0, batches, cfg, model = _setup(30, 30, 30, 2, 20, 5, 0.01, 5, 2, 2, 5, tau=1.5)
    h = _gpu_handle(T0, cfg, model, 30)
    try:
        with pytest.raises(L().SambatenError) as e:
            L().sambaten_update(h, L().dense(dev(batches[0])))
        assert e.value.name == "E_BATCH_REJECTED"
        assert L().sambaten_get_factors(h)["dims"][2] == 20
    finally:
        L().sambaten_destroy(h)


def test_init_als_on_gpu_matches_oracle_quality():
    """sambaten_init (full CP-ALS on X0) reaches the oracle's fit on the C1 initial tensor."""
    w = CONFIGS["C1"]
    T, truth = planted_dense(w.I, w.J, w.K, w.R, noise=w.noise, seed=w.seed)
    T0 = T[: w.K0]
    opts = L().default_opts(capacity=w.K, init_max_iters=200, init_tol=1e-9)
    h = L().sambaten_init(L().dense(dev(T0)), w.R, w.s, w.r, 0, opts)
    try:
        rel = L().sambaten_relative_error(h)
        cfg = O.Config(R=w.R, s=(2, 2, 2), r=4, seed=0)
        st = O.init_als(T0, cfg, w.I * w.J * w.K, maxit=200, tol=1e-9)
        rel_o = O.relative_error(T0, st.lam, st.A, st.B, st.C)
        assert abs(rel - rel_o) <= 1e-3, (rel, rel_o)
    finally:
        L().sambaten_destroy(h)


@pytest.mark.parametrize("s_mode,policy,moi", [((2, 3, 4), 0, 0), ((3, 2, 2), 1, 0), ((2, 2, 3), 0, 1)])
def test_variant_flags_parity(s_mode, policy, moi):
    """SURVEY 8(f) NEXT #4 flags against the oracle: per-mode sampling factors, the
    overwrite merge policy (R17) and the squared measure of importance (Eq. 1, R1)."""
    I, J, K, R, K0, batch = 60, 52, 40, 4, 30, 5
    T, truth = planted_dense(I, J, K, R, noise=0.01, seed=6)
    T0, batches = split_dense(T, K0, batch)
    model = [np.asarray(x, np.float32) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    cfg = O.Config(R=R, s=s_mode, r=4, seed=13, maxit=20, tol=0.0, tau=0.9, merge_policy=policy, moi=moi)
    st = O.init_factors(T0, cfg, *model, I * J * K)
    lam, A, B, C = model
    opts = L().default_opts(als_max_iters=20, als_tol=0.0, accept_tau=0.9, capacity=K, full_fit=1,
                            merge_policy=policy, moi=moi, s_mode=s_mode)
    h = L().sambaten_init_factors(L().dense(dev(T0)), R, 2, 4, 13, A, B, C, lam, opts)
    try:
        Kt = K0
        for b in batches[:2]:
            Kt += b.shape[0]
            gm, info, oinfo = _update_both(h, st, b, Kt)
            fms, rel_g, rel_o, gpu_rej = _check(h, st, gm, info, oinfo)
            assert gpu_rej == oinfo["rejected"]
            assert fms >= 0.99, fms
            assert abs(rel_g - rel_o) <= 1e-3, (rel_g, rel_o)
            st.lam, st.A, st.B, st.C = (np.asarray(x, np.float64) for x in gm)
    finally:
        L().sambaten_destroy(h)


@pytest.mark.parametrize("shape", [(60, 52, 40, 4, 30, 5, 4), (100, 100, 60, 10, 45, 5, 8)])
def test_warm_start_parity(shape):
    """Warm-started summary ALS (opts.warm_start, reading R34) against the
    oracle with the same flag: the small shape runs the multi-kernel ALS, the C2-like one the
    cluster kernel.  Same bars as the whole update."""
    I, J, K, R, K0, batch, r = shape
    T, truth = planted_dense(I, J, K, R, noise=0.01, seed=7)
    T0, batches = split_dense(T, K0, batch)
    model = [np.asarray(x, np.float32) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    cfg = O.Config(R=R, s=(2, 2, 2), r=r, seed=17, maxit=15, tol=0.0, tau=0.9, warm_start=True)
    st = O.init_factors(T0, cfg, *model, I * J * K)
    lam, A, B, C = model
    opts = L().default_opts(als_max_iters=15, als_tol=0.0, accept_tau=0.9, capacity=K, full_fit=1, warm_start=1)
    h = L().sambaten_init_factors(L().dense(dev(T0)), R, 2, r, 17, A, B, C, lam, opts)
    try:
        Kt = K0
        for b in batches[:2]:
            Kt += b.shape[0]
            gm, info, oinfo = _update_both(h, st, b, Kt)
            fms, rel_g, rel_o, gpu_rej = _check(h, st, gm, info, oinfo)
            assert gpu_rej == oinfo["rejected"]
            assert fms >= 0.99, fms
            assert abs(rel_g - rel_o) <= 1e-3, (rel_g, rel_o)
            assert abs(info.fit_summary - oinfo["fit_summary"]) <= 1e-4, (info.fit_summary, oinfo["fit_summary"])
            st.lam, st.A, st.B, st.C = (np.asarray(x, np.float64) for x in gm)
    finally:
        L().sambaten_destroy(h)


def test_warm_start_fixed_point():
    """The oracle pin on the GPU (tests/test_oracle_warm.py): a noiseless model with zero new
    slices is a fixed point of the warm-started sweep -> summary fits 1 to fp32 rounding after
    one iteration; the invalid flag combinations are refused."""
    rng = np.random.default_rng(2)
    I, J, K0, Kn, R = 64, 48, 40, 4, 3
    A, B, C = rng.random((I, R)), rng.random((J, R)), rng.random((K0, R))
    lam = rng.random(R) + 0.5
    A, B, C, lam = (np.asarray(x, np.float32) for x in (A, B, C, lam))
    X0 = np.einsum("if,jf,kf,f->kji", *(x.astype(np.float64) for x in (A, B, C, lam))).astype(np.float32)
    opts = L().default_opts(als_max_iters=1, als_tol=0.0, accept_tau=0.0, capacity=K0 + Kn, warm_start=1)
    h = L().sambaten_init_factors(L().dense(dev(X0)), R, 2, 4, 3, A, B, C, lam, opts)
    try:
        info = L().sambaten_update(h, L().dense(dev(np.zeros((Kn, J, I), np.float32))))
        # the summary fit is formed as ||Y||^2 - 2 <Y, M> + ||M||^2 from fp32 MTTKRP runs: at a
        # residual near 0 its square root exposes ~sqrt(1e-7) of rounding, hence 1e-3 (a cold
        # start after one sweep is below 0.99 here)
        assert info.fit_summary > 1.0 - 1e-3, info.fit_summary
    finally:
        L().sambaten_destroy(h)
    opts.warm_start = 0
    h = L().sambaten_init_factors(L().dense(dev(X0)), R, 2, 4, 3, A, B, C, lam, opts)
    try:
        info = L().sambaten_update(h, L().dense(dev(np.zeros((Kn, J, I), np.float32))))
        assert info.fit_summary < 0.99, info.fit_summary
    finally:
        L().sambaten_destroy(h)
    with pytest.raises(L().SambatenError):
        L().sambaten_init_factors(L().dense(dev(X0)), R, 2, 4, 3, A, B, C, lam,
                                  L().default_opts(warm_start=1, getrank=1))


@pytest.mark.parametrize("inc,ff", [(0, 1), (1, 1), (0, 2)])
def test_pipelined_parity(inc, ff):
    """R36: the pipelined update samples from the marginals the previous
    update committed (the tensor before the batch) while its own marginal pass runs on
    a side stream.  Against the oracle with the same flag over three consecutive batches:
    sampled indices bit-exact, identical rejected sets, FMS >= 0.99, |relerr diff| <= 1e-3;
    with incremental marginals and with the lag-1 fit as well."""
    I, J, K, R, K0, batch = 80, 64, 55, 4, 40, 5
    T, truth = planted_dense(I, J, K, R, noise=0.01, seed=19)
    T0, batches = split_dense(T, K0, batch)
    model = [np.asarray(x, np.float32) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    cfg = O.Config(R=R, s=(2, 2, 2), r=4, seed=23, maxit=15, tol=0.0, tau=0.9, pipelined=True)
    st = O.init_factors(T0, cfg, *model, I * J * K)
    lam, A, B, C = model
    opts = L().default_opts(als_max_iters=15, als_tol=0.0, accept_tau=0.9, capacity=K, full_fit=ff, pipelined=1,
                            incremental_marginals=inc)
    h = L().sambaten_init_factors(L().dense(dev(T0)), R, 2, 4, 23, A, B, C, lam, opts)
    try:
        Kt = K0
        for b in batches:
            Kt += b.shape[0]
            gm, info, oinfo = _update_both(h, st, b, Kt)
            fms, rel_g, rel_o, gpu_rej = _check(h, st, gm, info, oinfo)   # samples bit-exact inside
            assert gpu_rej == oinfo["rejected"]
            assert fms >= 0.99, fms
            assert abs(rel_g - rel_o) <= 1e-3, (rel_g, rel_o)
            st.lam, st.A, st.B, st.C = (np.asarray(x, np.float64) for x in gm)
    finally:
        L().sambaten_destroy(h)
