"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

C2 (500^3, R=10, s=5, r=8, 30 iterations): the oracle finishes a whole update in seconds, so
the first batch is checked end to end exactly as in test_gpu_update.py (marginals and sampled
indices bit-exact, identical rejected sets, FMS >= 0.99, |relerr diff| <= 1e-3).

C4 (3000 x 3000 x 2750 after the first batch, 99 GB, generated on the device): the oracle cannot
hold the tensor, so the update's marginals are checked through properties that hold at any
size and on sampled outputs the oracle computes one by one -- x1(i), x2(j), x3(k) for sampled
indices recomputed from the tensor's fibres / slices, the exact equality of the three marginal
totals -- and then the sampled indices are recomputed by the oracle from those marginals
(bit-exact), and sampled summary entries are compared with the tensor entries they copy."""
import numpy as np
import pytest

from oracle import sambaten as O
from synth import planted_dense, split_dense, CONFIGS
from tests._helpers import dev

pytestmark = pytest.mark.gpu


def L():
    from paper_1709_00668_b200 import _lib
    return _lib


def _samples(h, r):
    n = L().sambaten_last_samples(h)
    Is = np.empty(r * n[0], np.int32); Js = np.empty(r * n[1], np.int32); Ks = np.empty(r * n[2], np.int32)
    L().sambaten_last_samples(h, Is, Js, Ks)
    return Is.reshape(r, -1), Js.reshape(r, -1), Ks.reshape(r, -1)


def test_c2_full_size_update_parity():
    w = CONFIGS["C2"]
    T, truth = planted_dense(w.I, w.J, w.K, w.R, noise=w.noise, seed=w.seed)
    T0, batches = split_dense(T, w.K0, w.batch)
    model = [np.ascontiguousarray(np.asarray(x, np.float32)) for x in (truth[0], truth[1], truth[2], truth[3][:w.K0])]
    cfg = O.Config(R=w.R, s=(w.s,) * 3, r=w.r, seed=w.seed, maxit=w.maxit, tol=0.0, tau=0.9)
    st = O.init_factors(T0, cfg, *model, T.size)
    opts = L().default_opts(als_max_iters=w.maxit, als_tol=0.0, capacity=w.K, full_fit=1, accept_tau=0.9)
    h = L().sambaten_init_factors(L().dense(dev(T0)), w.R, w.s, w.r, w.seed, model[1], model[2], model[3],
                                  model[0], opts)
    try:
        Kt = w.K0 + w.batch
        A = np.empty((w.I, w.R), np.float32); B = np.empty((w.J, w.R), np.float32)
        C = np.empty((Kt, w.R), np.float32); lam = np.empty(w.R, np.float32)
        info = L().sambaten_update(h, L().dense(dev(batches[0])), A, B, C, lam)
        oinfo = O.update(st, batches[0])
        # marginals of the update's tensor through the same streaming kernel (stateless call)
        import torch
        Xd = dev(st.X)
        x = [torch.zeros(n, dtype=torch.int64, device="cuda") for n in (w.I, w.J, Kt)]
        L().sambaten_marginals(L().dense(Xd), 0, st.S, *x)
        for g, o in zip(x, oinfo["x"]):
            assert np.array_equal(g.cpu().numpy(), o)
        Is, Js, Ks = _samples(h, w.r)
        for rho, rp in enumerate(oinfo["reps"]):
            assert np.array_equal(Is[rho], rp["Is"]) and np.array_equal(Js[rho], rp["Js"])
            assert np.array_equal(Ks[rho], rp["Ks"])
        gpu_rej = [i for i in range(w.r) if info.reps_rejected_mask >> i & 1]
        assert gpu_rej == oinfo["rejected"]
        g64 = tuple(np.asarray(v, np.float64) for v in (lam, A, B, C))
        assert O.fms(g64, (st.lam, st.A, st.B, st.C)) >= 0.99
        rel_o = O.relative_error(st.X, st.lam, st.A, st.B, st.C)
        rel_g = O.relative_error(st.X, *g64)
        assert abs(rel_g - rel_o) <= 1e-3
        assert abs((1.0 - info.fit_full) - rel_g) <= 1e-5
    finally:
        L().sambaten_destroy(h)


def test_c4_full_size_marginals_sampling_gather():
    import torch
    from synth import gpu as G
    from synth.planted import planted_dense_factors, planted_sigma
    w = CONFIGS["C4"]
    if torch.cuda.get_device_properties(0).total_memory < 150e9:
        pytest.skip("C4 needs ~110 GB of device memory")
    G.build()
    Kt = w.K0 + w.batch
    A, B, Cf = planted_dense_factors(w.I, w.J, w.K, w.R, w.seed)
    sigma = planted_sigma(A, B, Cf, w.noise)
    dA, dB, dC = (torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (A, B, Cf))
    store = torch.empty((Kt, w.J, w.I), dtype=torch.float32, device="cuda")
    G.dense_slab(store, dA, dB, dC, sigma, w.seed, 0, Kt)
    batch = store[w.K0:Kt].clone()
    model = [np.ones(w.R, np.float32), A.astype(np.float32), B.astype(np.float32),
             np.ascontiguousarray(Cf[:w.K0].astype(np.float32))]
    # full_fit = 2: the bench's launch configuration -- the marginals of the old slices come from
    # the fused marginal + lag-1 fit kernel (32-bit arithmetic at this scale, q <= 2^27)
    opts = L().default_opts(als_max_iters=2, als_tol=0.0, capacity=Kt, full_fit=2, accept_tau=0.0,
                            borrow_store=1)
    h = L().sambaten_init_factors(L().dense(store[:w.K0]), w.R, w.s, w.r, w.seed, model[1], model[2],
                                  model[3], model[0], opts)
    try:
        info = L().sambaten_update(h, L().dense(batch))
        del batch
        # the lag-1 fit (the initial model over X0) equals the separate fit kernel's value
        rel = torch.zeros(1, dtype=torch.float64, device="cuda")
        dm = [dev(v) for v in model]
        L().sambaten_fit(L().dense(store[:w.K0]), dm[0], dm[1], dm[2], dm[3], w.R, rel)
        torch.cuda.synchronize()
        assert info.fit_full == -1.0
        assert abs(info.fit_full_prev - (1.0 - float(rel[0]))) <= 1e-6, (info.fit_full_prev, 1.0 - float(rel[0]))
        x = [torch.zeros(n, dtype=torch.int64, device="cuda") for n in (w.I, w.J, Kt)]
        mx = max(float(store[k0:min(k0 + 100, w.K0)].abs().max()) for k0 in range(0, w.K0, 100))
        S = O.fixed_point_scale(w.I * w.J * Kt, mx)
        assert S == info.scale_exp
        L().sambaten_marginals(L().dense(store), 0, S, *x)
        x1, x2, x3 = (v.cpu().numpy() for v in x)
        t = int(x1.sum(dtype=np.int64))
        assert t == int(x2.sum(dtype=np.int64)) == int(x3.sum(dtype=np.int64))
        rng = np.random.default_rng(1)
        q = lambda v: O.quantize(v.astype(np.float64), S, O.MOI_ABS)   # noqa: E731
        for i in rng.choice(w.I, 2, replace=False):
            assert int(q(store[:, :, int(i)].cpu().numpy()).sum()) == int(x1[i])
        for j in rng.choice(w.J, 2, replace=False):
            assert int(q(store[:, int(j), :].cpu().numpy()).sum()) == int(x2[j])
        for k in (0, w.K0 - 1, w.K0, Kt - 1):
            assert int(q(store[k].cpu().numpy()).sum()) == int(x3[k])
        # the update's sample = the oracle's sampling of these (verified) marginals
        Is, Js, Ks = _samples(h, w.r)
        for rho in (0, w.r - 1):
            assert np.array_equal(Is[rho], O.sample_mode(x1, O.sample_size(w.I, w.s), w.seed, 1, rho, 0))
            assert np.array_equal(Js[rho], O.sample_mode(x2, O.sample_size(w.J, w.s), w.seed, 1, rho, 1))
            assert np.array_equal(Ks[rho], O.sample_mode(x3[:w.K0], O.sample_size(w.K0, w.s), w.seed, 1, rho, 2))
        # sampled summary entries are bit copies of the tensor entries
        Kp = O.k_prime(Ks[0], w.K0, w.batch)
        nI, nJ, nK = len(Is[0]), len(Js[0]), len(Kp)
        Y = torch.empty((nK, nJ, nI), dtype=torch.float32, device="cuda")
        L().sambaten_gather(L().dense(store), dev(Is[0]), nI, dev(Js[0]), nJ, dev(Kp.astype(np.int32)), nK,
                            out_dense=Y)
        Yh = Y.cpu().numpy()
        for _ in range(200):
            p, qq, u = int(rng.integers(nI)), int(rng.integers(nJ)), int(rng.integers(nK))
            assert Yh[u, qq, p] == float(store[int(Kp[u]), int(Js[0][qq]), int(Is[0][p])])
    finally:
        L().sambaten_destroy(h)
