"""GPU parity of the sparse (COO) path against the oracle, through the C-ABI.

Same bars as the dense path (BASELINE north_star): sampled indices bit-exact, FMS >= 0.99
after alignment, |relative error difference| <= 1e-3; integer work (marginals) bit-exact."""
import numpy as np
import pytest

from oracle import sambaten as O
from synth import zipf_planted_coo, community_coo, split_coo
from tests._helpers import dev, host, torch_cuda

pytestmark = pytest.mark.gpu


def L():
    from paper_1709_00668_b200 import _lib
    return _lib


def _oc(X):
    return O.Coo(X.i.astype(np.int64), X.j.astype(np.int64), X.k.astype(np.int64), X.v, X.dims)


def _gc(X, on_device=True):
    f = dev if on_device else np.ascontiguousarray
    return L().coo(f(X.i.astype(np.int32)), f(X.j.astype(np.int32)), f(X.k.astype(np.int32)), f(X.v), X.dims)


def _samples(h, r):
    n = L().sambaten_last_samples(h)
    Is = np.empty(r * n[0], np.int32); Js = np.empty(r * n[1], np.int32); Ks = np.empty(r * n[2], np.int32)
    L().sambaten_last_samples(h, Is, Js, Ks)
    return Is.reshape(r, -1), Js.reshape(r, -1), Ks.reshape(r, -1)


def _run(X, truth, K0, batch, R, s, r, maxit, tol=0.0, seed=7, nb=None, tau=0.9, warm=False, models=None):
    X0, batches = split_coo(X, K0, batch)
    if nb is not None:
        batches = batches[:nb]
    lam, A, B, C = truth
    model = [np.ascontiguousarray(np.asarray(x, np.float32)) for x in (lam, A, B, C[:K0])]
    cfg = O.Config(R=R, s=(s, s, s), r=r, seed=seed, maxit=maxit, tol=tol, tau=tau, warm_start=warm)
    st = O.init_factors(_oc(X0), cfg, *model, X.nnz)
    opts = L().default_opts(als_max_iters=maxit, als_tol=tol, accept_tau=tau, capacity=X.nnz,
                            capacity_k=X.dims[2], full_fit=1, warm_start=int(warm))
    h = L().sambaten_init_factors(_gc(X0), R, s, r, seed, model[1], model[2], model[3], model[0], opts)
    out = []
    try:
        Kt = K0
        for b in batches:
            Kt += b.dims[2]
            gA = np.empty((X.dims[0], R), np.float32); gB = np.empty((X.dims[1], R), np.float32)
            gC = np.empty((Kt, R), np.float32); gl = np.empty(R, np.float32)
            info = L().sambaten_update(h, _gc(b), gA, gB, gC, gl)
            oinfo = O.update(st, _oc(b))
            Is, Js, Ks = _samples(h, r)
            for rho, rp in enumerate(oinfo["reps"]):
                assert np.array_equal(Is[rho], rp["Is"]), rho
                assert np.array_equal(Js[rho], rp["Js"]), rho
                assert np.array_equal(Ks[rho], rp["Ks"]), rho
            g64 = tuple(np.asarray(x, np.float64) for x in (gl, gA, gB, gC))
            fms = O.fms(g64, (st.lam, st.A, st.B, st.C))
            rel_o = O.relative_error(st.X, st.lam, st.A, st.B, st.C)
            rel_g = O.relative_error(st.X, *g64)
            gpu_rej = [i for i in range(r) if info.reps_rejected_mask >> i & 1]
            out.append((fms, rel_g, rel_o, gpu_rej, oinfo["rejected"], info))
            if models is not None:
                models.append((gl.copy(), gA.copy(), gB.copy(), gC.copy()))
            # continue both sides from the GPU model
            st.lam, st.A, st.B, st.C = g64
    finally:
        L().sambaten_destroy(h)
    return out


def test_coo_update_parity_planted():
    X, truth = zipf_planted_coo(400, 300, 60, 4, 30_000, alpha=1.2, seed=3)
    res = _run(X, truth, 50, 5, R=4, s=2, r=4, maxit=30, nb=2)
    for fms, rel_g, rel_o, gr, orr, info in res:
        assert gr == orr
        assert fms >= 0.99, fms
        assert abs(rel_g - rel_o) <= 1e-3, (rel_g, rel_o)
        assert abs((1 - info.fit_full) - rel_g) <= 1e-5


def test_coo_warm_start_parity():
    """The warm-started summary ALS (R34) on COO summaries: the model's rows as the start; the
    same bars as the plain COO update (samples bit-exact inside _run), over two batches."""
    X, truth = zipf_planted_coo(400, 300, 60, 4, 30_000, alpha=1.2, seed=13)
    res = _run(X, truth, 50, 5, R=4, s=2, r=4, maxit=8, nb=2, warm=True)
    for fms, rel_g, rel_o, gr, orr, info in res:
        assert gr == orr
        assert fms >= 0.99, fms
        assert abs(rel_g - rel_o) <= 1e-3, (rel_g, rel_o)


def test_coo_update_parity_communities_ragged():
    """C3-like community counts (Zipf 1.5), ragged sample sizes, paper-literal tau = 0."""
    X = community_coo(1000, 90, 5, 40_000, alpha=1.5, seed=4)
    rng = np.random.default_rng(0)
    truth = (np.ones(5), rng.random((1000, 5)), rng.random((1000, 5)), rng.random((90, 5)))
    res = _run(X, truth, 77, 13, R=5, s=3, r=3, maxit=10, nb=1, tau=0.0)
    for fms, rel_g, rel_o, gr, orr, info in res:
        assert gr == orr == []
        assert fms >= 0.99, fms
        assert abs(rel_g - rel_o) <= 1e-3, (rel_g, rel_o)


def test_coo_errors_leave_state_unchanged():
    X, truth = zipf_planted_coo(200, 100, 30, 3, 5_000, seed=5)
    X0, batches = split_coo(X, 25, 5)
    lam, A, B, C = (np.ascontiguousarray(np.asarray(x, np.float32)) for x in truth)
    opts = L().default_opts(als_max_iters=5, capacity=X.nnz, capacity_k=30)
    h = L().sambaten_init_factors(_gc(X0), 3, 2, 2, 0, A, B, C[:25].copy(), lam, opts)
    try:
        b = batches[0]
        bad = type(b)(b.i[::-1].copy(), b.j[::-1].copy(), b.k[::-1].copy(), b.v[::-1].copy(), b.dims)
        with pytest.raises(L().SambatenError) as e:
            L().sambaten_update(h, _gc(bad))
        assert e.value.name == "E_INVALID"
        oob = type(b)(b.i.copy(), b.j.copy(), b.k.copy(), b.v.copy(), b.dims)
        oob.k[-1] = 99
        with pytest.raises(L().SambatenError) as e:
            L().sambaten_update(h, _gc(oob))
        assert e.value.name == "E_INDEX_RANGE"
        assert L().sambaten_get_factors(h)["dims"][2] == 25
        info = L().sambaten_update(h, _gc(b, on_device=False))   # host arrays work too
        assert info.k_total == 30
    finally:
        L().sambaten_destroy(h)


def test_coo_init_als_quality():
    """sambaten_init on a COO tensor: full CP-ALS reaches the oracle's fit."""
    X, truth = zipf_planted_coo(300, 200, 40, 3, 20_000, seed=6)
    X0, _ = split_coo(X, 40, 10)
    opts = L().default_opts(capacity=X.nnz, capacity_k=60, init_max_iters=100, init_tol=1e-9)
    h = L().sambaten_init(_gc(X0), 3, 2, 2, 0, opts)
    try:
        rel = L().sambaten_relative_error(h)
        cfg = O.Config(R=3, s=(2, 2, 2), r=2, seed=0)
        st = O.init_als(_oc(X0), cfg, X.nnz, maxit=100, tol=1e-9)
        rel_o = O.relative_error(st.X, st.lam, st.A, st.B, st.C)
        assert abs(rel - rel_o) <= 1e-3, (rel, rel_o)
    finally:
        L().sambaten_destroy(h)


# ------------------------------------------------------------------- stateless primitives
def _rand_coo(dims, nnz, seed):
    rng = np.random.default_rng(seed)
    I, J, K = dims
    lin = np.unique(rng.integers(0, I * J * K, nnz))
    i = lin % I; j = (lin // I) % J; k = lin // (I * J)
    v = rng.standard_normal(len(lin)).astype(np.float32)
    return O.coo_canonical(i, j, k, v, dims)


@pytest.mark.parametrize("dims,ns", [((50, 40, 30), (25, 13, 7)), ((300, 200, 64), (30, 200, 64)),
                                     ((7, 5, 3), (7, 5, 3)), ((3000, 2000, 400), (700, 300, 120))])
def test_gather_coo_bit_exact(dims, ns):
    """The last case spans >= 4 x 148 tiles of 2048 entries: the persistent kernels with the I / J
    membership masks in shared memory."""
    torch = torch_cuda()
    X = _rand_coo(dims, 1_700_000 if dims[0] == 3000 else 4000, 11)
    rng = np.random.default_rng(3)
    idx = [np.sort(rng.choice(d, n, replace=False)).astype(np.int32) for d, n in zip(dims, ns)]
    cap = X.nnz
    oi, oj, ok = (torch.empty(cap, dtype=torch.int32, device="cuda") for _ in range(3))
    ov = torch.empty(cap, dtype=torch.float32, device="cuda")
    onnz = torch.zeros(1, dtype=torch.int64, device="cuda")
    L().sambaten_gather(_gc(X), dev(idx[0]), ns[0], dev(idx[1]), ns[1], dev(idx[2]), ns[2], oi=oi, oj=oj,
                        ok=ok, ov=ov, cap=cap, out_nnz=onnz)
    ref = O.gather_coo(X, idx[0], idx[1], idx[2])
    n = int(host(onnz)[0])
    assert n == ref.nnz
    for g, r in zip((oi, oj, ok), (ref.i, ref.j, ref.k)):
        assert np.array_equal(host(g)[:n], np.asarray(r, np.int32))
    assert np.array_equal(host(ov)[:n].view(np.uint32), ref.v.astype(np.float32).view(np.uint32))


@pytest.mark.parametrize("dims,nnz,R", [((60, 50, 40), 3000, 4), ((500, 400, 90), 40_000, 10),
                                        ((9, 8, 7), 50, 1), ((200, 100, 64), 10_000, 15)])
def test_mttkrp_coo(dims, nnz, R):
    torch = torch_cuda()
    X = _rand_coo(dims, nnz, R)
    rng = np.random.default_rng(R + 1)
    U = [rng.random((n, R)).astype(np.float32) for n in dims]
    Ud = [dev(u) for u in U]
    for mode in range(3):
        M = torch.empty((dims[mode], R), dtype=torch.float32, device="cuda")
        L().sambaten_mttkrp(_gc(X), Ud[0], Ud[1], Ud[2], R, mode, M)
        ref = O.mttkrp(X, [u.astype(np.float64) for u in U], mode)
        err = np.linalg.norm(host(M).astype(np.float64) - ref) / max(np.linalg.norm(ref), 1e-300)
        assert err <= 1e-5, (mode, err)


def test_fit_coo_and_cp_als_coo():
    torch = torch_cuda()
    X, truth = zipf_planted_coo(120, 100, 40, 3, 6000, seed=9)
    Xo = _oc(X)
    lam, A, B, C = (np.asarray(x, np.float32) for x in truth)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    L().sambaten_fit(_gc(X), dev(lam), dev(A), dev(B), dev(C), 3, out)
    ref = O.relative_error(Xo, *(x.astype(np.float64) for x in (lam, A, B, C)))
    assert abs(float(host(out)[0]) - ref) <= 1e-6
    U0 = O.als_init(X.dims, 3, 5, 1, 0)
    Ud = [dev(u.astype(np.float32)) for u in U0]
    lamd = torch.empty(3, dtype=torch.float64, device="cuda")
    fit = torch.empty(1, dtype=torch.float64, device="cuda")
    it = torch.empty(1, dtype=torch.int32, device="cuda")
    L().sambaten_cp_als(_gc(X), 3, Ud[0], Ud[1], Ud[2], lamd, 40, 0.0, fit, it)
    lo, Uo, fo, io, _ = O.cp_als(Xo, U0, 40, 0.0)
    assert int(host(it)[0]) == io == 40
    assert abs(float(host(fit)[0]) - fo) <= 1e-3
    g = (host(lamd), *[host(u).astype(np.float64) for u in Ud])
    assert O.fms(g, (lo, *Uo)) >= 0.99


def test_coo_update_persistent_als_matches_oracle_and_pipeline(monkeypatch):
    """The persistent cooperative COO ALS (als_plan kind 3, k_coo_als.cu) against the oracle on a
    Zipf-hot stream whose rows span several MTTKRP pieces (rows > 256 entries: multi-piece
    partials), and against the per-mode kernel pipeline (kind 4) on the same input."""
    X, truth = zipf_planted_coo(300, 250, 60, 6, 120_000, alpha=1.5, seed=11)
    res = _run(X, truth, 50, 5, R=6, s=2, r=4, maxit=25, nb=2, tau=0.0)
    for fms, rel_g, rel_o, gr, orr, info in res:
        assert info.als_plan[0] == 3, list(info.als_plan)
        assert fms >= 0.99, fms
        assert abs(rel_g - rel_o) <= 1e-3, (rel_g, rel_o)
    monkeypatch.setenv("SAMBATEN_COO_ALS_MULTI", "1")
    res_m = _run(X, truth, 50, 5, R=6, s=2, r=4, maxit=25, nb=2, tau=0.0)
    for (fms, rel_g, _, _, _, _), (fms_m, rel_m, _, _, _, info_m) in zip(res, res_m):
        assert info_m.als_plan[0] == 4, list(info_m.als_plan)
        assert abs(rel_g - rel_m) <= 1e-4, (rel_g, rel_m)


def test_coo_radix_scatter_tile_local_bit_identical(monkeypatch):
    """The summaries' stable radix sort (k_coo.cu) with the tile ordered by digit in shared memory
    before its runs are written (SAMBATEN_RADIX_LOCAL) gives the same permutation as the default
    per-element scatter: the updated models are bit-identical, at a size whose summaries span
    many 4096-entry tiles with a ragged last tile (two 8-bit passes of the (rep, index) keys)."""
    X, truth = zipf_planted_coo(3000, 700, 60, 5, 300_001, alpha=1.3, seed=5)
    ma, mb = [], []
    ra = _run(X, truth, 50, 5, R=5, s=2, r=4, maxit=6, nb=2, tau=0.0, models=ma)
    monkeypatch.setenv("SAMBATEN_RADIX_LOCAL", "1")
    rb = _run(X, truth, 50, 5, R=5, s=2, r=4, maxit=6, nb=2, tau=0.0, models=mb)
    assert len(ma) == len(mb) == 2
    for x, y in zip(ma, mb):
        for u, v in zip(x, y):
            assert np.array_equal(u, v)
    for (fms, rel_g, rel_o, _, _, _) in ra:
        assert fms >= 0.99, fms
        assert abs(rel_g - rel_o) <= 1e-3, (rel_g, rel_o)
