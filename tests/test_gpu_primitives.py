"""GPU parity of the exposed primitives against the oracle, through the C-ABI.

Bars (BASELINE north_star): marginals, sampled indices and gathered summaries bit-exact;
MTTKRP relative Frobenius error <= 1e-5; ALS compared by FMS and fit."""
import numpy as np
import pytest

from oracle import sambaten as O
from oracle.philox import philox4x32_10, detlog, uniform53
from tests._helpers import dev, host, rel_fro, random_dense, torch_cuda

pytestmark = pytest.mark.gpu


def L():
    from paper_1709_00668_b200 import _lib
    return _lib


# ---------------------------------------------------------------------------------- RNG
def test_philox_bit_exact():
    torch = torch_cuda()
    for (c0, c1, c2, c3, key) in ((0, 0, 0, 0, 0), (123, 7, 9, (1 << 24) | (3 << 8) | 2, 0xDEADBEEF12345678),
                                  (0xFFFFFF00, 1, 2, 3, 2 ** 64 - 1)):
        n = 5000
        out = torch.empty(4 * n, dtype=torch.int32, device="cuda")
        L().sambaten_philox(c0, c1, c2, c3, key, n, out)
        got = host(out).view(np.uint32).reshape(n, 4)
        idx = (np.arange(n, dtype=np.uint64) + c0) & 0xFFFFFFFF
        ref = philox4x32_10(idx, c1, c2, c3, key)
        for w in range(4):
            assert np.array_equal(got[:, w].astype(np.uint64), ref[w])


def test_detlog_bit_exact():
    torch = torch_cuda()
    rng = np.random.default_rng(0)
    x0 = rng.integers(0, 2 ** 32, 200_000, dtype=np.uint64)
    x1 = rng.integers(0, 2 ** 32, 200_000, dtype=np.uint64)
    u = uniform53(x0, x1)
    u = np.concatenate([u, [2.0 ** -53, 1 - 2.0 ** -53, 0.5, 0.75, float.fromhex("0x1.6a09e667f3bcdp-1"),
                            float.fromhex("0x1.6a09e667f3bccp-1"), 1e-300]])
    out = torch.empty(len(u), dtype=torch.float64, device="cuda")
    L().sambaten_detlog(dev(u), len(u), out)
    got = host(out)
    assert np.array_equal(got.view(np.uint64), detlog(u).view(np.uint64))


# ---------------------------------------------------------------------------- marginals
@pytest.mark.parametrize("shape", [(7, 5, 50), (13, 40, 500), (3, 2, 3000), (1, 1, 1), (6, 9, 33)])
@pytest.mark.parametrize("moi", [0, 1])
def test_marginals_dense_bit_exact(shape, moi):
    torch = torch_cuda()
    K, J, I = shape
    T = random_dense(K, J, I, seed=sum(shape), zero_frac=0.1, scale=3.0)
    S = O.fixed_point_scale(T.size, float(O.phi(T.ravel(), moi).max()))
    x = [torch.empty(n, dtype=torch.int64, device="cuda") for n in (I, J, K)]
    L().sambaten_marginals(L().dense(dev(T)), moi, S, *x)
    ref = O.marginals_dense(T, S, moi)
    for g, r in zip(x, ref):
        assert np.array_equal(host(g), r)


@pytest.mark.parametrize("shape", [(40, 30, 600), (9, 20, 3000), (5, 7, 1024), (3, 11, 2500), (37, 3, 600)])
@pytest.mark.parametrize("moi,magic", [(0, False), (1, False), (0, True)])
def test_marginals_dense_q32_bit_exact(shape, moi, magic, monkeypatch):
    """The 32-bit stream kernel (every q <= 2^27, as at C4 where ceil log2 of the capacity is 35):
    S chosen so that q = RNE(phi 2^S) <= 2^27 exactly at the maximum (phi <= 1 here), the bound
    passed through the SAMBATEN_MARG_QB hook; bit-exact against the oracle (column sums folded
    every 15 warp steps, row totals by 18-bit chunk sums).  magic: the data bound q <= 2^21 also
    passed (SAMBATEN_MARG_PHIMAX), the FMA rounding with biased sums C4's data take.  (37, 3, 600):
    an odd row count per stage step."""
    torch = torch_cuda()
    K, J, I = shape
    rng = np.random.default_rng(sum(shape) + moi)
    T = rng.random((K, J, I)).astype(np.float32)
    T[0, 0, 0] = 1.0                        # q = 2^27 exactly
    T[rng.random(T.shape) < 0.1] = 0.0
    T[..., -1] = np.nextafter(np.float32(1.0), np.float32(0.0))   # a column of near-maximal values
    S = 27
    monkeypatch.setenv("SAMBATEN_MARG_QB", "27")
    if magic:   # q <= 2^21 < 2^22: q = bits(fma(|x|, 2^S, 2^23)) - bits(2^23), biased 32-bit sums
        S = 21
        monkeypatch.setenv("SAMBATEN_MARG_PHIMAX", "1.0")
    x = [torch.empty(n, dtype=torch.int64, device="cuda") for n in (I, J, K)]
    L().sambaten_marginals(L().dense(dev(T)), moi, S, *x)
    for g, r in zip(x, O.marginals_dense(T, S, moi)):
        assert np.array_equal(host(g), r)


@pytest.mark.parametrize("moi", [0, 1])
def test_marginals_coo_bit_exact(moi):
    torch = torch_cuda()
    T = random_dense(40, 30, 20, seed=5, zero_frac=0.9)
    T[3, :, :] = 0.0                       # an empty slice
    kk, jj, ii = np.nonzero(T)
    X = O.coo_canonical(ii, jj, kk, T[kk, jj, ii], (20, 30, 40))
    S = O.fixed_point_scale(X.nnz, float(O.phi(X.v, moi).max()))
    x = [torch.empty(n, dtype=torch.int64, device="cuda") for n in (20, 30, 40)]
    t = L().coo(dev(X.i.astype(np.int32)), dev(X.j.astype(np.int32)), dev(X.k.astype(np.int32)),
                dev(X.v), (20, 30, 40))
    L().sambaten_marginals(t, moi, S, *x)
    for g, r in zip(x, O.marginals_coo(X, S, moi)):
        assert np.array_equal(host(g), r)


@pytest.mark.parametrize("moi,hot", [(0, True), (1, True), (0, False), (0, "rep"), (1, "rep")])
def test_marginals_coo_large_bit_exact(moi, hot):
    """COO marginals on larger inputs: Zipf-hot indices (a few i / j carry most entries, the
    C3 / C5 hazard) and near-uniform ones; bit-exact against the oracle.  "rep": nnz >= 8 (I + J),
    the replicated kernel (16 copies of x1 / x2, warp-combined j / k runs)."""
    from synth import zipf_planted_coo
    torch = torch_cuda()
    if hot == "rep":
        Xs, _ = zipf_planted_coo(12_000, 9_000, 300, 4, 1_500_000, alpha=1.2, seed=10)
        assert Xs.nnz >= 64 * (12_000 + 9_000)
    elif hot:
        Xs, _ = zipf_planted_coo(60_000, 50_000, 400, 4, 600_000, alpha=1.3, seed=8)
    else:
        rng = np.random.default_rng(9)
        n = 400_000
        ii, jj, kk = rng.integers(0, 60_000, n), rng.integers(0, 50_000, n), rng.integers(0, 400, n)
        Xs = O.coo_canonical(ii, jj, kk, rng.random(n).astype(np.float32) + 0.5, (60_000, 50_000, 400))
    X = O.Coo(np.asarray(Xs.i, np.int64), np.asarray(Xs.j, np.int64), np.asarray(Xs.k, np.int64), Xs.v, Xs.dims)
    assert X.nnz > 200_000
    S = O.fixed_point_scale(X.nnz, float(O.phi(X.v, moi).max()))
    x = [torch.zeros(n, dtype=torch.int64, device="cuda") for n in X.dims]
    t = L().coo(dev(X.i.astype(np.int32)), dev(X.j.astype(np.int32)), dev(X.k.astype(np.int32)), dev(X.v), X.dims)
    L().sambaten_marginals(t, moi, S, *x)
    for g, r in zip(x, O.marginals_coo(X, S, moi)):
        assert np.array_equal(host(g), r)


# ----------------------------------------------------------------------------- sampling
@pytest.mark.parametrize("n,ns", [(50, 25), (500, 100), (1, 1), (7, 7), (100_000, 5000), (65_536, 6554),
                                  (3000, 300), (33, 0)])
def test_sample_bit_exact(n, ns):
    torch = torch_cuda()
    rng = np.random.default_rng(n + ns)
    w = rng.integers(0, 2 ** 40, n).astype(np.int64)
    w[rng.random(n) < 0.2] = 0
    if n > 10:
        w[:5] = 12345                      # equal weights
    wd = dev(w)
    for rep, mode, uid in ((0, 0, 1), (3, 2, 7), (31, 1, 123456)):
        out = torch.full((max(ns, 1),), -1, dtype=torch.int32, device="cuda")
        L().sambaten_sample(wd, n, ns, 0xABCDEF, uid, rep, mode, out)
        ref = O.sample_mode(w, ns, 0xABCDEF, uid, rep, mode)
        assert np.array_equal(host(out)[:ns], ref)


def test_sample_all_zero_weights_and_huge_weights():
    torch = torch_cuda()
    for w in (np.zeros(40, np.int64), np.full(40, 2 ** 62, np.int64), np.array([0, 0, 7, 0], np.int64)):
        n = len(w)
        ns = min(n, 9)
        out = torch.empty(ns, dtype=torch.int32, device="cuda")
        L().sambaten_sample(dev(w), n, ns, 1, 1, 0, 0, out)
        assert np.array_equal(host(out), O.sample_mode(w, ns, 1, 1, 0, 0))


# ------------------------------------------------------------------------------- gather
@pytest.mark.parametrize("shape,ns", [((20, 30, 50), (25, 15, 12)), ((60, 70, 500), (100, 14, 30)),
                                      ((5, 4, 3), (3, 4, 5))])
def test_gather_dense_bit_exact(shape, ns):
    torch = torch_cuda()
    K, J, I = shape
    T = random_dense(K, J, I, seed=1)
    rng = np.random.default_rng(2)
    Is = np.sort(rng.choice(I, ns[0], replace=False)).astype(np.int32)
    Js = np.sort(rng.choice(J, ns[1], replace=False)).astype(np.int32)
    Kp = np.sort(rng.choice(K, ns[2], replace=False)).astype(np.int32)
    out = torch.empty(ns[2] * ns[1] * ns[0], dtype=torch.float32, device="cuda")
    L().sambaten_gather(L().dense(dev(T)), dev(Is), ns[0], dev(Js), ns[1], dev(Kp), ns[2], out_dense=out)
    ref = O.gather_dense(T, Is, Js, Kp)           # [p, q, u]
    got = host(out).reshape(ns[2], ns[1], ns[0]).transpose(2, 1, 0)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


# ------------------------------------------------------------------------------- MTTKRP
@pytest.mark.parametrize("shape,R", [((30, 20, 50), 3), ((108, 100, 100), 10), ((45, 40, 300), 10),
                                     ((9, 7, 5), 1), ((33, 17, 130), 15), ((20, 10, 3000), 10),
                                     ((12, 11, 10), 32)])
def test_mttkrp_dense(shape, R):
    torch = torch_cuda()
    K, J, I = shape
    T = random_dense(K, J, I, seed=K + R)
    rng = np.random.default_rng(R)
    U = [rng.random((n, R)).astype(np.float32) for n in (I, J, K)]
    Ud = [dev(u) for u in U]
    Yo = O.view_ijk(T)
    for mode in range(3):
        M = torch.empty((U[mode].shape[0], R), dtype=torch.float32, device="cuda")
        L().sambaten_mttkrp(L().dense(dev(T)), Ud[0], Ud[1], Ud[2], R, mode, M)
        ref = O.mttkrp(Yo, [u.astype(np.float64) for u in U], mode)
        assert rel_fro(host(M), ref) <= 1e-5, (mode, rel_fro(host(M), ref))


# ---------------------------------------------------------------------------------- ALS
@pytest.mark.parametrize("shape,R,its", [((25, 25, 30), 3, 50), ((60, 50, 40), 10, 30)])
def test_cp_als_tracks_oracle(shape, R, its):
    """Same Philox init, fixed iteration count (tol = 0): fp32 GPU vs fp64 oracle stay
    together (FMS >= 0.99, |fit difference| <= 1e-3)."""
    torch = torch_cuda()
    K, J, I = shape
    rng = np.random.default_rng(3)
    F = [rng.random((n, R)) for n in (I, J, K)]
    Tc = np.einsum("if,jf,kf->kji", *F)
    T = (Tc + 0.01 * np.linalg.norm(Tc) / np.sqrt(Tc.size) * rng.standard_normal(Tc.shape)).astype(np.float32)
    U0 = O.als_init((I, J, K), R, 77, 5, 2)
    Ud = [dev(u.astype(np.float32)) for u in U0]
    lam = torch.empty(R, dtype=torch.float64, device="cuda")
    fit = torch.empty(1, dtype=torch.float64, device="cuda")
    it = torch.empty(1, dtype=torch.int32, device="cuda")
    L().sambaten_cp_als(L().dense(dev(T)), R, Ud[0], Ud[1], Ud[2], lam, its, 0.0, fit, it)
    lo, Uo, fo, io, _ = O.cp_als(O.view_ijk(T), U0, its, 0.0)
    assert int(host(it)[0]) == io == its
    assert abs(float(host(fit)[0]) - fo) <= 1e-3
    g = (host(lam), *[host(u).astype(np.float64) for u in Ud])
    assert O.fms(g, (lo, *Uo)) >= 0.99


# ---------------------------------------------------------------------------------- fit
@pytest.mark.parametrize("K,J,I,R", [(40, 30, 50, 4), (40, 30, 64, 10), (6, 7, 3000, 3), (30, 20, 500, 16)])
def test_fit_dense(K, J, I, R):
    """Tiled (I % 4 != 0) and streamed (I % 4 == 0, column-chunked for I > 2048) fits."""
    torch = torch_cuda()
    rng = np.random.default_rng(4)
    F = [rng.random((n, R)).astype(np.float32) for n in (I, J, K)]
    lam = (rng.random(R) + 0.5).astype(np.float32)
    T = (np.einsum("f,if,jf,kf->kji", lam, *F) + 0.1 * rng.standard_normal((K, J, I))).astype(np.float32)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    L().sambaten_fit(L().dense(dev(T)), dev(lam), dev(F[0]), dev(F[1]), dev(F[2]), R, out)
    ref = O.relative_error(T, lam.astype(np.float64), *[f.astype(np.float64) for f in F])
    assert abs(float(host(out)[0]) - ref) <= 1e-6
