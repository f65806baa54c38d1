"""Planted low-rank tensors.  Input generation only."""
from dataclasses import dataclass
import numpy as np


@dataclass
class CooArrays:
    """Plain COO arrays, canonical (sorted by (k, j, i), unique, nonzero), int32 / float32."""
    i: np.ndarray
    j: np.ndarray
    k: np.ndarray
    v: np.ndarray
    dims: tuple

    @property
    def nnz(self):
        return int(self.v.shape[0])


def planted_dense_factors(I, J, K, R, seed):
    """Factors with iid U[0,1) entries (BASELINE configs 1, 2, 4; "randomly generated
    factors"), lambda = 1."""
    rng = np.random.default_rng(seed)
    A = rng.random((I, R))
    B = rng.random((J, R))
    C = rng.random((K, R))
    return A, B, C


def dense_from_factors(A, B, C, noise, seed, k_range=None):
    """float32 slab T[k, j, i] = sum_f A(i,f) B(j,f) C(k,f) + sigma * N(0,1),
    sigma = noise * ||clean||_F / sqrt(N) over the WHOLE I x J x K tensor."""
    I, J, K = A.shape[0], B.shape[0], C.shape[0]
    G = (A.T @ A) * (B.T @ B) * (C.T @ C)
    clean_norm = float(np.sqrt(G.sum()))
    sigma = noise * clean_norm / np.sqrt(float(I) * J * K)
    k0, k1 = (0, K) if k_range is None else k_range
    T = np.empty((k1 - k0, J, I), np.float32)
    rng = np.random.default_rng([seed, 7])
    # the noise stream is consumed slice by slice from k = 0 so that any k_range is a
    # sub-range of the same tensor
    for k in range(0, k1):
        eps = rng.standard_normal((J, I)) if noise > 0 else None
        if k < k0:
            continue
        sl = (B * C[k][None, :]) @ A.T
        if noise > 0:
            sl = sl + sigma * eps
        T[k - k0] = sl.astype(np.float32)
    return T


def planted_dense(I, J, K, R, noise=0.01, seed=0):
    A, B, C = planted_dense_factors(I, J, K, R, seed)
    return dense_from_factors(A, B, C, noise, seed), (np.ones(R), A, B, C)


def split_dense(T, K0, batch):
    """Initial K0 slices, then batches of ``batch`` slices (P:452 stream protocol)."""
    out = [T[:K0]]
    k = K0
    while k < T.shape[0]:
        out.append(T[k:k + batch])
        k += batch
    return out[0], out[1:]


def _canonical(i, j, k, v, dims):
    I, J, K = dims
    lin = (k.astype(np.int64) * J + j) * I + i
    order = np.argsort(lin, kind="stable")
    lin, v = lin[order], v[order].astype(np.float64)
    uniq, start = np.unique(lin, return_index=True)
    sums = np.add.reduceat(v, start).astype(np.float32)
    keep = sums != 0
    uniq, sums = uniq[keep], sums[keep]
    return CooArrays((uniq % I).astype(np.int32), ((uniq // I) % J).astype(np.int32),
                     (uniq // (I * J)).astype(np.int32), sums, tuple(int(d) for d in dims))


def community_coo(I, K, R, nnz, alpha=1.5, seed=0):
    """User x user x day counts (BASELINE config 3; stand-in for Facebook-wall/links):
    R communities = a random permutation of the I users split in R near-equal blocks; each
    community has two independent Zipf(alpha) rank orders over its members (owner, poster);
    a draw picks a community uniformly, i and j by Zipf rank, day k uniformly, and a
    Geometric(1/2) count (mean 2).  Duplicates are summed; draws continue until ``nnz``
    unique coordinates exist."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(I)
    blocks = np.array_split(perm, R)
    orders = [(rng.permutation(b), rng.permutation(b)) for b in blocks]
    cdfs = []
    for b in blocks:
        w = np.arange(1, len(b) + 1, dtype=np.float64) ** (-alpha)
        cdfs.append(np.cumsum(w) / w.sum())
    ii, jj, kk, vv = [], [], [], []
    have = 0
    seen = None
    while have < nnz:
        m = max(int((nnz - have) * 1.7), 1024)
        f = rng.integers(0, R, m)
        ri = np.empty(m, np.int64); rj = np.empty(m, np.int64)
        for c in range(R):
            sel = f == c
            n = int(sel.sum())
            ri[sel] = orders[c][0][np.minimum(np.searchsorted(cdfs[c], rng.random(n)), len(cdfs[c]) - 1)]
            rj[sel] = orders[c][1][np.minimum(np.searchsorted(cdfs[c], rng.random(n)), len(cdfs[c]) - 1)]
        rk = rng.integers(0, K, m)
        val = rng.geometric(0.5, m).astype(np.float32)
        ii.append(ri); jj.append(rj); kk.append(rk); vv.append(val)
        lin = np.unique((np.concatenate(kk) * I + np.concatenate(jj)) * I + np.concatenate(ii))
        have = len(lin)
        seen = lin
    i = np.concatenate(ii); j = np.concatenate(jj); k = np.concatenate(kk); v = np.concatenate(vv)
    if have > nnz:
        # keep the draws whose coordinate is among the first nnz distinct coordinates drawn
        lin = (k * I + j) * I + i
        _, first = np.unique(lin, return_index=True)
        keep_lin = lin[np.sort(first)[:nnz]]
        sel = np.isin(lin, keep_lin)
        i, j, k, v = i[sel], j[sel], k[sel], v[sel]
    del seen
    return _canonical(i, j, k, v, (I, I, K))


def zipf_planted_coo(I, J, K, R, nnz, alpha=1.2, seed=0):
    """Planted rank-R sparse tensor (BASELINE config 5; the 100K^3 shape of P:529):
    A(:,f), B(:,f) = Zipf(alpha) weights rank^-alpha on an independent random permutation
    per component, C(:,f) ~ U[0.5, 1.5]; a draw picks f uniformly, i ~ A(:,f), j ~ B(:,f),
    k ~ C(:,f); value = sum_f A(i,f) B(j,f) C(k,f) (no noise); unique coordinates up to nnz."""
    rng = np.random.default_rng(seed)
    w = np.arange(1, I + 1, dtype=np.float64) ** (-alpha)
    A = np.zeros((I, R)); B = np.zeros((J, R))
    wj = np.arange(1, J + 1, dtype=np.float64) ** (-alpha)
    for f in range(R):
        A[rng.permutation(I), f] = w
        B[rng.permutation(J), f] = wj
    C = rng.uniform(0.5, 1.5, (K, R))
    cdfA = [np.cumsum(A[:, f]) / A[:, f].sum() for f in range(R)]
    cdfB = [np.cumsum(B[:, f]) / B[:, f].sum() for f in range(R)]
    cdfC = [np.cumsum(C[:, f]) / C[:, f].sum() for f in range(R)]
    lins = []
    have = 0
    while have < nnz:
        m = max(int((nnz - have) * 1.1), 1024)
        f = rng.integers(0, R, m)
        ri = np.empty(m, np.int64); rj = np.empty(m, np.int64); rk = np.empty(m, np.int64)
        for c in range(R):
            sel = f == c
            n = int(sel.sum())
            ri[sel] = np.minimum(np.searchsorted(cdfA[c], rng.random(n)), I - 1)
            rj[sel] = np.minimum(np.searchsorted(cdfB[c], rng.random(n)), J - 1)
            rk[sel] = np.minimum(np.searchsorted(cdfC[c], rng.random(n)), K - 1)
        lins.append((rk * J + rj) * I + ri)
        allv = np.concatenate(lins)
        _, first = np.unique(allv, return_index=True)
        have = len(first)
    allv = np.concatenate(lins)
    _, first = np.unique(allv, return_index=True)
    lin = np.sort(allv[np.sort(first)[:nnz]])
    i = lin % I; j = (lin // I) % J; k = lin // (I * J)
    v = np.einsum("nf,nf,nf->n", A[i], B[j], C[k]).astype(np.float32)
    return _canonical(i, j, k, v, (I, J, K)), (np.ones(R), A, B, C)


def split_coo(X, K0, batch):
    """Initial slices [0, K0) and then batches of ``batch`` slices, each batch re-based to k=0."""
    def take(k0, k1):
        sel = (X.k >= k0) & (X.k < k1)
        return CooArrays(X.i[sel], X.j[sel], (X.k[sel] - k0).astype(np.int32), X.v[sel],
                         (X.dims[0], X.dims[1], k1 - k0))
    K = X.dims[2]
    init = take(0, K0)
    out = []
    k = K0
    while k < K:
        out.append(take(k, min(k + batch, K)))
        k += batch
    return init, out


# ---------------------------------------------------------------------------------------
# Counter-based dense generator (the large dense configs, C4): the same recipe as
# dense_from_factors, with the noise drawn from Philox4x32-10 (counter domain GEN = 3) by
# Box-Muller so that any slab can be produced independently -- on the device by
# synth/csrc/gen.cu (synth_dense_slab), here by the numpy twin below (small slabs; tests).
# ---------------------------------------------------------------------------------------
_M0, _M1, _W0, _W1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57), 0x9E3779B9, 0xBB67AE85
_MASK = np.uint64(0xFFFFFFFF)


def _philox_np(seed, c0, c1, c2, c3):
    """Philox4x32-10 on uint32 counter arrays (numpy uint64 carriers)."""
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    x0, x1, x2, x3 = (np.asarray(c, np.uint64) & _MASK for c in (c0, c1, c2, c3))
    for _ in range(10):
        p0 = _M0 * x0
        p1 = _M1 * x2
        n0 = (p1 >> np.uint64(32)) ^ x1 ^ np.uint64(k0)
        n2 = (p0 >> np.uint64(32)) ^ x3 ^ np.uint64(k1)
        x0, x1, x2, x3 = n0 & _MASK, p1 & _MASK, n2 & _MASK, p0 & _MASK
        k0 = (k0 + _W0) & 0xFFFFFFFF
        k1 = (k1 + _W1) & 0xFFFFFFFF
    return x0, x1, x2, x3


def _unit(a, b):
    m52 = (a << np.uint64(20)) | (b >> np.uint64(12))
    return (2.0 * m52.astype(np.float64) + 1.0) * 2.0 ** -53


def planted_sigma(A, B, C, noise):
    """sigma = noise * ||[[A, B, C]]||_F / sqrt(N) (closed-form norm from the Grams)."""
    G = (A.T @ A) * (B.T @ B) * (C.T @ C)
    return noise * float(np.sqrt(G.sum())) / np.sqrt(float(A.shape[0]) * B.shape[0] * C.shape[0])


def dense_philox_slab(A, B, C, sigma, seed, k0, nk):
    """numpy twin of synth_dense_slab: float32 [nk][J][I] of slices [k0, k0 + nk)."""
    I, J, R = A.shape[0], B.shape[0], A.shape[1]
    e0, e1 = k0 * I * J, (k0 + nk) * I * J
    e = np.arange(e0, e1, dtype=np.int64)
    k, rem = np.divmod(e, I * J)
    j, i = np.divmod(rem, I)
    s = np.zeros(e.shape[0])
    for f in range(R):
        s = s + (A[i, f] * B[j, f]) * C[k, f]
    if sigma != 0.0:
        p = (e >> 1).astype(np.uint64)
        x0, x1, x2, x3 = _philox_np(seed, p & _MASK, p >> np.uint64(32), 0, 3 << 24)
        u1, u2 = _unit(x0, x1), _unit(x2, x3)
        r = np.sqrt(-2.0 * np.log(u1))
        z = np.where((e & 1) == 0, r * np.cos(2.0 * np.pi * u2), r * np.sin(2.0 * np.pi * u2))
        s = s + sigma * z
    return s.astype(np.float32).reshape(nk, J, I)
