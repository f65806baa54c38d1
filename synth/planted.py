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
