"""GetRank quality control (Alg. 2 "GetRank"; section "Dealing with rank deficient
updates") -- FP64 CPU oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/, never by the product
package; shares no code with the CUDA path.

Alg. 2: for every candidate rank i = 1..R and trial j = 1..it, run a CP decomposition of the
(summary) tensor at rank i and rate it with CorConDia (core consistency diagnostic, cited at
P:266 as [bro2003new]); return the rank of the best rating.  Readings (R29-R31):

R29  CorConDia of a rank-F model [[lambda; A, B, C]] of X: with lambda absorbed into the first
     factor (A' = A diag(lambda)), the least-squares Tucker core given the loadings is
     G = X x1 pinv(A') x2 pinv(B) x3 pinv(C) (F x F x F); with T the superdiagonal unit core,
     cc = 100 (1 - sum (G - T)^2 / F).  cc = 100 for an exact, consistent model.
R30  The CP runs: cp_als (this oracle's Alg. 1 step) from the Philox initialisation als_init with
     update_id = GETRANK_ID + i (candidate rank) and rep = rep_base + j (trial j; inside an
     update rep_base = rho * trials for repetition rho), so the runs are reproducible and
     independent of launch geometry.
R31  "sort p and get top 1 index" taken literally always returns rank 1: a converged
     rank-1 model has cc = 100 (its core is the 1 x 1 x 1 scalar 1).  Reading: R_new = the
     largest candidate rank whose best trial reaches the threshold (default 90, the customary
     CorConDia cut-off), else 1.
"""
import numpy as np

from .sambaten import Coo, als_init, coo_to_dense, cp_als, view_ijk

GETRANK_ID = 0x47520000   # "GR" << 16: Philox update_id base of the GetRank trials (R30)


def superdiagonal(F):
    T = np.zeros((F, F, F))
    for f in range(F):
        T[f, f, f] = 1.0
    return T


def tucker_core(Y, lam, A, B, C):
    """Least-squares core G given the loadings (R29): mode products with the pseudo-inverses."""
    A1 = np.asarray(A, np.float64) * np.asarray(lam, np.float64)[None, :]
    PA, PB, PC = np.linalg.pinv(A1), np.linalg.pinv(np.asarray(B, np.float64)), np.linalg.pinv(np.asarray(C, np.float64))
    return np.einsum("ijk,fi,gj,hk->fgh", np.asarray(Y, np.float64), PA, PB, PC, optimize=True)


def corcondia(Y, lam, A, B, C):
    """Core consistency (R29) of the model [[lam; A, B, C]] of the tensor Y: dense Y[i, j, k], or
    a Coo (densified: the same core; the GPU forms it from the nonzeros)."""
    if isinstance(Y, Coo):
        Y = view_ijk(coo_to_dense(Y))
    F = np.asarray(A).shape[1]
    G = tucker_core(Y, lam, A, B, C)
    return 100.0 * (1.0 - float(np.sum((G - superdiagonal(F)) ** 2)) / F)


def getrank(Y, Rmax, trials, seed, maxit, tol, threshold=90.0, rep_base=0):
    """Alg. 2 (R30, R31): returns (R_new, cc[Rmax][trials]); Y dense [i, j, k] or a Coo."""
    if not isinstance(Y, Coo):
        Y = np.asarray(Y, np.float64)
    shape = Y.dims if isinstance(Y, Coo) else Y.shape
    cc = np.zeros((Rmax, trials))
    for F in range(1, Rmax + 1):
        for j in range(trials):
            U0 = als_init(shape, F, seed, GETRANK_ID + F, rep_base + j)
            lam, U, _, _, _ = cp_als(Y, U0, maxit, tol)
            cc[F - 1, j] = corcondia(Y, lam, *U)
    best = cc.max(axis=1)
    ok = [F for F in range(1, Rmax + 1) if best[F - 1] >= threshold]
    return (max(ok) if ok else 1), cc
