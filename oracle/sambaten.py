"""FP64 CPU oracle of SamBaTen's per-batch incremental CP update (Alg. 1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/, by
__graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference legs,
never by the product package.  It shares no code with the CUDA path.

Conventions
-----------
* A dense tensor is stored as a float32 numpy array ``T`` of shape (K, J, I),
  C-contiguous, i.e. X(i,j,k) = T[k, j, i] (i fastest, the layout of a stream
  of frontal slices X(:,:,k)).  ``view_ijk(T)`` gives X[i,j,k].
* A sparse tensor is a ``Coo`` (int64 i, j, k; float32 v; dims), canonical:
  sorted by (k, j, i), no duplicates, no explicit zeros.
* Factors are float64 (rows x R), lambda float64 (R,).
* All arithmetic is float64; the tensor values are the caller's float32 bits.
* Readings R1..R27 are listed in DESIGN.md (= SURVEY.md §8(c) A1..A27).
"""
from dataclasses import dataclass, field
from itertools import permutations
import math

import numpy as np
from scipy.optimize import linear_sum_assignment

from .philox import philox4x32_10, uniform53, detlog, DOMAIN_SAMPLE, DOMAIN_ALS_INIT


# ----------------------------------------------------------------------------------------
# Tensors
# ----------------------------------------------------------------------------------------
def view_ijk(T):
    """X[i, j, k] view of a (K, J, I) slice-stream array."""
    return T.transpose(2, 1, 0)


@dataclass
class Coo:
    i: np.ndarray
    j: np.ndarray
    k: np.ndarray
    v: np.ndarray
    dims: tuple

    @property
    def nnz(self):
        return int(self.v.shape[0])


def coo_canonical(i, j, k, v, dims):
    """Sum duplicates (float64, then rounded once to float32), drop exact zeros, sort by
    (k, j, i) (reading R28 / S:98)."""
    i = np.asarray(i, np.int64); j = np.asarray(j, np.int64); k = np.asarray(k, np.int64)
    I, J, K = dims
    lin = (k * J + j) * I + i
    order = np.argsort(lin, kind="stable")
    lin = lin[order]
    vv = np.asarray(v, np.float64)[order]
    uniq, start = np.unique(lin, return_index=True)
    sums = np.add.reduceat(vv, start) if len(vv) else vv
    sums = sums.astype(np.float32)
    keep = sums != 0
    uniq, sums = uniq[keep], sums[keep]
    ii = uniq % I
    jj = (uniq // I) % J
    kk = uniq // (I * J)
    return Coo(ii, jj, kk, sums, (int(I), int(J), int(K)))


def coo_append(X, batch):
    """X <- [X_old; X_new] along mode 3 (Problem 1): batch slices are shifted by K_old."""
    assert X.dims[:2] == batch.dims[:2]
    K_o = X.dims[2]
    return Coo(np.concatenate([X.i, batch.i]), np.concatenate([X.j, batch.j]),
               np.concatenate([X.k, batch.k + K_o]), np.concatenate([X.v, batch.v]),
               (X.dims[0], X.dims[1], K_o + batch.dims[2]))


def dense_append(T, batch):
    """X <- [X_old; X_new] along mode 3 (Problem 1)."""
    assert T.shape[1:] == batch.shape[1:]
    return np.concatenate([T, batch], axis=0)


def coo_to_dense(X):
    I, J, K = X.dims
    T = np.zeros((K, J, I), np.float32)
    T[X.k, X.j, X.i] = X.v
    return T


# ----------------------------------------------------------------------------------------
# Step 1: measure of importance (Eq. 1) in fixed point (readings R1, R2, R3, R7)
# ----------------------------------------------------------------------------------------
MOI_ABS, MOI_SQ = 0, 1


def ceil_log2(v):
    """Smallest integer e with 2**e >= v, for v > 0 (exact, via frexp)."""
    m, e = math.frexp(float(v))      # v = m * 2**e, m in [0.5, 1)
    return e - 1 if m == 0.5 else e


def fixed_point_scale(cap_entries, max_phi):
    """S = 62 - ceil(log2 cap) - ceil(log2 max phi) - 8, clamped to [-60, 120] (reading R7).

    With q = RNE(phi * 2**S), cap entries of phi <= 2**8 * 2**ceil(log2 max_phi) sum to at
    most 2**62, so no int64 marginal can overflow."""
    if max_phi <= 0:
        raise ValueError("DegenerateInput: all-zero tensor")
    S = 62 - ceil_log2(max(int(cap_entries), 1)) - ceil_log2(max_phi) - 8
    return int(min(max(S, -60), 120))


def phi(x, moi):
    """phi(x) = |x| (BASELINE north_star, reading R1) or x^2 (Eq. 1); exact in float64."""
    x = np.asarray(x, np.float32).astype(np.float64)
    return np.abs(x) if moi == MOI_ABS else x * x


def quantize(x, S, moi):
    """q = round-half-even(phi(x) * 2**S) as int64 (reading R7)."""
    return np.rint(phi(x, moi) * (2.0 ** S)).astype(np.int64)


def marginals_dense(T, S, moi=MOI_ABS):
    """x_1(i) = sum_{j,k} q(X(i,j,k)); x_2(j) = sum_{i,k} q; x_3(k) = sum_{i,j} q  (Eq. 1).

    Integer sums are exact, so the loop over frontal slices is just the sum over k."""
    K, J, I = T.shape
    x1 = np.zeros(I, np.int64); x2 = np.zeros(J, np.int64); x3 = np.zeros(K, np.int64)
    for k in range(K):
        q = quantize(T[k], S, moi)          # (J, I)
        x1 += q.sum(axis=0)
        x2 += q.sum(axis=1)
        x3[k] = q.sum()
    return x1, x2, x3


def marginals_coo(X, S, moi=MOI_ABS):
    """Eq. 1 over the stored entries of a sparse tensor (zeros contribute nothing)."""
    I, J, K = X.dims
    q = quantize(X.v, S, moi)
    x1 = np.zeros(I, np.int64); x2 = np.zeros(J, np.int64); x3 = np.zeros(K, np.int64)
    np.add.at(x1, X.i, q); np.add.at(x2, X.j, q); np.add.at(x3, X.k, q)
    return x1, x2, x3


# ----------------------------------------------------------------------------------------
# Step 2: biased sampling without replacement (Alg. 1 line 3 P:211; readings R4-R6)
# ----------------------------------------------------------------------------------------
def sample_size(n, s):
    """|I_s| = min(n, ceil(n/s)) ("I/s", reading R4)."""
    return min(n, -(-n // s))


def sample_keys(w, seed, update_id, rep, mode, domain=DOMAIN_SAMPLE):
    """Exponential keys key_i = E_i / w_i, E_i = -ln(u_i), +inf for w_i = 0 (reading R5).

    u_i comes from Philox4x32-10 with key = seed, counter =
    (i, 0, update_id, domain<<24 | rep<<8 | mode) (reading R6)."""
    w = np.asarray(w, np.int64)
    n = w.shape[0]
    idx = np.arange(n, dtype=np.uint64)
    word3 = (domain << 24) | (rep << 8) | mode
    x0, x1, _, _ = philox4x32_10(idx, 0, update_id, word3, seed)
    E = -detlog(uniform53(x0, x1))
    wf = w.astype(np.float64)           # int64 -> float64, round to nearest
    with np.errstate(divide="ignore"):
        key = np.where(w > 0, E / np.where(w > 0, wf, 1.0), np.inf)
    return key


def sample_mode(w, n_s, seed, update_id, rep, mode):
    """The n_s smallest (key_i, i) pairs in lexicographic order, returned sorted by i.

    Exponential-key sampling realises successive sampling without replacement with
    probability proportional to w (Efraimidis & Spirakis 2006), reading R5."""
    key = sample_keys(w, seed, update_id, rep, mode)
    n = key.shape[0]
    order = np.lexsort((np.arange(n), key))      # primary key, then index
    return np.sort(order[:n_s]).astype(np.int64)


# ----------------------------------------------------------------------------------------
# Step 3: the summary X_s = X(I_s, J_s, K_s U [K+1..K_new])  (Alg. 1 line 4 P:212)
# ----------------------------------------------------------------------------------------
def k_prime(Ks, K_old, K_new):
    """K' = sorted K_s followed by the new slice indices [K_old, K_old+K_new) (readings R8, R9)."""
    return np.concatenate([np.asarray(Ks, np.int64), np.arange(K_old, K_old + K_new, dtype=np.int64)])


def gather_dense(T, Is, Js, Kp):
    """Y(p, q, u) = X(I_s[p], J_s[q], K'[u]); returned as a float32 array indexed [p, q, u]."""
    return view_ijk(T)[np.ix_(np.asarray(Is), np.asarray(Js), np.asarray(Kp))].copy()


def gather_coo(X, Is, Js, Kp):
    """Entries whose three coordinates are all sampled, relabelled to local coordinates
    (position in the sorted lists); canonical (k, j, i) order is preserved."""
    I, J, K = X.dims
    li = -np.ones(I, np.int64); li[np.asarray(Is)] = np.arange(len(Is))
    lj = -np.ones(J, np.int64); lj[np.asarray(Js)] = np.arange(len(Js))
    lk = -np.ones(K, np.int64); lk[np.asarray(Kp)] = np.arange(len(Kp))
    keep = (li[X.i] >= 0) & (lj[X.j] >= 0) & (lk[X.k] >= 0)
    Y = Coo(li[X.i[keep]], lj[X.j[keep]], lk[X.k[keep]], X.v[keep].copy(),
            (len(Is), len(Js), len(Kp)))
    order = np.lexsort((Y.i, Y.j, Y.k))
    return Coo(Y.i[order], Y.j[order], Y.k[order], Y.v[order], Y.dims)


# ----------------------------------------------------------------------------------------
# Step 4: CP-ALS on a summary (readings R10-R12)
# ----------------------------------------------------------------------------------------
def khatri_rao(U, V):
    """Column-wise Kronecker product (Table of symbols): row (a, b) -> U[a]*V[b]."""
    return (U[:, None, :] * V[None, :, :]).reshape(U.shape[0] * V.shape[0], U.shape[1])


def mttkrp(Y, U, mode):
    """M_mode = Y_(mode) (Khatri-Rao product of the other two factors).

    Dense Y is indexed [p, q, u]; the unfolding Y_(mode) has the remaining two modes in
    increasing order, matching khatri_rao's row order.  For a Coo Y the same sum is taken
    over the stored entries:  M_0(i,f) = sum Y(i,j,k) U_1(j,f) U_2(k,f), etc."""
    others = [m for m in range(3) if m != mode]
    if isinstance(Y, Coo):
        idx = (Y.i, Y.j, Y.k)
        v = Y.v.astype(np.float64)
        contrib = v[:, None] * U[others[0]][idx[others[0]]] * U[others[1]][idx[others[1]]]
        M = np.zeros((Y.dims[mode], U[others[0]].shape[1]))
        np.add.at(M, idx[mode], contrib)
        return M
    Yd = np.moveaxis(np.asarray(Y, np.float64), mode, 0)
    unfold = Yd.reshape(Yd.shape[0], -1)
    return unfold @ khatri_rao(U[others[0]], U[others[1]])


def als_init(rows, R, seed, update_id, rep):
    """Initial factors U_m(p, f) = float32(u) with u from Philox counter
    (p*R + f, 0, update_id, ALS_INIT<<24 | rep<<8 | m)  (reading R10); widened to float64."""
    U = []
    for m, n in enumerate(rows):
        c = np.arange(n * R, dtype=np.uint64)
        word3 = (DOMAIN_ALS_INIT << 24) | (rep << 8) | m
        x0, x1, _, _ = philox4x32_10(c, 0, update_id, word3, seed)
        u = uniform53(x0, x1).astype(np.float32).astype(np.float64)
        U.append(u.reshape(n, R))
    return U


def solve_normal(M, V):
    """U = M V^{-1} by Cholesky; if V is not positive definite, the pseudo-inverse from the
    symmetric eigendecomposition with cutoff R*eps*lambda_max (reading R12); exactly
    zero rows / columns of V map to exactly zero rows / columns of V^+ (the exact pseudo-inverse
    of a matrix with a decoupled zero block)."""
    try:
        L = np.linalg.cholesky(V)
        Z = np.linalg.solve(L, M.T)
        return np.linalg.solve(L.T, Z).T, False
    except np.linalg.LinAlgError:
        # rows / columns of V that are exactly zero (a factor column that is exactly zero) are
        # decoupled: V^+ is zero there and the eigendecomposition is taken of the rest, so the
        # zero column stays exactly zero (no rounding-level mixing of eigenvectors into it)
        R = V.shape[0]
        live = np.flatnonzero(np.any(V != 0.0, axis=1))
        P = np.zeros((R, R))
        if live.size:
            Vl = V[np.ix_(live, live)]
            w, Q = np.linalg.eigh(Vl)
            cut = R * np.finfo(np.float64).eps * max(w.max(), 0.0)
            winv = np.where(w > cut, 1.0 / np.where(w > cut, w, 1.0), 0.0)
            P[np.ix_(live, live)] = (Q * winv) @ Q.T
        return M @ P, True


def tensor_sqnorm(Y):
    v = (Y.v if isinstance(Y, Coo) else np.asarray(Y)).astype(np.float64)
    return float(np.sum(v * v))


def cp_als(Y, U, maxit, tol, stats=None):
    """Alternating least squares for CP, starting from factors U (list of 3).

    Each iteration, for m = 0, 1, 2:  M = mttkrp(Y, U, m);  V = *_{n != m} U_n^T U_n;
    U_m = M V^{-1};  lambda_f = ||U_m(:, f)||_2;  U_m(:, f) /= lambda_f if lambda_f > 0.
    fit = 1 - sqrt(max(0, ||Y||^2 - 2 sum_f lambda_f sum_k U_2(k,f) M_2(k,f)
                          + lambda^T (*_n U_n^T U_n) lambda)) / ||Y||.
    Stops when it >= 2 and |fit - fit_prev| < tol, or after maxit iterations (reading R11).
    Returns (lambda, U, fit, iterations, fits); ``stats["pinv"]`` (if a dict is passed) records
    whether any solve fell back to the pseudo-inverse (reading R12)."""
    U = [np.array(u, np.float64) for u in U]
    R = U[0].shape[1]
    normY2 = tensor_sqnorm(Y)
    normY = math.sqrt(normY2)
    lam = np.ones(R)
    fits = []
    fit_prev = None
    it = 0
    for it in range(1, maxit + 1):
        for m in range(3):
            M = mttkrp(Y, U, m)
            V = np.ones((R, R))
            for n in range(3):
                if n != m:
                    V *= U[n].T @ U[n]
            Um, used_pinv = solve_normal(M, V)
            if stats is not None and used_pinv:
                stats["pinv"] = True
            lam = np.sqrt(np.sum(Um * Um, axis=0))
            Um = Um / np.where(lam > 0, lam, 1.0)
            U[m] = Um
        # M is the mode-2 MTTKRP computed with the final U_0, U_1.
        inner = float(np.sum(lam * np.sum(U[2] * M, axis=0)))
        G = (U[0].T @ U[0]) * (U[1].T @ U[1]) * (U[2].T @ U[2])
        mnorm2 = float(lam @ G @ lam)
        resid2 = max(0.0, normY2 - 2.0 * inner + mnorm2)
        fit = 1.0 - math.sqrt(resid2) / normY if normY > 0 else 0.0
        fits.append(fit)
        if it >= 2 and abs(fit - fit_prev) < tol:
            break
        fit_prev = fit
    return lam, U, fits[-1] if fits else 0.0, it, fits


# ----------------------------------------------------------------------------------------
# Step 5: normalise over anchors and match (Lemma 1; readings R13-R16, R26)
# ----------------------------------------------------------------------------------------
def best_assignment(S):
    """pi maximising sum_f S[f, pi(f)].  R <= 8: exhaustive search in lexicographic order
    (first maximum wins = lexicographically smallest pi); otherwise the Hungarian method."""
    R = S.shape[0]
    if R <= 8:
        best, best_pi = -np.inf, None
        for p in permutations(range(R)):
            v = sum(S[f, p[f]] for f in range(R))
            if v > best:
                best, best_pi = v, p
        return np.array(best_pi, np.int64)
    rows, cols = linear_sum_assignment(S, maximize=True)
    pi = np.empty(R, np.int64); pi[rows] = cols
    return pi


@dataclass
class RepMatch:
    pi: np.ndarray           # candidate column pi[f] matches old component f
    scale: list              # per mode, per f: sigma * (old anchor norm / candidate anchor norm)
    lam_hat: np.ndarray      # lambda_hat_f in the old frame
    score: np.ndarray        # S[f, pi f]
    accepted: bool
    congruence: list         # Phi_A, Phi_B, Phi_C
    valid: np.ndarray = None # old component f has a (non-padded) candidate (GetRank, R33)


def _anchor_congruence(old_rows, cand_rows):
    """Congruence Phi(f,g) = <old(:,f), cand(:,g)> / (||old(:,f)|| ||cand(:,g)||) over the anchor
    rows; 0 where a norm is 0 (Lemma 1)."""
    alpha = np.sqrt(np.sum(old_rows * old_rows, axis=0))
    a = np.sqrt(np.sum(cand_rows * cand_rows, axis=0))
    dots = old_rows.T @ cand_rows
    denom = alpha[:, None] * a[None, :]
    Phi = np.where(denom > 0, dots / np.where(denom > 0, denom, 1.0), 0.0)
    return Phi, alpha, a


def match_rep(A, B, C, Is, Js, Ks, lam_p, Up, tau, rnew=None):
    """Match candidate [lam'; A', B', C'] (rows at I_s, J_s, K' = K_s ++ new) to the old model.

    Anchors (reading R14): sampled rows whose old factor row is not all zero; for C only the
    first |K_s| rows of C' (old slices).  S = (|Phi_A| + |Phi_B| + |Phi_C|)/3 (reading R15),
    pi = argmax sum S, sigma = sign Phi(f, pi f) (0 -> +1), rescale to the old frame by the
    anchor norms and lambda_hat_f = lam'_{pi f} sigma_A sigma_B sigma_C abc/(alpha beta gamma)
    (reading R16).  Accepted iff min_f S(f, pi f) >= tau (reading R26).

    rnew < R (GetRank, reading R33): the candidate has R_new real columns followed by zero
    padding; zero columns have congruence 0, so the assignment matches the R_new real columns to
    their best old components and only those (valid f: pi f < R_new) count for the
    acceptance test and the merge."""
    nKs = len(Ks)
    olds = [A[np.asarray(Is)], B[np.asarray(Js)], C[np.asarray(Ks)]]
    cands = [Up[0], Up[1], Up[2][:nKs]]
    Phis, alphas, cs = [], [], []
    for o, c in zip(olds, cands):
        P = np.any(o != 0.0, axis=1)
        Phi, alpha, a = _anchor_congruence(o[P], c[P])
        Phis.append(Phi); alphas.append(alpha); cs.append(a)
    S = (np.abs(Phis[0]) + np.abs(Phis[1]) + np.abs(Phis[2])) / 3.0
    pi = best_assignment(S)
    R = len(pi)
    scale = []
    lam_hat = np.array(lam_p, np.float64)[pi].copy()
    for m in range(3):
        sig = np.where(Phis[m][np.arange(R), pi] < 0, -1.0, 1.0)
        al, a = alphas[m], cs[m][pi]
        ok = (al > 0) & (a > 0)
        scale.append(np.where(ok, sig * al / np.where(ok, a, 1.0), 0.0))
        lam_hat = np.where(ok, lam_hat * sig * a / np.where(ok, al, 1.0), 0.0)
    score = S[np.arange(R), pi]
    valid = pi < (R if rnew is None else rnew)
    return RepMatch(pi, scale, lam_hat, score, bool(score[valid].min() >= tau), Phis, valid)


def warm_init(U0, st, Is, Js, Ks):
    """Warm start (reading R34): the summary ALS starts from the model's
    rows instead of the random point -- U_0 = A(I_s, :), U_1 = B(J_s, :), the first |K_s| rows of
    U_2 = C(K_s, :) diag(lambda) (product rounded to float32, as the model is held in float32);
    the K_n new slices start at zero (the model has no rows for them; the first mode-0 and
    mode-1 solves then see the old slices only, and the mode-2 solve fills them)."""
    if st.cfg.getrank:
        raise ValueError("warm_start and getrank are exclusive (R34)")
    f32 = lambda x: np.asarray(x, np.float32).astype(np.float64)
    U2 = np.zeros_like(U0[2])
    U2[: len(Ks)] = (np.asarray(st.C, np.float32)[np.asarray(Ks)] * np.asarray(st.lam, np.float32)[None, :]).astype(np.float64)
    return [f32(st.A[np.asarray(Is)]), f32(st.B[np.asarray(Js)]), U2]


def rescaled(Up, rm, m):
    """Candidate factor of mode m in the old frame: U~(:, f) = scale_f * U'(:, pi f)."""
    return Up[m][:, rm.pi] * rm.scale[m][None, :]


# ----------------------------------------------------------------------------------------
# Whole update (Alg. 1) and state
# ----------------------------------------------------------------------------------------
@dataclass
class Config:
    R: int
    s: tuple                 # per-mode sampling factors
    r: int
    seed: int
    maxit: int = 30
    tol: float = 1e-6
    moi: int = MOI_ABS
    tau: float = 0.9         # reading R26 (0 = paper-literal)
    merge_policy: int = 0    # 0 = zero entries only, 1 = overwrite sampled rows
    getrank: bool = False    # GetRank before each summary decomposition (Alg. 2; R29-R33)
    getrank_trials: int = 1
    getrank_threshold: float = 90.0
    warm_start: bool = False # summary ALS started from the model's rows
    pipelined: bool = False  # sample update t+1 from update t's marginals


@dataclass
class State:
    cfg: Config
    X: object                # dense (K,J,I) float32 array or Coo
    lam: np.ndarray
    A: np.ndarray
    B: np.ndarray
    C: np.ndarray
    S: int
    max_phi_log2: int        # ceil(log2 max phi(X0)): the fixed-point range (reading R7)
    update_id: int = 0
    last: dict = field(default_factory=dict)
    marg: tuple = None       # pipelined (R36): marginals of the stored tensor, kept for the next update

    @property
    def dense(self):
        return not isinstance(self.X, Coo)

    @property
    def dims(self):
        if self.dense:
            K, J, I = self.X.shape
            return I, J, K
        return self.X.dims


def _values(X):
    return (X.v if isinstance(X, Coo) else np.asarray(X).ravel())


def init_factors(X0, cfg, lam, A, B, C, cap_entries):
    """State from given float32 factors (the fp32 model widened exactly to fp64)."""
    vals = _values(X0)
    max_phi = float(phi(vals, cfg.moi).max()) if vals.size else 0.0
    S = fixed_point_scale(cap_entries, max_phi)
    f64 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    return State(cfg, X0, f64(lam), f64(A), f64(B), f64(C), S, ceil_log2(max_phi))


def init_als(X0, cfg, cap_entries, maxit=1000, tol=1e-6):
    """Initial decomposition of the existing data by full CP-ALS ("10% as existing")."""
    if isinstance(X0, Coo):
        Y, rows = X0, X0.dims
    else:
        Y = view_ijk(X0)
        rows = Y.shape
    U0 = als_init(rows, cfg.R, cfg.seed, 0, 0)
    lam, U, fit, it, _ = cp_als(Y, U0, maxit, tol)
    st = init_factors(X0, cfg, np.ones(cfg.R, np.float32), U[0], U[1], U[2], cap_entries)
    st.lam, st.A, st.B, st.C = lam, U[0], U[1], U[2]
    return st


RECOMPUTE_REP = 255   # reading R35: the CP_ALS baseline's Philox repetition index


def recompute(X, R, seed, update_id, maxit, tol):
    """The paper's CP_ALS baseline ("re-compute CP using CP_ALS every time a new batch
    update arrives"): full CP-ALS of the whole current tensor X from the Philox point
    als_init(..., update_id, rep = 255) (reading R35).  Returns (lambda, [A, B, C], fit, iters)."""
    if isinstance(X, Coo):
        Y, rows = X, X.dims
    else:
        Y = view_ijk(X)
        rows = Y.shape
    U0 = als_init(rows, R, seed, update_id, RECOMPUTE_REP)
    lam, U, fit, it, _ = cp_als(Y, U0, maxit, tol)
    return lam, U, fit, it


def relative_fitness(X, model_s, model_b):
    """Relative Fitness = ||X - X_SamBaTen|| / ||X - X_BaseLine||: lower is better."""
    return relative_error(X, *model_s) / relative_error(X, *model_b)


class FixedPointRange(Exception):
    pass


class BatchRejected(Exception):
    pass


def update(st, batch, keep_reps=False):
    """One SamBaTen update (Alg. 1) of state ``st`` with batch ``batch``.

    Returns a dict with the sample sets, per-rep ALS/match results and fits.  On error the
    state is left unchanged."""
    cfg = st.cfg
    I, J, K_o = st.dims
    dense = st.dense
    K_n = batch.shape[0] if dense else batch.dims[2]
    if K_n == 0:
        raise ValueError("EmptyBatch")
    bvals = _values(batch)
    if bvals.size and float(phi(bvals, cfg.moi).max()) > 2.0 ** (st.max_phi_log2 + 8):
        raise FixedPointRange("batch value outside the fixed-point range")
    uid = st.update_id + 1
    # a0: append (Problem 1)
    X = dense_append(st.X, batch) if dense else coo_append(st.X, batch)
    # a1: marginals over X_old U X_new (readings R2, R3)
    x1, x2, x3 = (marginals_dense(X, st.S, cfg.moi) if dense else marginals_coo(X, st.S, cfg.moi))
    sx = (x1, x2, x3)
    if cfg.pipelined:
        # reading R36 ("X is the tensor prior to the update"): the
        # samples come from the marginals of the tensor BEFORE this batch (kept from the
        # previous update, or computed from the stored tensor after init), so the sampling and
        # the gather need not wait for this update's marginal pass
        sx = st.marg if st.marg is not None else (
            marginals_dense(st.X, st.S, cfg.moi) if dense else marginals_coo(st.X, st.S, cfg.moi))
    reps = []
    for rho in range(cfg.r):
        # a2: sampling (K_s only from the old slices, reading R2 / S:302)
        Is = sample_mode(sx[0], sample_size(I, cfg.s[0]), cfg.seed, uid, rho, 0)
        Js = sample_mode(sx[1], sample_size(J, cfg.s[1]), cfg.seed, uid, rho, 1)
        Ks = sample_mode(sx[2][:K_o], sample_size(K_o, cfg.s[2]), cfg.seed, uid, rho, 2)
        Kp = k_prime(Ks, K_o, K_n)
        # a3: gather the summary
        Y = gather_dense(X, Is, Js, Kp) if dense else gather_coo(X, Is, Js, Kp)
        # a4: CP-ALS at the universal rank R, or at the rank GetRank estimates for the
        # summary (Alg. 2; dense summaries, readings R29-R33)
        R_use = cfg.R
        if cfg.getrank:
            from .getrank import getrank
            R_use, _ = getrank(Y, cfg.R, cfg.getrank_trials, cfg.seed, cfg.maxit, cfg.tol,
                               cfg.getrank_threshold, rep_base=rho * cfg.getrank_trials)
        U0 = als_init((len(Is), len(Js), len(Kp)), R_use, cfg.seed, uid, rho)
        if cfg.warm_start:
            U0 = warm_init(U0, st, Is, Js, Ks)
        als_stats = {"pinv": False}
        lam_p, Up, fit, its, _ = cp_als(Y, U0, cfg.maxit, cfg.tol, als_stats)
        if R_use < cfg.R:   # zero columns up to R (reading R33)
            pad = cfg.R - R_use
            lam_p = np.concatenate([lam_p, np.zeros(pad)])
            Up = [np.hstack([u, np.zeros((u.shape[0], pad))]) for u in Up]
        # a5: match against the batch-start snapshot
        rm = match_rep(st.A, st.B, st.C, Is, Js, Ks, lam_p, Up, cfg.tau, rnew=R_use)
        reps.append(dict(Is=Is, Js=Js, Ks=Ks, Kp=Kp, Y=Y if keep_reps else None, lam_p=lam_p,
                         Up=Up, fit=fit, iters=its, match=rm, rank=R_use, pinv=als_stats["pinv"]))
    acc = [rp for rp in reps if rp["match"].accepted]
    if not acc:
        raise BatchRejected("every repetition failed the acceptance test")
    # a6: merge (readings R17-R20), element by element over the accepted reps that
    # carry component f (all of them unless GetRank reduced a rep's rank, reading R33)
    A, B, C = st.A.copy(), st.B.copy(), st.C.copy()
    for m, (F, key) in enumerate(((A, "Is"), (B, "Js"), (C, "Ks"))):
        tot = np.zeros_like(F); cnt = np.zeros_like(F)
        for rp in acc:
            rows = rp[key]
            v = rp["match"].valid.astype(np.float64)
            Ut = rescaled(rp["Up"], rp["match"], m)[: len(rows)]
            tot[rows] += Ut * v[None, :]
            cnt[rows] += v[None, :]
        hit = cnt > 0
        mean = np.where(hit, tot / np.where(hit, cnt, 1.0), 0.0)
        if cfg.merge_policy == 0:
            F[:] = np.where(hit & (F == 0.0), mean, F)
        else:
            F[:] = np.where(hit, mean, F)
    C_new = np.zeros((K_n, cfg.R))
    nval = np.zeros(cfg.R)
    lam_hat = np.zeros(cfg.R)
    for rp in acc:
        v = rp["match"].valid.astype(np.float64)
        C_new += rescaled(rp["Up"], rp["match"], 2)[len(rp["Ks"]):] * v[None, :]
        lam_hat += rp["match"].lam_hat * v
        nval += v
    C_new = np.where(nval > 0, C_new / np.where(nval > 0, nval, 1.0), 0.0)
    lam = np.where(nval > 0, (st.lam + lam_hat / np.where(nval > 0, nval, 1.0)) / 2.0, st.lam)
    # commit
    st.X, st.A, st.B, st.C, st.lam = X, A, B, np.vstack([C, C_new]), lam
    st.update_id = uid
    if cfg.pipelined:
        st.marg = (x1, x2, x3)
    st.last = dict(x=(x1, x2, x3), reps=reps, fit_summary=float(np.mean([rp["fit"] for rp in reps])),
                   rejected=[i for i, rp in enumerate(reps) if not rp["match"].accepted])
    return st.last


# ----------------------------------------------------------------------------------------
# Step 7/8: metrics (readings R21, R24)
# ----------------------------------------------------------------------------------------
def relative_error(X, lam, A, B, C):
    """||X - [[lam; A, B, C]]||_F / ||X||_F.  Dense materialisation up to 1e6
    entries; otherwise ||X||^2 - 2<X, M> + ||M||^2 with <X, M> = sum_f lam_f sum_k C(k,f)
    M_2(k,f), M_2 the mode-3 MTTKRP of X with A, B."""
    lam = np.asarray(lam, np.float64)
    A, B, C = (np.asarray(U, np.float64) for U in (A, B, C))
    if isinstance(X, Coo):
        I, J, K = X.dims
        normX2 = tensor_sqnorm(X)
        if I * J * K <= 10 ** 6:
            D = coo_to_dense(X)
            return relative_error(D, lam, A, B, C)
        M2 = mttkrp(X, [A, B, C], 2)
    else:
        K, J, I = X.shape
        normX2 = tensor_sqnorm(X)
        if I * J * K <= 10 ** 6:
            model = np.einsum("f,if,jf,kf->ijk", lam, A, B, C)
            diff = view_ijk(X).astype(np.float64) - model
            return math.sqrt(float(np.sum(diff * diff)) / normX2)
        M2 = np.zeros((K, A.shape[1]))
        for k in range(K):   # mode-3 MTTKRP slice by slice: M_2(k,f) = sum_ij X(i,j,k) A(i,f) B(j,f)
            M2[k] = np.einsum("ji,if,jf->f", X[k].astype(np.float64), A, B)
    inner = float(np.sum(lam * np.sum(C * M2, axis=0)))
    G = (A.T @ A) * (B.T @ B) * (C.T @ C)
    resid2 = max(0.0, normX2 - 2.0 * inner + float(lam @ G @ lam))
    return math.sqrt(resid2 / normX2)


def fms(m1, m2):
    """Factor match score (Eq. 2, reading R24): absorb all scale into lambda,
    score(f,g) = (1 - |l1_f - l2_g| / max(l1_f, l2_g)) * prod_n |u1_n(:,f)^T u2_n(:,g)|,
    best assignment, mean over components; in [0, 1]."""
    def norm(m):
        lam, Us = np.asarray(m[0], np.float64), [np.asarray(U, np.float64) for U in m[1:]]
        lb = np.abs(lam).copy()
        out = []
        for U in Us:
            n = np.sqrt(np.sum(U * U, axis=0))
            lb = lb * n
            out.append(U / np.where(n > 0, n, 1.0))
        return lb, out
    l1, U1 = norm(m1)
    l2, U2 = norm(m2)
    R = len(l1)
    S = np.ones((R, R))
    mx = np.maximum(l1[:, None], l2[None, :])
    S *= np.where(mx > 0, 1.0 - np.abs(l1[:, None] - l2[None, :]) / np.where(mx > 0, mx, 1.0), 1.0)
    for a, b in zip(U1, U2):
        S *= np.abs(a.T @ b)
    pi = best_assignment(S)
    return float(np.mean(S[np.arange(R), pi]))
