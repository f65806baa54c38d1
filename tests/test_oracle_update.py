"""Pins for the oracle's whole update (Alg. 1; merge P:216-227, readings R17-R20, R26)."""
import copy

import numpy as np
import pytest

from oracle import sambaten as O
from synth import planted_dense, split_dense, CONFIGS


def _state_from_truth(T0, truth, cfg, cap):
    lam, A, B, C = truth
    return O.init_factors(T0, cfg, lam, A, B, C[: T0.shape[0]], cap)


def test_update_from_truth_reproduces_new_rows():
    """SURVEY §8(c) merge pin: planted noiseless tensor, state initialised from the truth,
    ALS run to convergence: C_new = C_true(new rows), lambda unchanged, FMS vs truth ~ 1."""
    T, truth = planted_dense(40, 40, 40, 3, noise=0.0, seed=3)
    T0, batches = split_dense(T, 30, 10)
    cfg = O.Config(R=3, s=(2, 2, 2), r=4, seed=1, maxit=1000, tol=1e-12)
    st = _state_from_truth(T0, truth, cfg, T.size)
    C_true = np.asarray(truth[3], np.float32).astype(np.float64)
    info = O.update(st, batches[0])
    assert info["rejected"] == []
    new = st.C[30:]
    assert np.linalg.norm(new - C_true[30:]) / np.linalg.norm(C_true[30:]) <= 1e-5
    assert np.allclose(st.lam, 1.0, atol=1e-5)
    assert O.fms((st.lam, st.A, st.B, st.C), (np.ones(3), truth[1], truth[2], C_true)) >= 0.999
    assert O.relative_error(st.X, st.lam, st.A, st.B, st.C) <= 1e-5


def test_c1_config_accuracy():
    """BASELINE configs[0] (C1) end to end from a full initial ALS: fit at the 1% noise floor
    (SURVEY §8(c) expected accuracy 0.987-0.990; orientation, checked loosely)."""
    w = CONFIGS["C1"]
    T, truth = planted_dense(w.I, w.J, w.K, w.R, noise=w.noise, seed=w.seed)
    T0, batches = split_dense(T, w.K0, w.batch)
    cfg = O.Config(R=w.R, s=(w.s,) * 3, r=w.r, seed=0, maxit=w.maxit, tol=w.tol)
    st = O.init_als(T0, cfg, T.size)
    O.update(st, batches[0])
    assert st.C.shape == (50, 3)
    assert 1 - O.relative_error(st.X, st.lam, st.A, st.B, st.C) > 0.98


def test_zero_entry_only_merge_and_bookkeeping():
    """S:291 row counts; S:292 cells that were nonzero stay bit-identical; zero cells of
    sampled rows get filled."""
    T, truth = planted_dense(30, 30, 30, 2, noise=0.01, seed=4)
    T0, batches = split_dense(T, 20, 5)
    cfg = O.Config(R=2, s=(2, 2, 2), r=3, seed=2, maxit=30, tol=0.0)
    st = _state_from_truth(T0, truth, cfg, T.size)
    st.A[3, :] = 0.0                       # a row "not yet computed"
    st.B[5, 1] = 0.0
    A0, B0, C0 = st.A.copy(), st.B.copy(), st.C.copy()
    info = O.update(st, batches[0])
    assert st.A.shape == A0.shape and st.B.shape == B0.shape and st.C.shape == (25, 2)
    nz = A0 != 0
    assert np.array_equal(st.A[nz], A0[nz])
    assert np.array_equal(st.B[B0 != 0], B0[B0 != 0])
    assert np.array_equal(st.C[:20][C0 != 0], C0[C0 != 0])
    sampled_A = set(np.concatenate([rp["Is"] for i, rp in enumerate(info["reps"]) if i not in info["rejected"]]))
    if 3 in sampled_A:
        assert np.all(st.A[3] != 0)
    else:
        assert np.all(st.A[3] == 0)


def test_errors_leave_state_unchanged():
    T, truth = planted_dense(20, 20, 20, 2, noise=0.01, seed=5)
    T0, batches = split_dense(T, 15, 5)
    cfg = O.Config(R=2, s=(2, 2, 2), r=2, seed=3, maxit=5, tol=0.0, tau=1.01)   # reject all
    st = _state_from_truth(T0, truth, cfg, T.size)
    snap = copy.deepcopy(st)
    with pytest.raises(O.BatchRejected):
        O.update(st, batches[0])
    with pytest.raises(ValueError):
        O.update(st, batches[0][:0])
    big = batches[0].copy()
    big[0, 0, 0] = 2.0 ** (st.max_phi_log2 + 9)
    st.cfg = O.Config(R=2, s=(2, 2, 2), r=2, seed=3, maxit=5, tol=0.0)
    with pytest.raises(O.FixedPointRange):
        O.update(st, big)
    for a in ("A", "B", "C", "lam", "X"):
        assert np.array_equal(getattr(st, a), getattr(snap, a))
    assert st.update_id == snap.update_id


def test_update_deterministic():
    """identical seeds and inputs give a bit-identical state."""
    T, truth = planted_dense(24, 24, 24, 2, noise=0.01, seed=6)
    T0, batches = split_dense(T, 18, 6)
    cfg = O.Config(R=2, s=(2, 2, 2), r=3, seed=4, maxit=10, tol=0.0)
    a = _state_from_truth(T0, truth, cfg, T.size)
    b = _state_from_truth(T0, truth, cfg, T.size)
    O.update(a, batches[0]); O.update(b, batches[0])
    for n in ("A", "B", "C", "lam"):
        assert np.array_equal(getattr(a, n), getattr(b, n))


def test_sampled_work_bound_and_k_prime():
    """every summary has dims <= (ceil(I/s), ceil(J/s), ceil(K/s) + K_new); K_s is
    drawn from the old slices only and the new slices are appended whole."""
    T, truth = planted_dense(21, 17, 26, 2, noise=0.01, seed=7)
    T0, batches = split_dense(T, 20, 6)
    cfg = O.Config(R=2, s=(3, 2, 4), r=3, seed=5, maxit=3, tol=0.0)
    st = _state_from_truth(T0, truth, cfg, T.size)
    info = O.update(st, batches[0])
    for rp in info["reps"]:
        assert len(rp["Is"]) == 7 and len(rp["Js"]) == 9 and len(rp["Ks"]) == 5
        assert rp["Ks"].max() < 20 and list(rp["Kp"][5:]) == list(range(20, 26))


def test_coo_update_runs_and_matches_dense_of_same_tensor():
    """The sparse path on a COO tensor equals the dense path on its densification (same
    samples, same summaries up to representation, same factors)."""
    T, truth = planted_dense(16, 14, 12, 2, noise=0.0, seed=8)
    T[np.random.default_rng(0).random(T.shape) < 0.3] = 0
    T0, batches = split_dense(T, 9, 3)
    cfg = O.Config(R=2, s=(2, 2, 2), r=2, seed=6, maxit=8, tol=0.0, tau=0.0)
    sd = _state_from_truth(T0, truth, cfg, T.size)

    def coo(A):
        kk, jj, ii = np.nonzero(A)
        return O.coo_canonical(ii, jj, kk, A[kk, jj, ii], (A.shape[2], A.shape[1], A.shape[0]))
    sc = O.init_factors(coo(T0), cfg, *(np.asarray(x, np.float32) for x in (truth[0], truth[1], truth[2], truth[3][:9])), T.size)
    assert sc.S == sd.S
    di = O.update(sd, batches[0])
    ci = O.update(sc, coo(batches[0]))
    for a, b in zip(di["x"], ci["x"]):
        assert np.array_equal(a, b)
    for ra, rb in zip(di["reps"], ci["reps"]):
        assert np.array_equal(ra["Is"], rb["Is"]) and np.array_equal(ra["Kp"], rb["Kp"])
    assert np.allclose(sd.C, sc.C, rtol=1e-9, atol=1e-12)
    assert np.allclose(sd.lam, sc.lam, rtol=1e-9)


def _noiseless_from_truth(seed, R=3, I=30, K0=24, Kn=6, r=4, s=2):
    T, truth = planted_dense(I, I, K0 + Kn, R, noise=0.0, seed=seed)
    T0, batches = split_dense(T, K0, Kn)
    cfg = O.Config(R=R, s=(s, s, s), r=r, seed=seed, maxit=1000, tol=1e-13, tau=0.9)
    st = _state_from_truth(T0, truth, cfg, T.size)
    f32 = lambda x: np.asarray(x, np.float32).astype(np.float64)
    return st, batches, (np.ones(R), f32(truth[1]), f32(truth[2]), f32(truth[3]))


def test_zeroed_rows_restored_to_truth():
    """P:216 / P:256 ("update only zero entries"), P:198 with reading R14 (rows not yet
    computed are no anchors), R16 (old-frame rescale), R17 (mean over the reps that sampled
    the row).  Noiseless planted tensor, model = truth with some rows of A and B zeroed, ALS
    converged: every zeroed row that some accepted rep sampled comes back as the TRUE row (the
    anchor norms exclude the zeroed rows; a sum instead of a mean, or zero rows kept as anchors,
    scale it), every zeroed row no rep sampled stays exactly zero, every other cell is
    bit-unchanged."""
    st, batches, (lam_t, A_t, B_t, C_t) = _noiseless_from_truth(seed=11)
    zA, zB = [1, 4, 7, 12, 20, 27], [0, 5, 9, 18, 29]
    st.A[zA] = 0.0
    st.B[zB] = 0.0
    A0, B0 = st.A.copy(), st.B.copy()
    info = O.update(st, batches[0])
    assert info["rejected"] == []
    hitA = set(np.concatenate([rp["Is"] for rp in info["reps"]]).tolist())
    hitB = set(np.concatenate([rp["Js"] for rp in info["reps"]]).tolist())
    restored = 0
    for F, F0, T, zs, hit in ((st.A, A0, A_t, zA, hitA), (st.B, B0, B_t, zB, hitB)):
        for i in zs:
            if i in hit:
                assert np.linalg.norm(F[i] - T[i]) <= 1e-6 * np.linalg.norm(T[i]), (i, F[i], T[i])
                restored += 1
            else:
                assert np.all(F[i] == 0.0)
        keep = np.ones(F.shape[0], bool); keep[zs] = False
        assert np.array_equal(F[keep], F0[keep])
    assert restored >= 6          # the pin exercises the fill on several rows of both modes


def test_zeroed_row_sampled_by_one_rep_only():
    """The fill value of a row hit by exactly one accepted rep is that rep's old-frame row
    (R17: the mean over one rep), and a row hit by several reps is their mean: with a noisy
    tensor the reps' rows differ, so the two cases separate a mean from a sum or a first-rep
    pick.  Pinned by construction: the expected rows are re-derived here from the reps'
    candidate factors by the old-frame rescale of Lemma 1's equality case (alpha/a over the
    anchors) computed independently with numpy on the anchor rows."""
    T, truth = planted_dense(30, 30, 30, 3, noise=0.01, seed=12)
    T0, batches = split_dense(T, 24, 6)
    cfg = O.Config(R=3, s=(3, 3, 3), r=3, seed=5, maxit=200, tol=1e-10, tau=0.0)
    st = _state_from_truth(T0, truth, cfg, T.size)
    zA = list(range(0, 30, 3))
    st.A[zA] = 0.0
    A0 = st.A.copy()
    info = O.update(st, batches[0])
    counts = {i: [k for k, rp in enumerate(info["reps"]) if i in set(rp["Is"].tolist())] for i in zA}
    assert any(len(v) == 1 for v in counts.values()) and any(len(v) >= 2 for v in counts.values())
    for i, reps in counts.items():
        if not reps:
            assert np.all(st.A[i] == 0.0)
            continue
        rows = []
        for k in reps:
            rp = info["reps"][k]
            Is = rp["Is"]
            anc = np.any(A0[Is] != 0.0, axis=1)
            old, cand = A0[Is][anc], rp["Up"][0][anc]
            pi = rp["match"].pi
            row = np.empty(3)
            for f in range(3):
                g = pi[f]
                dot = float(old[:, f] @ cand[:, g])
                row[f] = np.sign(dot or 1.0) * np.linalg.norm(old[:, f]) / np.linalg.norm(cand[:, g]) \
                    * rp["Up"][0][list(Is).index(i), g]
            rows.append(row)
        assert np.allclose(st.A[i], np.mean(rows, axis=0), rtol=1e-12, atol=1e-14)


def test_lambda_average_of_old_and_new():
    """P:227 "lambda = (lambda + new value)/2" with R19 (new value = mean of lambda_hat over the
    accepted reps) and R16 (lambda_hat in the old frame).  Model = truth with lambda doubled on a
    noiseless tensor: every converged rep recovers lambda_hat = 1 (the true scale relative to
    the model's factor norms), so the update must give lambda = (2 + 1)/2 = 1.5 -- lambda <-
    mean lambda_hat gives 1, leaving lambda unchanged gives 2."""
    st, batches, _ = _noiseless_from_truth(seed=13)
    st.lam = 2.0 * st.lam
    info = O.update(st, batches[0])
    assert info["rejected"] == []
    for rp in info["reps"]:
        assert np.allclose(rp["match"].lam_hat, 1.0, rtol=1e-5)
    assert np.allclose(st.lam, 1.5, rtol=1e-5)


def test_pinv_zero_column_equals_reduced_rank_als():
    """R12 pseudo-inverse fallback: a start with factor column f of U_1 exactly zero makes every
    normal matrix singular (zero row / column f), so every solve takes the pseudo-inverse
    (cutoff R*eps*lambda_max).  Mathematically the pinv solve then equals the Cholesky solve of
    the R-1 other columns and keeps column f at zero: cp_als with the zero column must equal
    cp_als at rank R-1 from the same start without column f (a different code path: every
    normal matrix there is positive definite)."""
    T, truth = planted_dense(12, 11, 10, 3, noise=0.01, seed=14)
    Y = O.view_ijk(T).astype(np.float64)
    U0 = O.als_init(Y.shape, 3, 0, 1, 0)
    U0[1][:, 1] = 0.0
    st = {"pinv": False}
    lam, U, fit, it, _ = O.cp_als(Y, U0, 40, 0.0, st)
    assert st["pinv"]
    red = [np.delete(u, 1, axis=1) for u in U0]
    st2 = {"pinv": False}
    lam2, U2, fit2, it2, _ = O.cp_als(Y, red, 40, 0.0, st2)
    assert not st2["pinv"]
    assert lam[1] == 0.0 and all(np.all(u[:, 1] == 0.0) for u in U)
    assert np.allclose(np.delete(lam, 1), lam2, rtol=1e-8)
    for u, u2 in zip(U, U2):
        assert np.allclose(np.delete(u, 1, axis=1), u2, rtol=1e-7, atol=1e-10)
    assert abs(fit - fit2) <= 1e-10


def test_update_pinv_path_zero_model_column():
    """A model component whose B column is all zero (a warm start from it, R34) drives every
    summary ALS through the pseudo-inverse (R12); the paper-literal merge (tau = 0) then merges
    a zero candidate column: lambda_hat_f = 0 (no anchor norm, R16) so lambda_f halves (P:227,
    R19), and the new C rows of component f are zero."""
    T, truth = planted_dense(24, 24, 24, 3, noise=0.01, seed=15)
    T0, batches = split_dense(T, 18, 6)
    cfg = O.Config(R=3, s=(2, 2, 2), r=3, seed=6, maxit=10, tol=0.0, tau=0.0, warm_start=True)
    st = _state_from_truth(T0, truth, cfg, T.size)
    st.B[:, 2] = 0.0
    lam0 = st.lam.copy()
    info = O.update(st, batches[0])
    assert all(rp["pinv"] for rp in info["reps"])
    assert st.lam[2] == lam0[2] / 2.0
    assert np.all(st.C[18:, 2] == 0.0)


def test_pipelined_samples_from_the_previous_tensor():
    """R36: the pipelined update samples from the marginals of the tensor
    BEFORE its batch -- pinned against the plain update run on the old tensor's
    marginals: the first pipelined update's samples equal the samples the oracle draws from
    marginals_dense(X_old); the second's those of X_1 (the first batch included); a rejected
    batch keeps the stored marginals."""
    T, truth = planted_dense(30, 26, 34, 3, noise=0.01, seed=17)
    T0, batches = split_dense(T, 24, 5)
    cfg = O.Config(R=3, s=(2, 2, 2), r=3, seed=7, maxit=10, tol=0.0, tau=0.0, pipelined=True)
    st = _state_from_truth(T0, truth, cfg, T.size)
    X = T0
    for b in batches:
        x1, x2, x3 = O.marginals_dense(X, st.S)
        info = O.update(st, b)
        uid = st.update_id
        for rho, rp in enumerate(info["reps"]):
            assert np.array_equal(rp["Is"], O.sample_mode(x1, O.sample_size(30, 2), 7, uid, rho, 0))
            assert np.array_equal(rp["Js"], O.sample_mode(x2, O.sample_size(26, 2), 7, uid, rho, 1))
            assert np.array_equal(rp["Ks"], O.sample_mode(x3, O.sample_size(X.shape[0], 2), 7, uid, rho, 2))
        X = np.concatenate([X, b])
        for a, c in zip(st.marg, O.marginals_dense(X, st.S)):
            assert np.array_equal(a, c)
    marg = st.marg
    st.cfg = O.Config(R=3, s=(2, 2, 2), r=3, seed=7, maxit=2, tol=0.0, tau=1.5, pipelined=True)
    with pytest.raises(O.BatchRejected):
        O.update(st, batches[0])
    assert st.marg is marg
