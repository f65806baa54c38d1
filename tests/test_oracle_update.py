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
