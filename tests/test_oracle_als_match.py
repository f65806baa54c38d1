"""Pins for the oracle's CP-ALS, matching (Lemma 1) and metrics
(P:409-413)."""
from itertools import permutations

import numpy as np
import pytest

from oracle import sambaten as O


def planted(shape, R, seed, noise=0.0):
    rng = np.random.default_rng(seed)
    U = [rng.random((n, R)) for n in shape]
    Y = np.einsum("if,jf,kf->ijk", *U)
    if noise:
        Y = Y + noise * np.linalg.norm(Y) / np.sqrt(Y.size) * rng.standard_normal(Y.shape)
    return Y, U


def test_als_recovers_planted_noiseless():
    """BASELINE north_star pin: planted noiseless rank-R tensor -> fit > 0.999 (here with 500
    iterations, reading R27) and FMS vs truth >= 0.99."""
    Y, U = planted((50, 50, 30), 3, 0)
    U0 = O.als_init(Y.shape, 3, 0, 0, 0)
    lam, Uh, fit, it, fits = O.cp_als(Y, U0, 500, 1e-12)
    assert fit > 0.999
    assert O.fms((lam, *Uh), (np.ones(3), *U)) >= 0.99


def test_als_rank1_recovery():
    """5 a o b o c with unit vectors -> lambda = 5, |columns| = (a, b, c)."""
    rng = np.random.default_rng(1)
    a, b, c = (v / np.linalg.norm(v) for v in (rng.random(6), rng.random(5), rng.random(4)))
    Y = 5.0 * np.einsum("i,j,k->ijk", a, b, c)
    lam, Uh, fit, _, _ = O.cp_als(Y, O.als_init(Y.shape, 1, 3, 0, 0), 50, 1e-14)
    assert abs(lam[0] - 5.0) < 1e-9
    for u, v in zip(Uh, (a, b, c)):
        assert np.allclose(np.abs(u[:, 0]), v, atol=1e-9)
    assert fit > 1 - 1e-9


def test_als_fit_monotone_and_equals_relative_error():
    """S:158 objective non-increasing; the fit formula equals 1 - relative error of the
    returned model computed by dense materialisation."""
    Y, _ = planted((12, 11, 10), 4, 2, noise=0.1)
    lam, Uh, fit, it, fits = O.cp_als(Y, O.als_init(Y.shape, 4, 5, 0, 0), 40, 0.0)
    assert it == 40
    assert np.all(np.diff(fits) >= -1e-9)
    model = np.einsum("f,if,jf,kf->ijk", lam, *Uh)
    rel = np.linalg.norm(Y - model) / np.linalg.norm(Y)
    assert abs((1 - rel) - fit) < 1e-9


def test_als_normalised_columns_and_invariance():
    Y, _ = planted((8, 7, 6), 2, 3, noise=0.05)
    lam, Uh, *_ = O.cp_als(Y, O.als_init(Y.shape, 2, 1, 0, 0), 10, 0.0)
    for U in Uh:
        assert np.allclose(np.linalg.norm(U, axis=0), 1.0, atol=1e-12)


def test_als_init_is_float32_rounded_uniform():
    U = O.als_init((4, 3, 2), 2, 7, 1, 3)
    for m, u in enumerate(U):
        assert u.shape == ((4, 3, 2)[m], 2)
        assert np.all((u > 0) & (u <= 1))
        assert np.array_equal(u, u.astype(np.float32).astype(np.float64))
    assert not np.array_equal(U[0][:2], U[1][:2])


def test_solve_normal_pinv_fallback():
    M = np.array([[1.0, 2.0]])
    V = np.array([[1.0, 1.0], [1.0, 1.0]])        # singular
    U, used = O.solve_normal(M, V)
    assert used
    assert np.allclose(U, M @ np.linalg.pinv(V))


def test_best_assignment_brute_force_lexicographic():
    rng = np.random.default_rng(4)
    for R in (1, 2, 3, 5):
        S = rng.random((R, R))
        pi = O.best_assignment(S)
        best = max(permutations(range(R)), key=lambda p: sum(S[f, p[f]] for f in range(R)))
        assert tuple(pi) == best
    assert list(O.best_assignment(np.ones((3, 3)))) == [0, 1, 2]    # ties: lexicographic
    # Hungarian path (R > 8) vs brute force score on a planted permutation
    S = rng.random((10, 10)) * 0.1
    perm = rng.permutation(10)
    S[np.arange(10), perm] += 1.0
    assert np.array_equal(O.best_assignment(S), perm)


def _model(I, J, K, R, seed):
    rng = np.random.default_rng(seed)
    return rng.random(R) + 0.5, rng.random((I, R)), rng.random((J, R)), rng.random((K, R))


def test_match_identity():
    """S:268 / Lemma 1 equality case: candidate == anchors -> identity, scores 1."""
    lam, A, B, C = _model(20, 18, 16, 3, 5)
    Is, Js, Ks = np.arange(0, 20, 2), np.arange(0, 18, 3), np.arange(0, 16, 4)
    Up = [A[Is], B[Js], np.vstack([C[Ks], np.ones((2, 3))])]
    rm = O.match_rep(A, B, C, Is, Js, Ks, lam, Up, 0.9)
    assert list(rm.pi) == [0, 1, 2] and rm.accepted
    assert np.allclose(rm.score, 1.0, atol=1e-12)
    for m in range(3):
        assert np.allclose(rm.scale[m], 1.0)
    assert np.allclose(rm.lam_hat, lam)


def test_match_known_permutation_signs_scales():
    """permuted, sign-flipped, rescaled candidate -> exact pi; rescaled rows
    equal the old rows and lambda_hat reproduces the same tensor."""
    lam, A, B, C = _model(30, 25, 20, 4, 6)
    Is, Js, Ks = np.arange(0, 30, 3), np.arange(0, 25, 2), np.arange(0, 20, 5)
    perm = np.array([2, 0, 3, 1])          # candidate column perm[f] holds old component f
    sA = np.array([1.0, -1.0, 1.0, -1.0]); sB = np.array([-1.0, -1.0, 1.0, 1.0])
    nA = np.linalg.norm(A[Is], axis=0); nB = np.linalg.norm(B[Js], axis=0)
    Cp_old = C[Ks]; Cnew = np.random.default_rng(7).random((3, 4))
    nC = np.linalg.norm(Cp_old, axis=0)
    Ap = np.zeros((len(Is), 4)); Bp = np.zeros((len(Js), 4)); Cp = np.zeros((len(Ks) + 3, 4)); lp = np.zeros(4)
    for f in range(4):
        g = perm[f]
        Ap[:, g] = sA[f] * A[Is, f] / nA[f]
        Bp[:, g] = sB[f] * B[Js, f] / nB[f]
        Cp[:, g] = sA[f] * sB[f] * np.concatenate([Cp_old[:, f], Cnew[:, f]]) / nC[f] * 2.0
        lp[g] = lam[f] * nA[f] * nB[f] * nC[f] / 2.0
    rm = O.match_rep(A, B, C, Is, Js, Ks, lp, [Ap, Bp, Cp], 0.9)
    assert np.array_equal(rm.pi, perm) and rm.accepted
    assert np.allclose(O.rescaled([Ap, Bp, Cp], rm, 0), A[Is])
    assert np.allclose(O.rescaled([Ap, Bp, Cp], rm, 1), B[Js])
    Ct = O.rescaled([Ap, Bp, Cp], rm, 2)
    assert np.allclose(Ct[:len(Ks)], Cp_old) and np.allclose(Ct[len(Ks):], Cnew)
    assert np.allclose(rm.lam_hat, lam)


def test_match_noise_recovery_rate():
    """permuted anchors + N(0, 0.01^2) noise, R = 5, 40 anchor rows -> >= 95/100."""
    ok = 0
    for t in range(100):
        rng = np.random.default_rng(100 + t)
        R = 5
        A = rng.random((40, R)); B = rng.random((40, R)); C = rng.random((40, R))
        idx = np.arange(40)
        perm = rng.permutation(R)
        cand = []
        for F in (A, B, C):
            G = np.zeros_like(F)
            G[:, perm] = F + 0.01 * rng.standard_normal(F.shape)
            cand.append(G)
        rm = O.match_rep(A, B, C, idx, idx, idx, np.ones(R), cand, 0.0)
        ok += np.array_equal(rm.pi, perm)
    assert ok >= 95


def test_relative_error_expansion_vs_materialisation():
    """The expansion path (> 1e6 entries) equals direct materialisation; lambda = 0 -> 1."""
    rng = np.random.default_rng(8)
    K, J, I, R = 101, 100, 100, 3
    lam, A, B, C = rng.random(R), rng.random((I, R)), rng.random((J, R)), rng.random((K, R))
    T = (np.einsum("f,if,jf,kf->kji", lam, A, B, C) + 0.1 * rng.standard_normal((K, J, I))).astype(np.float32)
    model = np.einsum("f,if,jf,kf->kji", lam, A, B, C)
    direct = np.linalg.norm(T.astype(np.float64) - model) / np.linalg.norm(T.astype(np.float64))
    assert abs(O.relative_error(T, lam, A, B, C) - direct) < 1e-9
    assert O.relative_error(T, np.zeros(R), A, B, C) == pytest.approx(1.0, abs=1e-12)
    small = T[:10, :10, :10].copy()
    assert O.relative_error(small, np.zeros(R), A[:10], B[:10], C[:10]) == pytest.approx(1.0, abs=1e-14)


def test_fms_properties():
    lam, A, B, C = _model(10, 9, 8, 4, 9)
    m = (lam, A, B, C)
    assert O.fms(m, m) == pytest.approx(1.0, abs=1e-12)
    p = np.array([3, 1, 0, 2])
    mp = (lam[p], A[:, p] * 2.0, B[:, p], C[:, p] * 0.5)
    assert O.fms(m, mp) == pytest.approx(1.0, abs=1e-12)
    other = (lam[:1], np.eye(3)[:, :1], np.ones((2, 1)), np.ones((2, 1)))
    orth = (lam[:1], np.eye(3)[:, 1:2], np.ones((2, 1)), np.ones((2, 1)))
    assert O.fms(other, orth) == 0.0
    m2 = _model(10, 9, 8, 4, 10)
    assert O.fms(m, m2) == pytest.approx(O.fms(m2, m), abs=1e-12)


def test_recompute_is_cp_als_from_the_r35_point():
    """R35: the CP_ALS baseline starts from Philox repetition 255 of the current update id; on a
    noiseless planted tensor it converges to the planted model (fit > 0.999 at 500 iterations,
    R27) and the relative fitness of the planted truth against it is ~1 (both exact)."""
    from synth import planted_dense
    T, truth = planted_dense(30, 28, 26, 3, noise=0.0, seed=61)
    lam, U, fit, it = O.recompute(T, 3, seed=4, update_id=2, maxit=500, tol=1e-12)
    assert fit > 0.999
    U0 = O.als_init(O.view_ijk(T).shape, 3, 4, 2, 255)
    lam2, U2, fit2, it2, _ = O.cp_als(O.view_ijk(T), U0, 500, 1e-12)
    assert fit == fit2 and all(np.array_equal(a, b) for a, b in zip(U, U2))
    # a different repetition index starts elsewhere (the stream is keyed by rep)
    assert not np.array_equal(U0[0], O.als_init(O.view_ijk(T).shape, 3, 4, 2, 0)[0])


def test_relative_fitness_definition_pins():
    """RF(X, M, M) = 1; a model with twice the baseline's residual has RF = 2 (the
    residual of lam * M scales linearly when X = 0 outside the model's span: here X = M_b + E
    with E orthogonal to both models' span is built by an exact rank-1 construction)."""
    rng = np.random.default_rng(3)
    a, b, c = (rng.random(n) for n in (5, 4, 3))
    X = np.einsum("i,j,k->kji", a, b, c).astype(np.float32)
    m = (np.ones(1), a[:, None], b[:, None], c[:, None])
    assert O.relative_fitness(X, m, m) == 1.0
    # scaled models: residual |1 - s| * ||X|| -> RF = |1 - s1| / |1 - s2|
    m1 = (np.array([0.8]), a[:, None], b[:, None], c[:, None])
    m2 = (np.array([0.9]), a[:, None], b[:, None], c[:, None])
    assert abs(O.relative_fitness(X, m1, m2) - 2.0) < 1e-6
