"""Pins for the oracle's importance sampling without replacement (readings R4-R6)."""
from itertools import permutations

import numpy as np

from oracle import sambaten as O


def successive_inclusion(w, n_s):
    """Exact inclusion probabilities of successive sampling without replacement (each draw
    proportional to the weight among the remaining items), by enumerating ordered draws."""
    w = np.asarray(w, float)
    n = len(w)
    pi = np.zeros(n)
    for seq in permutations(range(n), n_s):
        p, rest = 1.0, w.sum()
        for a in seq:
            p *= w[a] / rest
            rest -= w[a]
        for a in seq:
            pi[a] += p
    return pi


def test_sample_size():
    assert O.sample_size(50, 2) == 25 and O.sample_size(450, 5) == 90 and O.sample_size(65536, 10) == 6554
    assert O.sample_size(3, 5) == 1 and O.sample_size(7, 1) == 7


def test_distinct_sorted_and_sized():
    w = np.random.default_rng(0).integers(0, 1000, 500)
    for rep in range(4):
        idx = O.sample_mode(w, 100, 0, 1, rep, 0)
        assert len(idx) == 100 and np.all(np.diff(idx) > 0)
        assert idx.min() >= 0 and idx.max() < 500


def test_s1_gives_full_set():
    """S:250."""
    w = np.arange(1, 40)
    assert np.array_equal(O.sample_mode(w, len(w), 3, 1, 0, 0), np.arange(len(w)))


def test_single_positive_weight_is_certain():
    """weights (0,0,7,0), sample size 1 -> index 2."""
    for uid in range(1, 50):
        assert list(O.sample_mode(np.array([0, 0, 7, 0]), 1, 11, uid, 0, 2)) == [2]


def test_zero_weights_fill_in_index_order():
    w = np.array([0, 5, 0, 0, 3, 0])
    assert list(O.sample_mode(w, 4, 0, 1, 0, 0)) == [0, 1, 2, 4]


def test_inclusion_probabilities_match_successive_sampling():
    """Exponential keys realise successive sampling: empirical inclusion frequencies over
    40,000 update ids agree with the exact enumeration for w = (1,2,3,4,0.5)*2, n_s = 2
    (SURVEY §8(c) pins: (0.21911, 0.41346, 0.57313, 0.68212, 0.11219))."""
    w = np.array([2, 4, 6, 8, 1], np.int64)
    exact = successive_inclusion(w, 2)
    assert np.allclose(exact, [0.21911, 0.41346, 0.57313, 0.68212, 0.11219], atol=1e-5)
    N = 40_000
    cnt = np.zeros(5)
    for uid in range(1, N + 1):
        cnt[O.sample_mode(w, 2, 1234, uid, 0, 1)] += 1
    freq = cnt / N
    sigma = np.sqrt(exact * (1 - exact) / N)
    assert np.all(np.abs(freq - exact) <= 4.5 * sigma), (freq, exact)


def test_single_draw_frequencies():
    """one index from weights (1,2,3,4) lands within 3 sigma of (.1,.2,.3,.4)."""
    w = np.array([1, 2, 3, 4])
    N = 10_000
    cnt = np.zeros(4)
    for uid in range(1, N + 1):
        cnt[O.sample_mode(w, 1, 99, uid, 3, 0)] += 1
    p = np.array([0.1, 0.2, 0.3, 0.4])
    assert np.all(np.abs(cnt / N - p) <= 3 * np.sqrt(p * (1 - p) / N) + 1e-12)


def test_deterministic_and_stream_separated():
    w = np.random.default_rng(1).integers(1, 100, 300)
    a = O.sample_mode(w, 30, 7, 2, 1, 0)
    assert np.array_equal(a, O.sample_mode(w, 30, 7, 2, 1, 0))
    assert not np.array_equal(a, O.sample_mode(w, 30, 7, 2, 2, 0))
    assert not np.array_equal(a, O.sample_mode(w, 30, 7, 3, 1, 0))
    assert not np.array_equal(a, O.sample_mode(w, 30, 8, 2, 1, 0))
