"""Pins for the oracle's Philox4x32-10, uniform and detlog (readings R6, R7)."""
import math
import os

import numpy as np

from oracle.philox import philox4x32_10, uniform53, detlog, LOG_COEF, LN2_HI, LN2_LO

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def _kat():
    rows = []
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        rows.append(w)
    return rows


def test_philox_known_answers():
    """Random123's published known-answer vectors (tests/golden/philox4x32_10_kat.txt)."""
    rows = _kat()
    assert len(rows) == 3
    for c0, c1, c2, c3, k0, k1, *out in rows:
        got = philox4x32_10(c0, c1, c2, c3, (k1 << 32) | k0)
        assert [int(g) for g in got] == out


def test_philox_vectorised_equals_scalar():
    c = np.arange(17, dtype=np.uint64)
    vec = philox4x32_10(c, 5, 7, 9, 0x123456789ABCDEF)
    for n in range(17):
        sc = philox4x32_10(n, 5, 7, 9, 0x123456789ABCDEF)
        assert [int(v[n]) for v in vec] == [int(s) for s in sc]


def test_uniform53_exact_and_open_interval():
    assert uniform53(0, 0) == 2.0 ** -53
    assert uniform53(0xFFFFFFFF, 0xFFFFFFFF) == 1.0 - 2.0 ** -53
    # mid point: m52 = 2**51 -> (2**52 + 1) * 2**-53
    assert uniform53(0x80000000, 0) == (2.0 ** 52 + 1.0) * 2.0 ** -53


def test_detlog_constants():
    for n, c in enumerate(LOG_COEF):
        assert c == 2.0 / (2 * n + 1)
    assert abs((LN2_HI + LN2_LO) - math.log(2.0)) <= math.ulp(math.log(2.0))
    # LN2_HI has its low 32 mantissa bits zero so that e * LN2_HI is exact
    m = int(LN2_HI.hex().split(".")[1].split("p")[0].ljust(13, "0"), 16)
    assert m & 0xFFFFFFFF == 0


def test_detlog_close_to_log_and_exact_points():
    rng = np.random.default_rng(1)
    u = rng.random(1_000_000)
    u = u[u > 0]
    a = detlog(u)
    b = np.log(u)
    ulp = np.abs(a - b) / np.spacing(np.abs(b))
    assert ulp.max() <= 4
    for x in (0.5, 0.25, 2.0 ** -53, 2.0 ** -30):
        assert detlog(np.array([x]))[0] == math.log(x)
    v = detlog(np.array([1.0 - 2.0 ** -53]))[0]
    assert abs(v - math.log1p(-(2.0 ** -53))) <= math.ulp(v) * 4


def test_detlog_monotone():
    u = np.sort(np.random.default_rng(2).random(200_000))
    u = u[u > 0]
    d = detlog(u)
    assert np.all(np.diff(d) >= 0)


def test_synth_philox_twin_matches_oracle_philox():
    """The generator's own numpy Philox (synth, input tooling) agrees with the oracle's."""
    import numpy as np
    from synth.planted import _philox_np
    rng = np.random.default_rng(4)
    for _ in range(20):
        seed = int(rng.integers(0, 2**63))
        c = [int(x) for x in rng.integers(0, 2**32, 4)]
        got = [int(v) for v in _philox_np(seed, *c)]
        assert tuple(got) == tuple(int(v) for v in philox4x32_10(*c, seed))
