"""Counter-based random numbers for the oracle (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

The paper does not say how its MATLAB code draws random numbers (P:188, P:211
only say "sample ... without replacement").  DESIGN.md reading R6 fixes a
counter-based generator so that the CUDA path and this oracle draw the very
same numbers: Philox4x32-10 (Salmon et al., SC'11), a uniform built from 52
random bits, and a logarithm made only of correctly rounded IEEE operations
(reading R7), so that the exponential keys E = -ln(u) are bit-identical on
both sides.

Everything here is written out from those definitions in numpy uint64 /
float64 arithmetic.  numpy never fuses a*b+c into an FMA, so each line is one
correctly rounded IEEE operation.
"""
import numpy as np

_MASK32 = np.uint64(0xFFFFFFFF)
# Philox4x32 round multipliers and Weyl key increments (Salmon et al. 2011, Table 2).
_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = 0x9E3779B9
_W1 = 0xBB67AE85

# Counter domains (reading R6): word 3 of the counter is  domain<<24 | rep<<8 | mode.
DOMAIN_SAMPLE = 1
DOMAIN_ALS_INIT = 2
DOMAIN_GEN = 3


def philox4x32_10(c0, c1, c2, c3, key):
    """Philox4x32 with 10 rounds.

    c0..c3: arrays (or scalars) of counter words < 2**32; key: 64-bit integer,
    split as (k0, k1) = (low 32 bits, high 32 bits).  Returns four uint64
    arrays holding 32-bit outputs.

    One round maps (c0,c1,c2,c3) with key (k0,k1) to
        (hi(M1*c2) ^ c1 ^ k0,  lo(M1*c2),  hi(M0*c0) ^ c3 ^ k1,  lo(M0*c0))
    and the key is bumped by (W0, W1) between rounds.
    """
    c0 = np.asarray(c0, dtype=np.uint64) & _MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & _MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & _MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & _MASK32
    k0 = int(key) & 0xFFFFFFFF
    k1 = (int(key) >> 32) & 0xFFFFFFFF
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + _W0) & 0xFFFFFFFF
            k1 = (k1 + _W1) & 0xFFFFFFFF
        p0 = _M0 * c0          # exact: 32x32 -> 64 bit product
        p1 = _M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1,
                          hi0 ^ c3 ^ np.uint64(k1), lo0)
    return c0, c1, c2, c3


def uniform53(x0, x1):
    """u = (2*m52 + 1) * 2**-53 with m52 = (x0 << 20) | (x1 >> 12).

    m52 < 2**52, so the numerator is an odd integer < 2**53 and u is exact,
    strictly inside (0, 1).  Only x0 and x1 are used (reading R6).
    """
    m52 = (np.asarray(x0, dtype=np.uint64) << np.uint64(20)) | (np.asarray(x1, dtype=np.uint64) >> np.uint64(12))
    return (m52.astype(np.float64) * 2.0 + 1.0) * 2.0 ** -53


# detlog constants (reading R7).  LN2_HI has its low 32 mantissa bits zero, so e*LN2_HI
# is exact for |e| < 2**21.
LN2_HI = float.fromhex("0x1.62e42p-1")
LN2_LO = float.fromhex("0x1.fdf473dep-22")
SQRT_HALF = float.fromhex("0x1.6a09e667f3bcdp-1")
# 2/(2n+1), n = 0..10: the series ln(m) = 2 atanh(s) = s * sum_n (2/(2n+1)) s^(2n).
LOG_COEF = [float.fromhex(h) for h in (
    "0x1p+1", "0x1.5555555555555p-1", "0x1.999999999999ap-2", "0x1.2492492492492p-2",
    "0x1.c71c71c71c71cp-3", "0x1.745d1745d1746p-3", "0x1.3b13b13b13b14p-3",
    "0x1.1111111111111p-3", "0x1.e1e1e1e1e1e1ep-4", "0x1.af286bca1af28p-4",
    "0x1.8618618618618p-4")]


def detlog(u):
    """Deterministic natural log for u in (0, 1) (reading R7).

    u = m * 2**e with m in [1/2, 1) (frexp, exact); if m < sqrt(1/2): m <- 2m,
    e <- e-1, so m in [sqrt(1/2), sqrt(2)).  With f = m-1, s = f/(2+f), z = s*s:
        ln m = s * (c0 + z*(c1 + z*(c2 + ... + z*c10)))      (Horner, no FMA)
        ln u = e*LN2_HI + (e*LN2_LO + ln m)
    """
    u = np.asarray(u, dtype=np.float64)
    m, e = np.frexp(u)
    small = m < SQRT_HALF
    m = np.where(small, m * 2.0, m)
    e = np.where(small, e - 1, e).astype(np.float64)
    f = m - 1.0
    s = f / (2.0 + f)
    z = s * s
    p = np.full_like(s, LOG_COEF[10])
    for n in range(9, -1, -1):
        p = LOG_COEF[n] + z * p
    P = s * p
    return e * LN2_HI + (e * LN2_LO + P)
