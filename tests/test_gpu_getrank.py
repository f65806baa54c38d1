"""GetRank (Alg. 2) on the GPU against the oracle
(oracle/getrank.py; readings R29-R31).

* CorConDia of given models: |cc_gpu - cc_oracle| <= 1e-6 max(1, |cc|) (both fp64; the GPU
  forms pinv from the normal equations, the oracle by SVD -- equal for full column rank).
* GetRank on planted tensors: the same R_new as the oracle; for candidate ranks up to the
  planted one (well-posed, converged models) the ratings agree within 0.05 (fp32 vs fp64 ALS
  trajectories from the same Philox start, R30); above it both stay under the threshold.
"""
import numpy as np
import pytest

from oracle import getrank as GR
from tests._helpers import dev

pytestmark = pytest.mark.gpu


def L():
    from paper_1709_00668_b200 import _lib
    return _lib


def _dense(Y_ijk):
    """oracle X[i, j, k] -> device (K, J, I) layout."""
    import torch
    return L().dense(torch.from_numpy(np.ascontiguousarray(np.transpose(Y_ijk, (2, 1, 0)).astype(np.float32))).cuda())


@pytest.mark.parametrize("F,seed", [(1, 0), (3, 1), (6, 2)])
def test_corcondia_matches_oracle(F, seed):
    rng = np.random.default_rng(seed)
    I, J, K = 30, 26, 22
    A, B, C = rng.random((I, F)), rng.random((J, F)), rng.random((K, F))
    Y = np.einsum("if,jf,kf->ijk", A, B, C) + 0.05 * rng.standard_normal((I, J, K))
    Y32 = Y.astype(np.float32).astype(np.float64)
    lam = rng.random(F) + 0.5
    A32, B32, C32 = (x.astype(np.float32) for x in (A, B, C))
    got = L().sambaten_corcondia(_dense(Y32), F, dev(A32), dev(B32), dev(C32), dev(lam))
    want = GR.corcondia(Y32, lam, A32.astype(np.float64), B32.astype(np.float64), C32.astype(np.float64))
    assert abs(got - want) <= 1e-6 * max(1.0, abs(want)), (got, want)
    # the exact model of its own tensor rates 100
    Ye = np.einsum("if,jf,kf,f->ijk", A32.astype(np.float64), B32.astype(np.float64), C32.astype(np.float64), lam)
    got_e = L().sambaten_corcondia(_dense(Ye), F, dev(A32), dev(B32), dev(C32), dev(lam))
    assert abs(got_e - 100.0) < 1e-2   # the tensor itself is rounded to fp32


@pytest.mark.parametrize("F,seed", [(2, 0), (3, 1)])
def test_getrank_matches_oracle(F, seed):
    rng = np.random.default_rng(seed)
    A, B, C = rng.random((12, F)), rng.random((11, F)), rng.random((10, F))
    Y = np.einsum("if,jf,kf->ijk", A, B, C).astype(np.float32).astype(np.float64)
    rn_o, cc_o = GR.getrank(Y, 4, 2, 7, 300, 0.0)
    rn_g, cc_g = L().sambaten_getrank(_dense(Y), 4, 2, 7, 300, 0.0)
    assert rn_g == rn_o == F, (cc_g, cc_o)
    assert np.all(np.abs(cc_g[:F] - cc_o[:F]) <= 0.05), (cc_g, cc_o)
    assert cc_g[F:].max() < 90.0 and cc_o[F:].max() < 90.0


def test_getrank_on_a_noisy_planted_summary():
    """A 1 %-noise planted rank-5 tensor of summary size: both sides pick 5."""
    rng = np.random.default_rng(4)
    F = 5
    A, B, C = rng.random((40, F)), rng.random((36, F)), rng.random((32, F))
    Y = np.einsum("if,jf,kf->ijk", A, B, C)
    Y = Y + 0.01 * np.linalg.norm(Y) / np.sqrt(Y.size) * rng.standard_normal(Y.shape)
    Y = Y.astype(np.float32).astype(np.float64)
    rn_o, cc_o = GR.getrank(Y, 7, 1, 3, 100, 0.0)
    rn_g, cc_g = L().sambaten_getrank(_dense(Y), 7, 1, 3, 100, 0.0)
    assert rn_g == rn_o == F, (cc_g.ravel(), cc_o.ravel())
