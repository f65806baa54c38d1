"""Incremental marginals (opts.incremental_marginals): adding the batch's
contribution to the committed marginals is bit-identical to the full pass (integer sums), so
an incremental handle must produce the bit-identical model, samples and fits of a full-pass
handle over a stream of updates, across checkpoint / restore, for dense, COO and the sharded
(world-1) handle."""
import os
import subprocess
import sys

import numpy as np
import pytest

from synth import planted_dense, split_dense, zipf_planted_coo, split_coo
from tests._helpers import dev

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def L():
    from paper_1709_00668_b200 import _lib
    return _lib


def _state(h, r, K, I, J, R):
    A = np.empty((I, R), np.float32); B = np.empty((J, R), np.float32)
    C = np.empty((K, R), np.float32); lam = np.empty(R, np.float32)
    L().sambaten_copy_factors(h, A, B, C, lam)
    n = L().sambaten_last_samples(h)
    Is = np.empty(r * n[0], np.int32); Js = np.empty(r * n[1], np.int32); Ks = np.empty(r * n[2], np.int32)
    L().sambaten_last_samples(h, Is, Js, Ks)
    return [A, B, C, lam, Is, Js, Ks]


def _same(a, b):
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))


def test_dense_incremental_equals_full_pass():
    I, J, K, R, K0, bs, r = 60, 44, 50, 4, 30, 4, 4
    T, truth = planted_dense(I, J, K, R, noise=0.01, seed=8)
    T0, batches = split_dense(T, K0, bs)
    model = [np.ascontiguousarray(np.asarray(x, np.float32)) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    hs = []
    for inc in (0, 1):
        opts = L().default_opts(als_max_iters=8, als_tol=0.0, capacity=K, full_fit=1, accept_tau=0.0,
                                incremental_marginals=inc)
        hs.append(L().sambaten_init_factors(L().dense(dev(T0)), R, 2, r, 3, model[1], model[2], model[3],
                                            model[0], opts))
    try:
        for h in hs:
            L().sambaten_checkpoint(h)
        for rnd in range(2):   # the second round starts from restore: xm must come back too
            Kt = K0
            for b in batches:
                Kt += b.shape[0]
                fits = [L().sambaten_update(h, L().dense(dev(b))).fit_full for h in hs]
                assert fits[0] == fits[1]
                _same(_state(hs[0], r, Kt, I, J, R), _state(hs[1], r, Kt, I, J, R))
            for h in hs:
                L().sambaten_restore(h)
    finally:
        for h in hs:
            L().sambaten_destroy(h)


def test_coo_incremental_equals_full_pass():
    import torch
    I, J, K, R, K0, bs, r = 300, 260, 60, 4, 40, 5, 4
    X, truth = zipf_planted_coo(I, J, K, R, 30000, alpha=1.2, seed=4)
    X0, batches = split_coo(X, K0, bs)
    model = [np.ascontiguousarray(np.asarray(x, np.float32)) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]

    def coo(x):
        return L().coo(*[torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (x.i, x.j, x.k, x.v)], x.dims)
    hs = []
    for inc in (0, 1):
        opts = L().default_opts(als_max_iters=6, als_tol=0.0, capacity=X.nnz, full_fit=1, accept_tau=0.0,
                                incremental_marginals=inc)
        opts.capacity_k = K
        hs.append(L().sambaten_init_factors(coo(X0), R, 2, r, 5, model[1], model[2], model[3], model[0], opts))
    try:
        Kt = K0
        for b in batches:
            Kt += b.dims[2]
            fits = [L().sambaten_update(h, coo(b)).fit_full for h in hs]
            assert fits[0] == fits[1]
            _same(_state(hs[0], r, Kt, I, J, R), _state(hs[1], r, Kt, I, J, R))
    finally:
        for h in hs:
            L().sambaten_destroy(h)


SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
from paper_1709_00668_b200 import _lib as L
from synth import planted_dense, split_dense
I, J, K, R, K0, bs = 64, 48, 40, 4, 30, 5
T, truth = planted_dense(I, J, K, R, noise=0.01, seed=3)
T0, batches = split_dense(T, K0, bs)
model = [np.ascontiguousarray(np.asarray(x, np.float32)) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
hs = []
for inc in (0, 1):
    opts = L.default_opts(als_max_iters=10, als_tol=0.0, capacity=K, full_fit=1, incremental_marginals=inc)
    dist = L.make_dist(0, 1, L.sambaten_dist_unique_id(), 0, K0)
    hs.append(L.sambaten_init_factors_dist(L.dense(torch.from_numpy(T0).cuda()), dist, R, 2, 4, 9,
                                           model[1], model[2], model[3], model[0], opts))
Kt = K0
for b in batches:
    Kt += b.shape[0]
    out = []
    for h in hs:
        A = np.empty((I, R), np.float32); B = np.empty((J, R), np.float32)
        C = np.empty((Kt, R), np.float32); lam = np.empty(R, np.float32)
        info = L.sambaten_update(h, L.dense(torch.from_numpy(b).cuda()), A, B, C, lam)
        out.append((A, B, C, lam, info.fit_full))
    for x, y in zip(out[0][:4], out[1][:4]):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    assert out[0][4] == out[1][4]
for h in hs:
    L.sambaten_destroy(h)
print("INC_DIST_OK")
'''


def test_sharded_incremental_equals_full_pass():
    env = dict(os.environ)
    env["SAMBATEN_DIST_LOOPBACK"] = "1"
    r = subprocess.run([sys.executable, "-c", "ROOT = %r\n" % ROOT + SCRIPT], env=env, capture_output=True,
                       text=True, timeout=600)
    assert "INC_DIST_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
