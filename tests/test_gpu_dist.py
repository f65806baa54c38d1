"""The sharded update (sambaten_init_factors_dist, NCCL) on one GPU: a world-1 handle, with the
exchange either short-circuited or forced through pack / ncclSend-to-self / ncclRecv /
unpack (SAMBATEN_DIST_LOOPBACK), must produce the bit-identical model of the single-GPU
handle on the same inputs (integer marginals, identical summaries, identical ALS)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
from paper_1709_00668_b200 import _lib as L
from synth import planted_dense, split_dense
I, J, K, R, K0, bs = 64, 48, 40, 4, 30, 5
T, truth = planted_dense(I, J, K, R, noise=0.01, seed=3)
T0, batches = split_dense(T, K0, bs)
model = [np.ascontiguousarray(np.asarray(x, np.float32)) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
import os
opts = L.default_opts(als_max_iters=15, als_tol=0.0, capacity=K, full_fit=int(os.environ.get("SBT_T_FF", "1")),
                      warm_start=int(os.environ.get("SBT_T_WARM", "0")), getrank=int(os.environ.get("SBT_T_GR", "0")))
dist = L.make_dist(0, 1, L.sambaten_dist_unique_id(), 0, K0)
if os.environ.get("SBT_T_BORROW") == "1":
    # opts.borrow_store on the sharded handle: the slab in place in a caller buffer of Kcap_local =
    # K0 + ceil((capacity - K0) / world) + 1 slices whose unused slices hold NaN (never read)
    od = L.default_opts(als_max_iters=15, als_tol=0.0, capacity=K, full_fit=int(os.environ.get("SBT_T_FF", "1")),
                        warm_start=int(os.environ.get("SBT_T_WARM", "0")), getrank=int(os.environ.get("SBT_T_GR", "0")),
                        borrow_store=1)
    xbuf = torch.full((K0 + (K - K0) + 1, J, I), float("nan"), device="cuda")
    xbuf[:K0] = torch.from_numpy(T0).cuda()
    hd = L.sambaten_init_factors_dist(L.dense(xbuf[:K0]), dist, R, 2, 4, 9, model[1], model[2], model[3],
                                      model[0], od)
else:
    hd = L.sambaten_init_factors_dist(L.dense(torch.from_numpy(T0).cuda()), dist, R, 2, 4, 9,
                                      model[1], model[2], model[3], model[0], opts)
hs = L.sambaten_init_factors(L.dense(torch.from_numpy(T0).cuda()), R, 2, 4, 9,
                             model[1], model[2], model[3], model[0], opts)
Kt = K0
for b in batches:
    Kt += b.shape[0]
    assert L.sambaten_batch_partition(hd, b.shape[0]) == (0, b.shape[0])
    out = []
    for h in (hd, hs):
        A = np.empty((I, R), np.float32); B = np.empty((J, R), np.float32)
        C = np.empty((Kt, R), np.float32); lam = np.empty(R, np.float32)
        info = L.sambaten_update(h, L.dense(torch.from_numpy(b).cuda()), A, B, C, lam)
        out.append((A, B, C, lam, info.fit_full, info.reps_rejected_mask, info.fit_full_prev, list(info.rep_rank[:4])))
    for x, y in zip(out[0][:4], out[1][:4]):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    assert out[0][7] == out[1][7], (out[0][7], out[1][7])   # GetRank's per-rep ranks (R33)
    # the single-GPU handle keeps its full fit incrementally (k_fitinc.cu), the sharded one by a
    # pass over the slabs: the same quantity in two summation orders
    assert abs(out[0][4] - out[1][4]) <= 1e-6 and out[0][5] == out[1][5] and out[0][6] == out[1][6], (out[0][4:7], out[1][4:7])
    if opts.full_fit == 2:
        assert out[0][4] == -1.0 and 0.9 < out[0][6] <= 1.0
L.sambaten_destroy(hd); L.sambaten_destroy(hs)
print("DIST_OK")
'''


@pytest.mark.parametrize("loopback,ff,warm,gr,borrow", [(False, 1, 0, 0, 0), (True, 1, 0, 0, 0), (False, 2, 0, 0, 0),
                                                         (True, 2, 1, 0, 0), (True, 1, 0, 1, 0), (False, 1, 1, 0, 1),
                                                         (True, 2, 0, 0, 1)])
def test_world1_dist_handle_matches_single_gpu_bitwise(loopback, ff, warm, gr, borrow):
    """full_fit = 2 (lag-1 fit in the a1 pass), the warm start (R34) and
    opts.borrow_store (the slab used in place) on the sharded handle: bit-identical to the
    single-GPU handle with the same options."""
    env = dict(os.environ)
    env["SBT_T_BORROW"] = str(borrow)
    env.pop("SAMBATEN_DIST_LOOPBACK", None)
    if loopback:
        env["SAMBATEN_DIST_LOOPBACK"] = "1"
    env["SBT_T_FF"] = str(ff)
    env["SBT_T_WARM"] = str(warm)
    env["SBT_T_GR"] = str(gr)   # GetRank in the sharded update (R33): ranks shared by an allgather
    r = subprocess.run([sys.executable, "-c", "ROOT = %r\n" % ROOT + SCRIPT], env=env, capture_output=True,
                       text=True, timeout=600)
    assert "DIST_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


SCRIPT_COO = r"""
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
from paper_1709_00668_b200 import _lib as L
from synth import zipf_planted_coo, split_coo
I, J, K, R, K0, bs = 400, 300, 60, 4, 40, 5
X, truth = zipf_planted_coo(I, J, K, R, 40000, alpha=1.2, seed=6)
X0, batches = split_coo(X, K0, bs)
model = [np.ascontiguousarray(np.asarray(x, np.float32)) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
def coo(x):
    return L.coo(*[torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (x.i, x.j, x.k, x.v)], x.dims)
opts = L.default_opts(als_max_iters=8, als_tol=0.0, capacity=X.nnz, full_fit=1, accept_tau=0.0,
                      incremental_marginals=INC, getrank=GR)
opts.capacity_k = K
dist = L.make_dist(0, 1, L.sambaten_dist_unique_id(), 0, K0)
hd = L.sambaten_init_factors_dist(coo(X0), dist, R, 2, 4, 9, model[1], model[2], model[3], model[0], opts)
hs = L.sambaten_init_factors(coo(X0), R, 2, 4, 9, model[1], model[2], model[3], model[0], opts)
for h in (hd, hs):
    L.sambaten_checkpoint(h)
for rnd in range(2):
    Kt = K0
    for b in batches:
        Kt += b.dims[2]
        assert L.sambaten_batch_partition(hd, b.dims[2]) == (0, b.dims[2])
        out = []
        for h in (hd, hs):
            A = np.empty((I, R), np.float32); B = np.empty((J, R), np.float32)
            C = np.empty((Kt, R), np.float32); lam = np.empty(R, np.float32)
            info = L.sambaten_update(h, coo(b), A, B, C, lam)
            out.append((A, B, C, lam, info.fit_full, info.reps_rejected_mask, list(info.rep_rank[:4])))
        for x, y in zip(out[0][:4], out[1][:4]):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
        assert out[0][6] == out[1][6]
        # the single-GPU handle keeps its fit incrementally (k_fitinc.cu), the sharded one by a pass
        assert abs(out[0][4] - out[1][4]) <= 1e-6 and out[0][5] == out[1][5]
    for h in (hd, hs):
        L.sambaten_restore(h)
L.sambaten_destroy(hd); L.sambaten_destroy(hs)
print("DIST_COO_OK")
"""


@pytest.mark.parametrize("loopback,inc,gr", [(False, 0, 0), (True, 0, 0), (True, 1, 0), (True, 0, 1)])
def test_world1_coo_dist_handle_matches_single_gpu_bitwise(loopback, inc, gr):
    env = dict(os.environ)
    env.pop("SAMBATEN_DIST_LOOPBACK", None)
    if loopback:
        env["SAMBATEN_DIST_LOOPBACK"] = "1"
    code = "ROOT = %r\nINC = %d\nGR = %d\n" % (ROOT, inc, gr) + SCRIPT_COO
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert "DIST_COO_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
