"""The incremental exact fit (opts.full_fit = 1 on dense handles, k_fitinc.cu; SURVEY 8(f)
NEXT #1): each update's relative error is formed from the previous model's
per-component inner products, the batch's slices and the rows the merge changed
(telescoping identity), or one full per-component pass when the device plan says so.
Checks through the C-ABI:
* fit_full equals the oracle's relative error of the GPU model over the whole tensor
  (<= 1e-6) on every update, for the plain path (a dense model: only new slices), for
  zeroed B / C rows (the changed-row terms), for zeroed A rows (the full-pass fallback), and
  for the overwrite merge;
* the committed models are bit-identical to a handle using the separate full pass
  (SAMBATEN_FULL_FIT_PASS), so the fit path never touches the method's arithmetic;
* checkpoint / restore carries the state (a replay gives the same fits bit for bit)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import sambaten as O
from synth import planted_dense, split_dense
from tests._helpers import dev

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def L():
    from paper_1709_00668_b200 import _lib
    return _lib


def _model(h, I, J, K, R):
    A = np.empty((I, R), np.float32); B = np.empty((J, R), np.float32)
    C = np.empty((K, R), np.float32); lam = np.empty(R, np.float32)
    L().sambaten_copy_factors(h, A, B, C, lam)
    return lam, A, B, C


def _stream(zero_rows=None, policy=0, inc=0, I=96, J=80, K0=40, bs=5, nb=3, R=4, seed=51):
    T, truth = planted_dense(I, J, K0 + bs * nb, R, noise=0.01, seed=seed)
    T0, batches = split_dense(T, K0, bs)
    model = [np.ascontiguousarray(np.asarray(x, np.float32)) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    if zero_rows:
        for m, rows in zero_rows.items():
            model[m][rows] = 0.0
    opts = L().default_opts(als_max_iters=12, als_tol=0.0, accept_tau=0.0, capacity=K0 + bs * nb, full_fit=1,
                            merge_policy=policy, incremental_marginals=inc)
    h = L().sambaten_init_factors(L().dense(dev(T0)), R, 2, 4, 7, model[1], model[2], model[3], model[0], opts)
    return h, T0, batches, (I, J, R)


@pytest.mark.parametrize("case", ["dense", "zero_B_C", "zero_A", "overwrite", "incremental_marginals"])
def test_incremental_fit_matches_oracle(case):
    kw = {"dense": {}, "zero_B_C": {"zero_rows": {2: [1, 7, 30], 3: [0, 5, 33]}},
          "zero_A": {"zero_rows": {1: [4, 50]}}, "overwrite": {"policy": 1},
          "incremental_marginals": {"inc": 1}}[case]
    h, X, batches, (I, J, R) = _stream(**kw)
    paths = []
    try:
        for b in batches:
            info = L().sambaten_update(h, L().dense(dev(b)))
            X = np.concatenate([X, b])
            m = tuple(np.asarray(v, np.float64) for v in _model(h, I, J, X.shape[0], R))
            rel_o = O.relative_error(X, *m)
            assert abs((1.0 - info.fit_full) - rel_o) <= 1e-6, (case, info.fit_full, 1 - rel_o, info.fit_path)
            paths.append(info.fit_path)
    finally:
        L().sambaten_destroy(h)
    if case in ("dense", "incremental_marginals", "zero_B_C"):
        assert all(p == 3 for p in paths), paths      # incremental (the dB / dC terms included)
    if case == "zero_A":
        assert paths[0] == 4, paths                     # a changed A row: the full pass


def _coo_stream(zero_A=None, R=4, seed=53):
    from synth import zipf_planted_coo, split_coo
    X, truth = zipf_planted_coo(300, 260, 60, R, 40_000, alpha=1.2, seed=seed)
    K0, bs = 45, 5
    X0, batches = split_coo(X, K0, bs)
    lam, A, B, C = (np.ascontiguousarray(np.asarray(x, np.float32)) for x in truth)
    C = np.ascontiguousarray(C[:K0])
    if zero_A:
        A[zero_A] = 0.0
        B[list(range(1, 260, 11))] = 0.0
        C[[3, 17, 30]] = 0.0
    opts = L().default_opts(als_max_iters=12, als_tol=0.0, accept_tau=0.0, capacity=X.nnz,
                            capacity_k=X.dims[2], full_fit=1)
    gc = lambda Y: L().coo(dev(Y.i.astype(np.int32)), dev(Y.j.astype(np.int32)), dev(Y.k.astype(np.int32)),
                           dev(Y.v), Y.dims)
    h = L().sambaten_init_factors(gc(X0), R, 2, 4, 9, A, B, C, lam, opts)
    oc = lambda Y: O.Coo(Y.i.astype(np.int64), Y.j.astype(np.int64), Y.k.astype(np.int64), Y.v, Y.dims)
    return h, X0, batches, gc, oc


@pytest.mark.parametrize("case", ["coo", "coo_zero_rows"])
def test_incremental_fit_coo_matches_oracle(case):
    """COO stores: the batch's entries with the new model plus, when the merge refilled zeroed
    rows of A, B or old C, the old entries of those rows with the difference of the two
    models (fit_path 3); fit_full vs the oracle's relative error of the GPU model over the whole
    tensor <= 1e-6."""
    from synth import CooArrays

    def concat_coo(X, b):   # b's slices re-based to k = 0 follow X's
        return CooArrays(np.concatenate([X.i, b.i]), np.concatenate([X.j, b.j]),
                         np.concatenate([X.k, (b.k + X.dims[2]).astype(np.int32)]), np.concatenate([X.v, b.v]),
                         (X.dims[0], X.dims[1], X.dims[2] + b.dims[2]))
    zero = list(range(0, 300, 7)) if case == "coo_zero_rows" else None
    h, X, batches, gc, oc = _coo_stream(zero_A=zero)
    I, J, R = X.dims[0], X.dims[1], 4
    paths = []
    try:
        for b in batches[:3]:
            info = L().sambaten_update(h, gc(b))
            X = concat_coo(X, b)
            m = tuple(np.asarray(v, np.float64) for v in _model(h, I, J, X.dims[2], R))
            rel_o = O.relative_error(oc(X), *m)
            assert abs((1.0 - info.fit_full) - rel_o) <= 1e-6, (case, info.fit_full, 1 - rel_o, info.fit_path)
            paths.append(info.fit_path)
    finally:
        L().sambaten_destroy(h)
    assert all(p == 3 for p in paths), paths


SCRIPT = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, ROOT)
from paper_1709_00668_b200 import _lib as L
from synth import planted_dense, split_dense
I, J, K0, bs, R = 96, 80, 40, 5, 4
T, truth = planted_dense(I, J, K0 + 3 * bs, R, noise=0.01, seed=52)
T0, batches = split_dense(T, K0, bs)
model = [np.ascontiguousarray(np.asarray(x, np.float32)) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
model[2][[3, 9]] = 0.0
opts = L.default_opts(als_max_iters=10, als_tol=0.0, accept_tau=0.0, capacity=K0 + 3 * bs, full_fit=1)
h = L.sambaten_init_factors(L.dense(torch.from_numpy(T0).cuda()), R, 2, 4, 5, model[1], model[2], model[3], model[0], opts)
L.sambaten_checkpoint(h)
out = []
for rep in range(2):
    for b in batches:
        info = L.sambaten_update(h, L.dense(torch.from_numpy(b).cuda()))
        A = np.empty((I, R), np.float32); L.sambaten_copy_factors(h, A)
        out.append((info.fit_full, info.fit_path, A.tobytes()))
    L.sambaten_restore(h)
n = len(batches)
assert out[:n] == out[n:], "replay after restore differs"
np.save(OUT, np.array([(o[0], o[1]) for o in out[:n]]))
import hashlib
open(OUT + ".models", "w").write(hashlib.sha256(b"".join(o[2] for o in out[:n])).hexdigest())
L.sambaten_destroy(h)
print("FITINC_OK")
'''


def test_fit_path_does_not_touch_the_model_and_survives_restore(tmp_path):
    """The same stream with the incremental fit and with the separate full pass
    (SAMBATEN_FULL_FIT_PASS=1): identical models bit for bit, fits within 1e-7; a replay after
    sambaten_restore reproduces the incremental fits exactly (the state is checkpointed)."""
    res = {}
    for mode in ("inc", "pass"):
        env = dict(os.environ)
        env.pop("SAMBATEN_FULL_FIT_PASS", None)
        if mode == "pass":
            env["SAMBATEN_FULL_FIT_PASS"] = "1"
        out = str(tmp_path / f"{mode}.npy")
        r = subprocess.run([sys.executable, "-c", f"ROOT = {ROOT!r}\nOUT = {out!r}\n" + SCRIPT], env=env,
                           capture_output=True, text=True, timeout=600)
        assert "FITINC_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
        res[mode] = (np.load(out), open(out + ".models").read())
    assert res["inc"][1] == res["pass"][1]
    assert np.all(res["inc"][0][:, 1] == 3) and np.all(res["pass"][0][:, 1] == 1)
    # two summation orders of the same quantity (the oracle bar is 1e-6)
    assert np.allclose(res["inc"][0][:, 0], res["pass"][0][:, 0], rtol=0, atol=1e-7)
