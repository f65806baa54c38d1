"""Multi-process (gloo, CPU) tests of the sharded update's host logic and decomposition.

1. The exchange plan (sambaten_dist_plan, host-only C-ABI call): what every rank plans to send
   to every owner equals what that owner plans to receive, and every summary slice of every
   repetition is delivered exactly once (world 2 and 3).
2. The decomposition itself, run with the oracle's building blocks: slab-local fixed-point
   marginals summed by an all-reduce equal the full-tensor marginals bit for bit; the
   per-rank summary slices assembled on the repetition owners equal the full gather; owned
   repetitions' ALS + all-gather + replicated merge equal the single-process oracle update.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sambaten as O
from synth import planted_dense, split_dense


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, fn, *args):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def partition(Kn, world, rank):
    base, rem = divmod(Kn, world)
    return rank * base + min(rank, rem), base + (1 if rank < rem else 0)


# --------------------------------------------------------------------------- 1. the plan
def _plan_worker(rank, world, seed):
    from paper_1709_00668_b200 import _lib as L
    rng = np.random.default_rng(seed)
    Ko, Kn, r, nKs = 53, 7, 6, 11
    owner = rng.integers(0, world, Ko).astype(np.int32)       # arbitrary ownership of old slices
    Kp = np.stack([np.concatenate([np.sort(rng.choice(Ko, nKs, replace=False)), np.arange(Ko, Ko + Kn)])
                   for _ in range(r)]).astype(np.int32)
    send, recv = L.sambaten_dist_plan(Kp, owner, Ko, Kn, world, rank)
    mats = [None] * world
    dist.all_gather_object(mats, (send.tolist(), recv.tolist()))
    S = np.array([m[0] for m in mats])   # S[g][o]: g sends to o
    Rv = np.array([m[1] for m in mats])  # Rv[o][g]: o receives from g
    assert np.array_equal(S, Rv.T)
    # every (rho, u) is delivered exactly once: local (own) + received = r_owned * nKp
    def own_of(k):
        if k < Ko:
            return owner[k]
        for g in range(world):
            b, n = partition(Kn, world, g)
            if b <= k - Ko < b + n:
                return g
    for o in range(world):
        owned = [rho for rho in range(r) if rho % world == o]
        local = sum(1 for rho in owned for k in Kp[rho] if own_of(k) == o)
        assert local + Rv[o].sum() == len(owned) * Kp.shape[1]
        assert Rv[o][o] == 0


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_plan_consistent_across_ranks(world):
    _run(world, _plan_worker, 7)


# ------------------------------------------------------------------ 2. the decomposition
def _update_worker(rank, world, out_path):
    I, J, K, R, K0, bs = 24, 20, 30, 3, 24, 6
    T, truth = planted_dense(I, J, K, R, noise=0.01, seed=5)
    T0, batches = split_dense(T, K0, bs)
    model = [np.asarray(x, np.float32).astype(np.float64) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    r = 2 * world
    cfg = O.Config(R=R, s=(2, 2, 2), r=r, seed=3, maxit=8, tol=0.0, tau=0.0)
    # reference: single-process oracle update
    ref = O.init_factors(T0, cfg, *(x.astype(np.float32) for x in model), T.size)
    O.update(ref, batches[0])
    # sharded: slabs of X0 (contiguous), the batch split by the partition rule
    b0, n0 = partition(K0, world, rank)
    Kn = batches[0].shape[0]
    bb, bn = partition(Kn, world, rank)
    slab = np.concatenate([T0[b0:b0 + n0], batches[0][bb:bb + bn]])          # local slices
    kmap = np.concatenate([np.arange(b0, b0 + n0), K0 + np.arange(bb, bb + bn)])
    st = O.init_factors(T0, cfg, *(x.astype(np.float32) for x in model), T.size)
    S = st.S
    # a1: local marginals -> all-reduce (int64)
    x1, x2, x3l = O.marginals_dense(slab, S, cfg.moi)
    x3 = np.zeros(K0 + Kn, np.int64)
    x3[kmap] = x3l
    buf = torch.from_numpy(np.concatenate([x1, x2, x3]).astype(np.int64))
    dist.all_reduce(buf)
    xs = buf.numpy()
    g1, g2, g3 = O.marginals_dense(np.concatenate([T0, batches[0]]), S, cfg.moi)
    assert np.array_equal(xs, np.concatenate([g1, g2, g3]))
    x1, x2, x3 = xs[:I], xs[I:I + J], xs[I + J:]
    uid = 1
    owner_of = {int(k): g for g in range(world)
                for k in np.concatenate([np.arange(*[partition(K0, world, g)[0], sum(partition(K0, world, g))]),
                                         K0 + np.arange(partition(Kn, world, g)[0], sum(partition(Kn, world, g)))])}
    local_of = {int(k): i for i, k in enumerate(kmap)}
    owned = {}
    parts = {}
    for rho in range(r):
        Is = O.sample_mode(x1, O.sample_size(I, 2), cfg.seed, uid, rho, 0)
        Js = O.sample_mode(x2, O.sample_size(J, 2), cfg.seed, uid, rho, 1)
        Ks = O.sample_mode(x3[:K0], O.sample_size(K0, 2), cfg.seed, uid, rho, 2)
        Kp = O.k_prime(Ks, K0, Kn)
        # a3: the slices of rep rho this rank stores
        mine = {u: O.gather_dense(slab, Is, Js, np.array([local_of[int(k)]]))[:, :, 0]
                for u, k in enumerate(Kp) if owner_of[int(k)] == rank}
        parts[rho] = (Is, Js, Ks, Kp, mine)
    # exchange (all-gather of the parts stands in for the all-to-all-v)
    allparts = [None] * world
    dist.all_gather_object(allparts, {rho: p[4] for rho, p in parts.items()})
    recs = {}
    for rho in range(r):
        if rho % world != rank:
            continue
        Is, Js, Ks, Kp, _ = parts[rho]
        Y = np.empty((len(Is), len(Js), len(Kp)), np.float32)
        for g in range(world):
            for u, sl in allparts[g][rho].items():
                Y[:, :, u] = sl
        assert np.array_equal(Y, O.gather_dense(np.concatenate([T0, batches[0]]), Is, Js, Kp))
        U0 = O.als_init((len(Is), len(Js), len(Kp)), R, cfg.seed, uid, rho)
        lam_p, Up, fit, its, _ = O.cp_als(Y, U0, cfg.maxit, cfg.tol)
        rm = O.match_rep(st.A, st.B, st.C, Is, Js, Ks, lam_p, Up, cfg.tau)
        recs[rho] = (Up, rm)
    allrecs = [None] * world
    dist.all_gather_object(allrecs, recs)
    allr = {}
    for d_ in allrecs:
        allr.update(d_)
    # a6: replicated merge in rep order (as O.update)
    acc = [rho for rho in range(r) if allr[rho][1].accepted]
    A, B, C = st.A.copy(), st.B.copy(), st.C.copy()
    for m, (F, key) in enumerate(((A, 0), (B, 1), (C, 2))):
        tot = np.zeros_like(F); cnt = np.zeros(F.shape[0])
        for rho in acc:
            rows = parts[rho][key]
            Ut = O.rescaled(allr[rho][0], allr[rho][1], m)[:len(rows)]
            tot[rows] += Ut
            cnt[rows] += 1.0
        hit = cnt > 0
        mean = tot[hit] / cnt[hit][:, None]
        F[hit] = np.where(F[hit] == 0.0, mean, F[hit])
    C_new = sum(O.rescaled(allr[rho][0], allr[rho][1], 2)[len(parts[rho][2]):] for rho in acc) / len(acc)
    lam = (st.lam + sum(allr[rho][1].lam_hat for rho in acc) / len(acc)) / 2.0
    C = np.vstack([C, C_new])
    for x, y in zip((lam, A, B, C), (ref.lam, ref.A, ref.B, ref.C)):
        assert np.array_equal(x, y)
    if rank == 0:
        open(out_path, "w").write("ok")


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_decomposition_equals_single_process_oracle(world, tmp_path):
    out = tmp_path / "done"
    _run(world, _update_worker, str(out))
    assert out.read_text() == "ok"


# ------------------------------------------------------------- 3. the sharded COO summaries
def _coo_worker(rank, world, out_path):
    """COO store sharded by slice ownership (X0 slabs, then every batch split by the partition
    rule, so after the first update a rank's old slices interleave with the others'): local
    marginals + all-reduce equal the global ones; each rank's local gather of a summary
    (canonical within its slices), concatenated on the owner in rank order and stably sorted by
    u, equals the gather over the whole tensor -- the owner assembly of the sharded COO update."""
    from synth import zipf_planted_coo, split_coo
    I, J, K, R, K0, bs = 300, 240, 60, 3, 40, 5
    Xa, truth = zipf_planted_coo(I, J, K, R, 30000, alpha=1.2, seed=3)
    X = O.Coo(Xa.i.astype(np.int64), Xa.j.astype(np.int64), Xa.k.astype(np.int64), Xa.v, Xa.dims)
    owner = np.empty(K, np.int64)
    b0, n0 = partition(K0, world, rank)
    for g in range(world):
        gb, gn = partition(K0, world, g)
        owner[gb:gb + gn] = g
    for k0 in range(K0, K, bs):
        kn = min(bs, K - k0)
        for g in range(world):
            gb, gn = partition(kn, world, g)
            owner[k0 + gb:k0 + gb + gn] = g
    S = O.fixed_point_scale(X.nnz, float(np.abs(X.v).max()))
    for Ko in (K0, K0 + bs, K0 + 2 * bs):      # three consecutive updates
        Kt = Ko + bs
        sel = X.k < Kt
        full = O.Coo(X.i[sel], X.j[sel], X.k[sel], X.v[sel], (I, J, Kt))
        mine = sel & (owner[X.k] == rank)
        loc = O.Coo(X.i[mine], X.j[mine], X.k[mine], X.v[mine], (I, J, Kt))
        x = np.concatenate(O.marginals_coo(loc, S, O.MOI_ABS)).astype(np.int64)
        t = torch.from_numpy(x.copy())
        dist.all_reduce(t)
        g1, g2, g3 = O.marginals_coo(full, S, O.MOI_ABS)
        assert np.array_equal(t.numpy(), np.concatenate([g1, g2, g3]))
        for rho in range(2 * world):
            Is = O.sample_mode(g1, O.sample_size(I, 2), 5, 1, rho, 0)
            Js = O.sample_mode(g2, O.sample_size(J, 2), 5, 1, rho, 1)
            Ks = O.sample_mode(g3[:Ko], O.sample_size(Ko, 2), 5, 1, rho, 2)
            Kp = O.k_prime(Ks, Ko, bs)
            part = O.gather_coo(loc, Is, Js, Kp)
            parts = [None] * world
            dist.all_gather_object(parts, (part.i, part.j, part.k, part.v))
            cat = [np.concatenate([p[a] for p in parts]) for a in range(4)]
            order = np.argsort(cat[2], kind="stable")   # stable sort by u
            ref = O.gather_coo(full, Is, Js, Kp)
            for got, want in zip((c[order] for c in cat), (ref.i, ref.j, ref.k, ref.v)):
                assert np.array_equal(got, want)
    if rank == 0:
        open(out_path, "w").write("ok")


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_coo_summaries_equal_full_gather(world, tmp_path):
    out = tmp_path / "done"
    _run(world, _coo_worker, str(out))
    assert out.read_text() == "ok"


# --------------------------------------------------------------------------- 3. full-tensor ALS
def _full_als_worker(rank, world, iters):
    """The sharded full-tensor CP-ALS (run_dense_als_sharded) written with
    the oracle's building blocks: slab MTTKRP partials of modes 0 and 1 all-reduced, mode-2
    rows all-gathered, replicated solves -- must reproduce the single-process oracle CP-ALS."""
    T, truth = planted_dense(18, 15, 23, 3, noise=0.01, seed=62)
    K = T.shape[0]
    k0, kn = partition(K, world, rank)
    slab = O.view_ijk(T[k0:k0 + kn]).astype(np.float64)
    U = O.als_init(O.view_ijk(T).shape, 3, 9, 0, 0)
    U_ref = [u.copy() for u in U]
    R = 3
    for _ in range(iters):
        for m in range(3):
            V = np.ones((R, R))
            for n in range(3):
                if n != m:
                    V *= U[n].T @ U[n]
            loc = [U[0], U[1], U[2][k0:k0 + kn]]
            M = O.mttkrp(slab, loc, m)
            if m < 2:
                t = torch.from_numpy(M.copy())
                dist.all_reduce(t)
                M = t.numpy()
            else:
                parts = [None] * world
                dist.all_gather_object(parts, (k0, M))
                M = np.zeros((K, R))
                for b0, Mp in parts:
                    M[b0:b0 + Mp.shape[0]] = Mp
            Um, _ = O.solve_normal(M, V)
            lam = np.sqrt(np.sum(Um * Um, axis=0))
            U[m] = Um / np.where(lam > 0, lam, 1.0)
    lam_ref, U_ref, fit_ref, it_ref, _ = O.cp_als(O.view_ijk(T), U_ref, iters, 0.0)
    for a, b in zip(U, U_ref):
        assert np.allclose(a, b, rtol=1e-9, atol=1e-12)
    assert np.allclose(lam, lam_ref, rtol=1e-9)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_full_als_decomposition(world):
    _run(world, _full_als_worker, 6)


# ------------------------------------------------- 5. GetRank in the sharded update (R33)
def _getrank_worker(rank, world, out_path):
    """Each rank rates its owned repetitions' summaries (rho = rank + t G, Philox reps
    rho * trials + j as on one GPU); an allgather in rank-major order, read back as repetition
    g + t G (capi_dist.inc dist_share_ranks), must give the single-process update's ranks."""
    from oracle import getrank as GR
    rng = np.random.default_rng(1)
    I, J, K, K0, R, F_true = 40, 36, 30, 24, 3, 2
    A, B, C = rng.random((I, R)), rng.random((J, R)), rng.random((K, R))
    C[:, F_true:] = 0.0
    T = np.ascontiguousarray(np.transpose(np.einsum("if,jf,kf->ijk", A, B, C), (2, 1, 0))).astype(np.float32)
    T0, batch = T[:K0], T[K0:]
    r, trials = 2 * world, 2
    cfg = O.Config(R=R, s=(2, 2, 2), r=r, seed=6, maxit=60, tol=1e-9, tau=0.0, getrank=True, getrank_trials=trials)
    ref = O.init_factors(T0, cfg, np.ones(R), A, B, C[:K0], T0.size * 2)
    want = [rp["rank"] for rp in O.update(ref, batch)["reps"]]
    st = O.init_factors(T0, cfg, np.ones(R), A, B, C[:K0], T0.size * 2)
    X = np.concatenate([T0, batch])
    x1, x2, x3 = O.marginals_dense(X, st.S, cfg.moi)
    uid, Kn = 1, batch.shape[0]
    own = []
    for t in range(r // world):
        rho = rank + t * world
        Is = O.sample_mode(x1, O.sample_size(I, 2), cfg.seed, uid, rho, 0)
        Js = O.sample_mode(x2, O.sample_size(J, 2), cfg.seed, uid, rho, 1)
        Ks = O.sample_mode(x3[:K0], O.sample_size(K0, 2), cfg.seed, uid, rho, 2)
        Y = O.gather_dense(X, Is, Js, O.k_prime(Ks, K0, Kn))
        rn, _ = GR.getrank(Y, R, trials, cfg.seed, cfg.maxit, cfg.tol, cfg.getrank_threshold, rep_base=rho * trials)
        own.append(rn)
    gathered = [None] * world
    dist.all_gather_object(gathered, own)
    flat = [x for g in gathered for x in g]          # rank-major, as the NCCL allgather
    rloc = r // world
    got = [0] * r
    for g in range(world):
        for t in range(rloc):
            got[g + t * world] = flat[g * rloc + t]
    assert got == want, (got, want)
    if rank == 0:
        open(out_path, "w").write("ok")


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_getrank_ranks_equal_single_process(world, tmp_path):
    out = tmp_path / "done"
    _run(world, _getrank_worker, str(out))
    assert out.read_text() == "ok"
