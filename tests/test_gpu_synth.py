"""On-device planted generator (synth/csrc/gen.cu) against its numpy twin, and the
borrowed-store init (opts.borrow_store) against the copying init."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_device_generator_matches_numpy_twin():
    import torch
    from synth import gpu as G
    from synth.planted import dense_philox_slab, planted_dense_factors, planted_sigma
    G.build()
    A, B, Cf = planted_dense_factors(36, 22, 17, 4, 3)
    sigma = planted_sigma(A, B, Cf, 0.01)
    dA, dB, dC = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (A, B, Cf))
    for k0, nk, sg in ((0, 17, sigma), (5, 7, sigma), (3, 4, 0.0)):
        out = torch.empty((nk, 22, 36), dtype=torch.float32, device="cuda")
        G.dense_slab(out, dA, dB, dC, sg, 11, k0, nk)
        ref = dense_philox_slab(A, B, Cf, sg, 11, k0, nk)
        got = out.cpu().numpy()
        if sg == 0.0:
            assert np.array_equal(got, ref)          # the clean part: same fp64 ops, same order
        else:                                      # libm vs CUDA log/sincos: <= 1 ulp after fl32
            assert np.max(np.abs(got.view(np.int32).astype(np.int64) - ref.view(np.int32))) <= 1


def test_borrowed_store_matches_copied_store():
    import torch
    from paper_1709_00668_b200 import _lib as L
    from synth import planted_dense, split_dense
    I, J, K, R, K0 = 40, 24, 30, 3, 20
    T, truth = planted_dense(I, J, K, R, noise=0.01, seed=2)
    T0, batches = split_dense(T, K0, 5)
    model = [np.ascontiguousarray(np.asarray(x, np.float32)) for x in (truth[0], truth[1], truth[2], truth[3][:K0])]
    store = torch.zeros((K, J, I), dtype=torch.float32, device="cuda")
    store[:K0] = torch.from_numpy(T0).cuda()
    outs = []
    for borrow in (0, 1):
        opts = L.default_opts(als_max_iters=10, als_tol=0.0, capacity=K, full_fit=1, borrow_store=borrow)
        X0 = L.dense(store[:K0]) if borrow else L.dense(torch.from_numpy(T0).cuda())
        h = L.sambaten_init_factors(X0, R, 2, 4, 5, model[1], model[2], model[3], model[0], opts)
        res = []
        for b in batches:
            info = L.sambaten_update(h, L.dense(torch.from_numpy(b).cuda()))
            res.append(info.fit_full)
        Ah = np.empty((I, R), np.float32); Bh = np.empty((J, R), np.float32)
        Ch = np.empty((K, R), np.float32); lh = np.empty(R, np.float32)
        L.sambaten_copy_factors(h, Ah, Bh, Ch, lh)
        outs.append((res, Ah, Bh, Ch, lh))
        L.sambaten_destroy(h)
    assert outs[0][0] == outs[1][0]
    for x, y in zip(outs[0][1:], outs[1][1:]):
        assert np.array_equal(x, y)
    # the borrowed buffer now holds every ingested slice
    assert np.array_equal(store.cpu().numpy(), T)


def test_borrow_store_rejects_host_memory():
    from paper_1709_00668_b200 import _lib as L
    T0 = np.ones((4, 6, 8), np.float32)
    opts = L.default_opts(capacity=8, borrow_store=1)
    with pytest.raises(L.SambatenError):
        L.sambaten_init_factors(L.dense(T0), 2, 2, 2, 0, np.ones((8, 2), np.float32), np.ones((6, 2), np.float32),
                                np.ones((4, 2), np.float32), np.ones(2, np.float32), opts)
