"""GPU probe: COO marginals at C5 scale (100K^3, 1e8 entries, Zipf 1.2 over 10 permuted
components, sorted by (k, j, i)), timed per kernel variant (dev tool; env knobs of k_marginals.cu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1709_00668_b200 import _lib as L

N, R, nnz, a = 100_000, 10, int(os.environ.get("PROBE_NNZ", 100_000_000)), 1.2
g = torch.Generator(device="cuda").manual_seed(0)
w = torch.arange(1, N + 1, device="cuda", dtype=torch.float64) ** -a
cdf = torch.cumsum(w / w.sum(), 0)
perms = torch.stack([torch.randperm(N, device="cuda", generator=g) for _ in range(R)])
def draw(n):
    f = torch.randint(0, R, (n,), device="cuda", generator=g)
    r = torch.searchsorted(cdf, torch.rand(n, device="cuda", generator=g, dtype=torch.float64)).clamp_(max=N - 1)
    return perms[f, r]
i, j = draw(nnz), draw(nnz)
k = torch.randint(0, N, (nnz,), device="cuda", generator=g)
key = (k * N + j) * N + i
key, _ = torch.sort(key)
i, j, k = (key % N).int(), ((key // N) % N).int(), (key // (N * N)).int()
del key
v = torch.rand(nnz, device="cuda", generator=g).float() + 0.1
x = [torch.zeros(N, dtype=torch.int64, device="cuda") for _ in range(3)]
t = L.coo(i, j, k, v, (N, N, N))
ref = None
for rep in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); L.sambaten_marginals(t, 0, 6, *x); e1.record(); torch.cuda.synchronize()
    if ref is None:
        ref = [y.clone() for y in x]
    else:
        assert all(torch.equal(y, z) for y, z in zip(x, ref))
print(os.environ.get("PROBE_TAG", ""), "ms", round(e0.elapsed_time(e1), 3), "GB/s", round(16 * nnz / e0.elapsed_time(e1) / 1e6, 1))
