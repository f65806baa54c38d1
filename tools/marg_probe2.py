"""GPU probe: dense marginal pass on 3000 x 3000 x K (dev tool; SBT_MARG_* env experiments)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1709_00668_b200 import _lib as L
I = J = 3000; K = int(os.environ.get("PROBE_K", 600))
X = torch.rand((K, J, I), device="cuda")
x = [torch.zeros(n, dtype=torch.int64, device="cuda") for n in (I, J, K)]
best = 1e9
for rep in range(5):
    for v in x: v.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); L.sambaten_marginals(L.dense(X), 0, 20, *x); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(os.environ.get("PROBE_TAG", ""), round(best, 3), "ms", round(4 * I * J * K / best / 1e6, 1), "GB/s")
