import sys, torch, numpy as np
sys.path.insert(0, "/root/repo")
from paper_1709_00668_b200 import _lib as L
I = J = 3000
for K in (50, 100, 300):
    X = torch.rand((K, J, I), device="cuda")
    x = [torch.zeros(n, dtype=torch.int64, device="cuda") for n in (I, J, K)]
    for rep in range(3):
        for v in x: v.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); L.sambaten_marginals(L.dense(X), 0, 20, *x); e1.record(); torch.cuda.synchronize()
    print(K, "slices", round(e0.elapsed_time(e1), 3), "ms", round(4 * I * J * K / e0.elapsed_time(e1) / 1e6, 1), "GB/s")
