"""BASELINE.json configs C1..C5 (configs[0..4]) as workload descriptions."""
from dataclasses import dataclass


@dataclass(frozen=True)
class Workload:
    name: str
    fmt: str            # "dense" | "coo"
    I: int
    J: int
    K: int              # final extent of the growing mode
    K0: int             # initial slices
    batch: int          # slices per batch
    R: int
    s: int
    r: int
    maxit: int
    tol: float
    noise: float = 0.01
    nnz: int = 0
    alpha: float = 0.0
    seed: int = 0

    @property
    def n_batches(self):
        return -(-(self.K - self.K0) // self.batch)


CONFIGS = {
    # configs[0]: 50^3, R=3, K0=40 + 1 batch of 10, s=2, r=4, 50 iterations, tol 1e-6, seed 0
    "C1": Workload("C1", "dense", 50, 50, 50, 40, 10, 3, 2, 4, 50, 1e-6),
    # configs[1]: 500^3, R=10, K0=450 + 5 batches of 10, s=5, r=8, 30 iterations
    "C2": Workload("C2", "dense", 500, 500, 500, 450, 10, 10, 5, 8, 30, 1e-6),
    # configs[2]: 64K x 64K x 1600, ~2M nnz, Zipf 1.5 communities R=15, 1400 + 4 x 50 days, s=10, r=8
    "C3": Workload("C3", "coo", 65536, 65536, 1600, 1400, 50, 15, 10, 8, 30, 1e-6,
                   nnz=2_000_000, alpha=1.5),
    # configs[3]: 3000^2 x (2700 -> 3000) in batches of 50, R=10, 1% noise, s=10, r=16
    "C4": Workload("C4", "dense", 3000, 3000, 3000, 2700, 50, 10, 10, 16, 30, 1e-6),
    # profiling stand-in for C4 (not a BASELINE config): the same 3000 x 3000 slices, K = 300,
    # small enough for ncu kernel replay
    "C4s": Workload("C4s", "dense", 3000, 3000, 300, 270, 5, 10, 10, 16, 30, 1e-6),
    # profiling stand-in for C4's a4 grid plan (not a BASELINE config): 3000 x 3000 x 600 slices
    # (K0 = 550 + 50), summaries 300 x 300 x 105 -> 12 slices per CTA of the 9-CTA grid plan
    "C4p": Workload("C4p", "dense", 3000, 3000, 600, 550, 50, 10, 10, 16, 30, 1e-6),
    # configs[4]: 100K^3, ~100M nnz, planted rank 10 Zipf 1.2, 90K + batches of 1K, s=20, r=8
    "C5": Workload("C5", "coo", 100_000, 100_000, 100_000, 90_000, 1000, 10, 20, 8, 30, 1e-6,
                   nnz=100_000_000, alpha=1.2),
}
