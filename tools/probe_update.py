"""GPU probe: run a few updates of a config and print per-step times (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1709_00668_b200 import _lib as L
from synth import planted_dense, split_dense, CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = CONFIGS[cfg]
T, truth = planted_dense(w.I, w.J, w.K, w.R, noise=w.noise, seed=w.seed)
T0, batches = split_dense(T, w.K0, w.batch)
model = [np.ascontiguousarray(np.asarray(x, np.float32)) for x in (truth[0], truth[1], truth[2], truth[3][:w.K0])]
tol = float(os.environ.get("PROBE_TOL", w.tol))   # PROBE_TOL=0: fixed iteration count
opts = L.default_opts(als_max_iters=w.maxit, als_tol=tol, capacity=w.K, full_fit=1, accept_tau=0.0 if os.environ.get("PROBE_TOL") else w.tau if hasattr(w, "tau") else 0.9)
h = L.sambaten_init_factors(L.dense(torch.from_numpy(T0).cuda()), w.R, w.s, w.r, w.seed,
                            model[1], model[2], model[3], model[0], opts)
L.sambaten_checkpoint(h)
db = [torch.from_numpy(b).cuda() for b in batches]
for i in range(n):
    if i % len(db) == 0 and i:
        L.sambaten_restore(h)
    info = L.sambaten_update(h, L.dense(db[i % len(db)]))
    d = info.as_dict()
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in d.items() if k != "step_ms"}),
          [round(x, 3) for x in d["step_ms"]])
L.sambaten_destroy(h)
