"""bench.py -- SamBaTen per-batch incremental CP update on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]

A step is one whole update (a0..a7: ingest, marginals, sampling, gather, batched CP-ALS,
matching, merge, full fit) of one batch of a BASELINE.json workload with synthetic planted
data.  Default: configs[3] = C4 (3000^2 x 2700 -> 3000 dense, 108 GB on the device, batches of
50 slices, R=10, s=10, r=16, 30 ALS iterations), the largest config that fits one GPU; its
summary ALS is warm-started from the model's rows (reading R34) with the acceptance test
(tau = 0.9, R26), the setting whose model keeps converging (a cold 30-iteration start on the
300 x 300 x 320 summaries does not converge and the paper-literal merge decays the model; that
run is reported as the variant "cold_start_paper_literal").  --config C1/C2/C3/C5 select the
other workloads (C3/C5: COO).
The metric is BASELINE.json's: new tensor entries (dense) / nonzeros (COO) ingested per
second per update.  Rank 0 prints one JSON line.

Timing: W untimed warm-up steps, then K steps, each bracketed by a barrier and a device
synchronisation and timed with CUDA events on the library's stream; L2 is flushed (a 512 MB
write) before every step; the stream cycles through the config's batches, restoring the
K0 checkpoint (untimed) after the last one.  Multi-GPU (torchrun): ONE update of the same
workload sharded over the N ranks (sambaten_init_factors_dist: time-mode slabs,
int64 allreduce of the marginals, all-to-all-v of summary slices, repetition rho on rank
rho mod N, allgather before the replicated merge) -- strong scaling;
the time is the max over ranks and `value` counts the batch's entries once (dense and COO
stores alike).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=60)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C4",
                   help="BASELINE workload; default C4 = configs[3], the largest single-GPU config")
    p.add_argument("--als-init", default="config", choices=["config", "cold", "warm"],
                   help="summary ALS start: the config's setting (C4: warm, R34), the Philox point "
                        "(P:213, R10) or the model's rows (R34)")
    p.add_argument("--tau", type=float, default=None, help="override the acceptance threshold (R26)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-variant", action="store_true", help="skip the incremental-marginals variant run")
    p.add_argument("--no-getrank", action="store_true", help="skip the GetRank timing (SURVEY 8(f) NEXT #2)")
    p.add_argument("--no-full-fit", action="store_true", help="return the summary fit only (R21)")
    p.add_argument("--full-fit", type=int, default=None, choices=[1, 2],
                   help="1 (single-GPU default): the committed model's fit (dense: incremental -- the batch "
                        "plus the rows the merge changed, k_fitinc.cu); 2 (sharded dense default: the sharded "
                        "handle has no incremental fit, so its exact fit would be a second pass over the slab): "
                        "lag-1 fit inside the next update's a1 pass (SURVEY 8(f) NEXT #1; dense only, COO "
                        "configs use 1)")
    p.add_argument("--no-recompute", action="store_true", help="skip the CP_ALS recompute / relative fitness report")
    p.add_argument("--recompute-iters", type=int, default=150, help="CP_ALS baseline iteration cap (P:441 uses 1000)")
    p.add_argument("--sharded", action="store_true",
                   help="use the sharded (NCCL) handle even at N=1 (always used at N>1, dense configs)")
    return p.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 20 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.05)
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0])); smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- workloads
class Work:
    """Synthetic stand-in of a BASELINE config."""

    def __init__(self, w):
        self.w = w
        self.coo = w.fmt == "coo"
        if not self.coo:
            from synth import planted_dense, split_dense
            T, truth = planted_dense(w.I, w.J, w.K, w.R, noise=w.noise, seed=w.seed)
            self.X0, self.batches = split_dense(T, w.K0, w.batch)
            self.model = [np.asarray(x, np.float32) for x in (truth[0], truth[1], truth[2], truth[3][:w.K0])]
            self.entries = [b.size for b in self.batches]
            self.cap = w.I * w.J * w.K
        else:
            from synth import community_coo, zipf_planted_coo, split_coo
            if w.name == "C3":
                X = community_coo(w.I, w.K, w.R, w.nnz, alpha=w.alpha, seed=w.seed)
                self.model = None           # no planted factors: sambaten_init (full ALS, untimed)
            else:
                X, truth = zipf_planted_coo(w.I, w.J, w.K, w.R, w.nnz, alpha=w.alpha, seed=w.seed)
                self.model = [np.asarray(x, np.float32) for x in (truth[0], truth[1], truth[2], truth[3][:w.K0])]
            self.X0, self.batches = split_coo(X, w.K0, w.batch)
            self.entries = [b.nnz for b in self.batches]
            self.cap = X.nnz
        self.nb = len(self.batches)

    def tensor(self, L, x, device, pin=False):
        import torch
        if not self.coo:
            t = torch.from_numpy(np.ascontiguousarray(x))
            return L.dense(t.cuda() if device else (t.pin_memory() if pin else t))
        arrs = [torch.from_numpy(np.ascontiguousarray(a)) for a in (x.i, x.j, x.k, x.v)]
        arrs = [a.cuda() if device else (a.pin_memory() if pin else a) for a in arrs]
        return L.coo(*arrs, x.dims)

    def bytes_in(self, i):
        b = self.batches[i]
        return int(b.size * 4) if not self.coo else int(b.nnz * 16)

    def oracle_tensor(self, x):
        from oracle import sambaten as O
        if not self.coo:
            return x
        return O.Coo(x.i.astype(np.int64), x.j.astype(np.int64), x.k.astype(np.int64), x.v, x.dims)


class DeviceWork:
    """The large dense config (C4: 3000^2 x 3000, 108 GB) generated ON THE DEVICE by the
    counter-based planted generator (synth/csrc/gen.cu): the
    store buffer holds X0 in place (opts.borrow_store) and each batch is its own device buffer."""

    def __init__(self, w, world, rank):
        import torch
        from synth import gpu as G
        from synth.planted import planted_dense_factors, planted_sigma
        self.w, self.coo, self.device_gen = w, False, True
        A, B, Cf = planted_dense_factors(w.I, w.J, w.K, w.R, w.seed)
        self.sigma = planted_sigma(A, B, Cf, w.noise)
        dA, dB, dC = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (A, B, Cf))
        self.gen = lambda out, k0, nk: G.dense_slab(out, dA, dB, dC, self.sigma, w.seed, k0, nk)
        self.model = [np.ones(w.R, np.float32), A.astype(np.float32), B.astype(np.float32),
                      np.ascontiguousarray(Cf[:w.K0].astype(np.float32))]
        self.cap = w.I * w.J * w.K
        self.nb = w.n_batches
        self.batches = []
        for b in range(self.nb):
            k0 = w.K0 + b * w.batch
            nk = min(w.batch, w.K - k0)
            t = torch.empty((nk, w.J, w.I), dtype=torch.float32, device="cuda")
            self.gen(t, k0, nk)
            self.batches.append(t)
        self.entries = [int(b.numel()) for b in self.batches]
        torch.cuda.synchronize()

    def tensor(self, L, x, device, pin=False):
        if device:
            return L.dense(x)
        return L.dense(x.cpu().pin_memory() if pin else x.cpu())

    def bytes_in(self, i):
        return int(self.batches[i].numel() * 4)


def describe(w):
    if w.fmt == "dense":
        shape = f"dense {w.I}x{w.J}x{w.K}, K0={w.K0}, batch={w.batch} slices"
    else:
        shape = f"COO {w.I}x{w.J}x{w.K} ~{w.nnz} nnz (Zipf {w.alpha}), K0={w.K0}, batch={w.batch} slices"
    return f"{w.name}: {shape}, R={w.R}, s={w.s}, r={w.r}, ALS {w.maxit} it tol {w.tol}"


FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4: SMs x FP32 lanes x FMA x max clock
L2_RESIDENT_BYTES = 100e6                           # summaries below this stay in the 126 MB L2


# read-only HBM ceiling: tools/micro/read_bw.cu (40 GB, cp.async.bulk ring of 2-6 stages per SM, no
# compute; LDG.128 streaming 7.41 TB/s) on this pool's B200 -> profiles/r02_read_ceiling.txt
READ_CEILING_GBS = 7433.0


def kernel_rooflines(w, work, infos, peaks, peak_kind, G, k_local, args):
    """Per-step roofline of the dominant kernel of each streaming / ALS step, from the steps'
    CUDA-event times (info.step_ms, on the library's stream) and the algorithmic work of
    DESIGN.md "Kernels": a1 4 B per stored entry (+ 8 B per marginal), a3 8 B per summary entry
    (read + write), a4 per ALS iteration 2 passes x 4 B (HBM) or 2R flops (fp32 FMA) per summary
    entry, a7 4 B per stored entry."""
    def ms(k):
        return statistics.mean(inf["step_ms"][k] for inf in infos)
    traffic = {}
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(w.name, {})
        except Exception:
            traffic = {}
    hbm = peaks["hbm_gbs"]
    out = {}

    def hbm_line(name, step, byts):
        t = ms(step)
        ach = byts / (t / 1e3) / 1e9
        # MEASURED_PEAKS' hbm_gbs is a copy (read + write) figure; a read-only stream can exceed it:
        # the read ceiling measured on this pool's B200 (TMA ring, no compute) is reported beside it
        return {"kernel": name, "bound": "hbm", "achieved": ach, "peak": hbm, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": ach / hbm, "traffic": traffic.get(f"a{step}"),
                "read_ceiling": READ_CEILING_GBS, "frac_of_read_ceiling": ach / READ_CEILING_GBS,
                "bytes_per_launch": byts, "ms_per_launch": t}
    Ks = [inf["k_total"] for inf in infos]
    if work.coo:
        nnz_avg = work.X0.nnz + statistics.mean(
            sum(work.entries[:(j % work.nb) + 1]) for j in range(args.warmup, args.warmup + args.steps))
        out["a1"] = hbm_line("marg_coo_kernel", 1, 16.0 * nnz_avg + 8.0 * (w.I + w.J + statistics.mean(Ks)))
        # per ALS iteration, 3 mode passes of 16 B (i, j, k, v) per summary nonzero
        nz = statistics.mean(inf["summary_entries"] for inf in infos)
        it = statistics.mean(inf["als_iters_sum"] for inf in infos) / w.r
        kinds = {inf["als_plan"][0] for inf in infos}
        kname = ("coo_als_persist_kernel (all iterations, one cooperative launch; sort + piece plan before it)"
                 if kinds == {3} else "COO ALS per-mode pipeline (piece MTTKRP, row solves)" if kinds == {4}
                 else f"COO ALS (plan kinds {sorted(kinds)})")
        out["a4"] = dict(hbm_line(kname, 4, it * 3 * 16.0 * nz),
                         note="algorithmic bytes: iterations x 3 mode passes x 16 B per summary nonzero "
                              "(SURVEY 8(d)); summaries smaller than L2 can exceed the HBM line")
        return out
    Kloc = k_local if k_local is not None else Ks
    IJ = w.I * w.J
    lag = all(inf.get("fit_full_prev", -1.0) != -1.0 for inf in infos)
    incfit = all(inf.get("fit_path", 0) == 3 for inf in infos)
    out["a1"] = hbm_line("margfit_stream_kernel (a1 + lag-1 fit) + marg_stream_kernel (batch)" if lag
                         else "marg_stream_kernel", 1,
                         statistics.mean(4.0 * IJ * kl for kl in Kloc) + 8.0 * (w.I + w.J + statistics.mean(Ks)))
    if incfit:   # the batch's slices (+ changed rows): 4 B per new entry
        out["a7"] = dict(hbm_line("fitrows_kernel (incremental fit: the batch's slices)", 7,
                                  statistics.mean(4.0 * IJ * w.batch for _ in Kloc)),
                         note="incremental exact fit (k_fitinc.cu): reads only the new slices")
    elif not lag:
        out["a7"] = hbm_line("fit_stream_kernel", 7, statistics.mean(4.0 * IJ * kl for kl in Kloc))
    nI, nJ = -(-w.I // w.s), -(-w.J // w.s)
    Y = []
    for inf, kt in zip(infos, Ks):
        Kn = w.batch if kt - w.K0 >= w.batch else kt - w.K0
        Ko = kt - Kn
        Y.append(nI * nJ * (-(-Ko // w.s) + Kn))
    Ymean = statistics.mean(Y)
    rl = w.r / G
    out["a3"] = hbm_line("gather_dense_kernel", 3, 8.0 * rl * Ymean)
    it = statistics.mean(inf["als_iters_sum"] for inf in infos) / G
    t4 = ms(4)
    kinds = {inf["als_plan"][0] for inf in infos}
    a4name = {frozenset({1}): "als_cluster_kernel (cluster plan: one thread-block cluster per repetition)",
              frozenset({2}): "als_cluster_kernel (grid plan: CTA groups of one cooperative grid)",
              frozenset({0}): "multi-kernel ALS (mttkrp0 / dpass / solve kernels)"}.get(
                  frozenset(kinds), f"dense ALS (plan kinds {sorted(kinds)})")
    if rl * Ymean * 8.0 <= L2_RESIDENT_BYTES:     # Y and its transpose stay in L2: fp32 FMA bound
        fl = it * 2 * Ymean * 2 * w.R
        ach = fl / (t4 / 1e3) / 1e12
        out["a4"] = {"kernel": a4name, "bound": "alu", "achieved": ach,
                     "peak": FP32_PEAK_TFLOPS, "peak_kind": "derived (148 SMs x 128 FP32 lanes x 2 x 1.965 GHz)",
                     "unit": "TFLOP/s", "frac": ach / FP32_PEAK_TFLOPS, "traffic": traffic.get("a4"),
                     "flops_per_launch": fl, "ms_per_launch": t4,
                     "note": "summaries L2-resident (SURVEY 8(d)): HBM fraction not meaningful"}
    else:
        out["a4"] = hbm_line(a4name, 4, it * 2 * Ymean * 4.0)
    return out


def init_single(L, work, w, opts, config):
    """A single-GPU handle for the workload (untimed): planted factors, full CP-ALS of X0 (C3),
    or the device-generated store held in place (C4)."""
    import torch
    if work.model is None:
        X0 = work.tensor(L, work.X0, device=True)
        opts.init_max_iters = 50
        h = L.sambaten_init(X0, w.R, w.s, w.r, w.seed, opts)
        m = [np.empty(w.R, np.float32), np.empty((w.I, w.R), np.float32), np.empty((w.J, w.R), np.float32),
             np.empty((w.K0, w.R), np.float32)]
        L.sambaten_copy_factors(h, m[1], m[2], m[3], m[0])
        work.model = m                  # the oracle baseline (and a re-init) start from the same model
        return h
    if getattr(work, "device_gen", False):
        # the whole-tensor store is one device buffer holding X0 in place (no second copy)
        if getattr(work, "store", None) is None:
            work.store = torch.empty((w.K, w.J, w.I), dtype=torch.float32, device="cuda")
            work.gen(work.store[:w.K0], 0, w.K0)
        opts.borrow_store = 1
        config["store"] = "caller buffer (opts.borrow_store), X0 generated in place on the device"
        return L.sambaten_init_factors(L.dense(work.store[:w.K0]), w.R, w.s, w.r, w.seed, work.model[1],
                                       work.model[2], work.model[3], work.model[0], opts)
    X0 = work.tensor(L, work.X0, device=True)
    return L.sambaten_init_factors(X0, w.R, w.s, w.r, w.seed, work.model[1], work.model[2],
                                   work.model[3], work.model[0], opts)


def slab_of(x, k0, n, coo):
    """Slices [k0, k0 + n) of a dense (K, J, I) array or of a canonical COO (k re-based to 0)."""
    if not coo:
        return x[k0:k0 + n]
    from synth import CooArrays
    a, b = np.searchsorted(x.k, [k0, k0 + n])
    return CooArrays(x.i[a:b], x.j[a:b], (x.k[a:b] - k0).astype(np.int32), x.v[a:b], (x.dims[0], x.dims[1], n))


def getrank_timing(L, w, stream):
    """GetRank (Alg. 2) on one summary-sized planted tensor of the config
    (n_I x n_J x n_K' of the first batch, rank R, 1 % noise): candidate ranks 1..R+2, one trial,
    the config's ALS iterations; device time with CUDA events on the library's stream."""
    import torch
    from synth import planted_dense
    nI, nJ = -(-w.I // w.s), -(-w.J // w.s)
    nK = -(-w.K0 // w.s) + w.batch
    T, _ = planted_dense(nI, nJ, nK, w.R, noise=0.01, seed=w.seed + 17)
    X = L.dense(torch.from_numpy(T).cuda())
    Rmax = w.R + 2
    L.sambaten_getrank(X, Rmax, 1, w.seed, w.maxit, 0.0, 90.0, stream.cuda_stream)   # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    rn, cc = L.sambaten_getrank(X, Rmax, 1, w.seed, w.maxit, 0.0, 90.0, stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    return {"ms": e0.elapsed_time(e1), "R_new": rn, "R_planted": w.R, "candidate_ranks": Rmax, "trials": 1,
            "shape": [nI, nJ, nK], "als_iters": w.maxit,
            "best_cc": [round(float(x), 3) for x in cc.max(axis=1)]}


def partition(n, world, rank):
    """The library's balanced split (sambaten_batch_partition's rule) of n slices."""
    base, rem = divmod(n, world)
    return rank * base + min(rank, rem), base + (1 if rank < rem else 0)


def threads_used():
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count()


def oracle_state(work, model=None, tau=None, warm=False):
    from oracle import sambaten as O
    w = work.w
    cfg = O.Config(R=w.R, s=(w.s,) * 3, r=w.r, seed=w.seed, maxit=w.maxit, tol=w.tol,
                   tau=(0.9 if not work.coo else 0.0) if tau is None else tau, warm_start=warm)
    m = model if model is not None else work.model
    return O.init_factors(work.oracle_tensor(work.X0), cfg, *m, work.cap), O


def method_settings(w, args):
    """Summary-ALS start and acceptance threshold of the headline run of config w.
    C4, C5 (the large planted configs): warm start (R34) + tau = 0.9 -- the setting whose model
    keeps converging (the cold 30-iteration start decays both); dense C1/C2: cold
    start + tau = 0.9 (R26); C3: cold start, paper-literal tau = 0 (no planted model; its
    30-iteration summaries would fail the test)."""
    warm = w.name.startswith("C4") or w.name == "C5"   # C4s / C4p: C4's profiling stand-ins
    tau = 0.9 if w.fmt == "dense" else 0.0
    if args.als_init == "cold":
        warm, tau = False, (0.0 if w.name.startswith("C4") else tau)
    if w.name == "C5" and warm:
        tau = 0.9   # the planted model stays converged: the acceptance test applies (R26)
    elif args.als_init == "warm":
        warm = True
    if args.tau is not None:
        tau = args.tau
    return warm, tau


def oracle_sampled_update(w, warm, als_iters_per_rep, nslab=3, als_probe_iters=2):
    """The oracle (oracle/, as it stands) on a BOUNDED SAMPLE of one update of a device-sized
    dense config (C4: the 108 GB tensor does not fit the sample budget): each step of Alg. 1 is
    timed on a part of the real workload and scaled to the whole update by its work count.
      a1 marginals: `nslab` slices of the tensor (synth numpy twin of the device generator),
                    scaled by the update's stored entries;
      a2 sampling:  all r x 3 draws at the real sizes (weights from the slab's marginals);
      a3 gather:    one summary's rows over the slab's slices, scaled by r x |I_s||J_s||K'|;
      a4 ALS:       `als_probe_iters` iterations on one full-size |I_s| x |J_s| x |K'| summary
                    (planted, the config's rank), scaled by r x the GPU run's iterations per rep;
      a5 match:     one repetition, x r;   a7 fit: the slab, scaled by the stored entries.
    Returns (seconds per update, dict of per-step seconds, sample description)."""
    from oracle import sambaten as O
    from synth.planted import planted_dense_factors, planted_sigma, dense_philox_slab, dense_from_factors
    A, B, Cf = planted_dense_factors(w.I, w.J, w.K, w.R, w.seed)
    sigma = planted_sigma(A, B, Cf, w.noise)
    k0 = w.K0 - nslab
    slab = dense_philox_slab(A, B, Cf, sigma, w.seed, k0, nslab)
    Ktot = w.K0 + w.batch
    stored = float(w.I) * w.J * Ktot
    per = float(w.I) * w.J * nslab
    S = O.fixed_point_scale(w.I * w.J * w.K, float(np.abs(slab).max()))
    t = {}
    t0 = time.perf_counter()
    x1, x2, _ = O.marginals_dense(slab, S)
    t["a1"] = (time.perf_counter() - t0) * stored / per
    rng = np.random.default_rng(1)
    x3 = rng.integers(1, 1 << 40, size=w.K0, dtype=np.int64)
    nI, nJ, nK = O.sample_size(w.I, w.s), O.sample_size(w.J, w.s), O.sample_size(w.K0, w.s)
    t0 = time.perf_counter()
    for rho in range(w.r):
        Is = O.sample_mode(x1, nI, w.seed, 1, rho, 0)
        Js = O.sample_mode(x2, nJ, w.seed, 1, rho, 1)
        Ks = O.sample_mode(x3, nK, w.seed, 1, rho, 2)
    t["a2"] = time.perf_counter() - t0
    nKp = nK + w.batch
    t0 = time.perf_counter()
    Ys = O.gather_dense(slab, Is, Js, np.arange(nslab))
    t["a3"] = (time.perf_counter() - t0) * w.r * nKp / nslab
    Ksub = np.sort(np.concatenate([Ks[: nK], np.arange(w.K0, Ktot)]))[:nKp]
    Y = O.view_ijk(dense_from_factors(A[Is], B[Js], Cf[Ksub], w.noise, w.seed))
    U0 = O.als_init(Y.shape, w.R, w.seed, 1, 0)
    t0 = time.perf_counter()
    lam_p, Up, _, _, _ = O.cp_als(Y, U0, als_probe_iters, 0.0)
    t["a4"] = (time.perf_counter() - t0) / als_probe_iters * als_iters_per_rep * w.r
    if warm:
        t["a4"] += 0.0   # the warm rows are a copy (no arithmetic worth timing)
    lam = np.ones(w.R)
    t0 = time.perf_counter()
    O.match_rep(A, B, Cf, Is, Js, Ksub[: nK], lam_p, Up, 0.9)
    t["a5_a6"] = (time.perf_counter() - t0) * w.r
    t0 = time.perf_counter()
    O.relative_error(slab, lam, A, B, Cf[k0:k0 + nslab])
    t["a7"] = (time.perf_counter() - t0) * stored / per
    del Ys
    total = sum(t.values())
    desc = (f"oracle steps timed on parts of one {w.name} update and scaled by work: a1/a7 on {nslab} "
            f"slices ({per:.3g} of {stored:.3g} stored entries), a2 all {w.r}x3 draws, a3 one summary over "
            f"{nslab} slices (x {w.r} reps x {nKp}/{nslab}), a4 {als_probe_iters} ALS iterations on one "
            f"{nI}x{nJ}x{nKp} summary (x {w.r} reps x {als_iters_per_rep:.1f} iterations/rep), a5 one rep (x {w.r})")
    return total, t, desc


def cpu_baseline_run(work, model, tau, warm, budget_s=20.0):
    """The oracle as it stands (oracle/), on this host's cores: consecutive updates of the
    config's batches from the K0 state until ~budget_s seconds (bounded sample)."""
    st, O = oracle_state(work, model, tau=tau, warm=warm)
    t0 = time.perf_counter()
    entries, nb = 0, 0
    for i, b in enumerate(work.batches):
        try:
            O.update(st, work.oracle_tensor(b))
        except O.BatchRejected:
            pass
        entries += work.entries[i]
        nb += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return entries / dt, dt, nb


def main():
    args = parse()
    from synth import CONFIGS
    w = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    metric = "new tensor entries ingested/sec per update" if w.fmt == "dense" else \
        "new tensor nonzeros ingested/sec per update"
    unit = "entries/s" if w.fmt == "dense" else "nnz/s"
    config = {"workload": describe(w), "l2": "flushed (512 MB write) before every step",
              "init": "planted truth factors" if w.name != "C3" else "full CP-ALS of X0 (sambaten_init)",
              "full_fit": not args.no_full_fit}
    device_gen = w.name.startswith("C4")
    work = None if device_gen else Work(w)

    if args.impl == "reference":
        if rank != 0:
            return
        warm, tau = method_settings(w, args)
        config["accept_tau"] = tau
        config["als_init"] = "warm (R34)" if warm else "cold (Philox point, P:213)"
        cores = threads_used()
        times, ents = [], []
        if device_gen:
            # each step: the oracle on a bounded sample of one update, scaled to the whole update
            it_rep = 3.0 if warm else float(w.maxit)
            for i in range(args.warmup + args.steps):
                tot, parts, desc = oracle_sampled_update(w, warm, it_rep, nslab=2, als_probe_iters=1)
                if i >= args.warmup:
                    times.append(tot)
                    ents.append(w.I * w.J * w.batch)
            sample = desc + "; ALS iterations per rep assumed " + ("3 (warm start)" if warm else str(w.maxit))
        else:
            # consecutive updates of the config's batch stream from the K0 state (restored after
            # the last batch), as the GPU arm replays it; a rejected batch (R26) leaves the
            # state unchanged and still counts its work
            import copy
            from oracle import sambaten as O
            if work.model is None:
                cfg = O.Config(R=w.R, s=(w.s,) * 3, r=w.r, seed=w.seed)
                st0 = O.init_als(work.oracle_tensor(work.X0), cfg, work.cap, maxit=50, tol=1e-6)
                work.model = [np.asarray(x, np.float32) for x in (st0.lam, st0.A, st0.B, st0.C)]
            st_k0, O = oracle_state(work, tau=tau, warm=warm)
            st = copy.deepcopy(st_k0)
            rejected = 0
            for i in range(args.warmup + args.steps):
                bi = i % work.nb
                if bi == 0 and i > 0:
                    st = copy.deepcopy(st_k0)
                t0 = time.perf_counter()
                try:
                    O.update(st, work.oracle_tensor(work.batches[bi]))
                except O.BatchRejected:
                    rejected += 1
                dt = time.perf_counter() - t0
                if i >= args.warmup:
                    times.append(dt)
                    ents.append(work.entries[bi])
            sample = (f"each step = one full oracle update of the next batch of the {w.name} stream from the "
                      f"K0 state (restored after the last batch); {rejected} batch(es) rejected (R26)")
        tot = sum(times)
        val = sum(ents) / tot
        line = {"impl": "reference", "metric": metric, "value": val, "unit": unit, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / len(times),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded generators; DESIGN.md 'Synthetic inputs')", "config": config,
                "cpu_baseline": {"value": val, "unit": unit, "cores": cores, "kind": "oracle", "sample": sample},
                "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1709_00668_b200 import _lib as L
    if device_gen:
        work = DeviceWork(w, world, rank)

    sharded = world > 1 or args.sharded
    stream = torch.cuda.Stream()
    # summary-ALS start and acceptance threshold (method_settings: C4 warm + tau 0.9, dense
    # cold + tau 0.9, COO cold + tau 0)
    warm, tau = method_settings(w, args)
    config["accept_tau"] = tau
    config["als_init"] = "warm (model rows, R34)" if warm else "cold (Philox point, P:213)"
    ff_default = 2 if sharded else 1
    ff = 0 if args.no_full_fit else ((args.full_fit or ff_default) if not work.coo else 1)
    config["full_fit"] = {0: "none (summary fit only)",
                          1: "the committed model's exact fit (dense: incremental from the previous model's "
                             "per-component inner products -- the batch's slices plus the rows the merge changed; "
                             "COO: a pass over the nonzeros)",
                          2: "lag-1: the previous model's fit inside this update's a1 pass (NEXT #1)"}[ff]
    opts = L.default_opts(als_max_iters=w.maxit, als_tol=w.tol, capacity=work.cap, full_fit=ff,
                          accept_tau=tau, stream=stream.cuda_stream, warm_start=int(warm))
    if work.coo:
        opts.capacity_k = w.K
    else:
        opts.capacity = w.K
    local_batches = work.batches
    if sharded:
        nid = L.sambaten_dist_unique_id() if rank == 0 else None
        if world > 1:
            box = [nid]
            dist.broadcast_object_list(box, src=0)
            nid = box[0]
        if work.model is None:
            # C3: the initial model = full CP-ALS of X0, computed identically on every rank
            L.sambaten_destroy(init_single(L, work, w, opts, config))
        k0b, k0n = partition(w.K0, world, rank)
        if device_gen:
            # the slab generated in place in a buffer with room for this rank's share of the
            # stream (Kcap_local slices), used as the local store (opts.borrow_store, no copy)
            kcap_local = k0n + -(-(w.K - w.K0) // world) + 1
            work.x0buf = torch.empty((kcap_local, w.J, w.I), dtype=torch.float32, device="cuda")
            work.gen(work.x0buf[:k0n], k0b, k0n)
            X0 = L.dense(work.x0buf[:k0n])
            opts.borrow_store = 1
            config["store"] = "caller buffer (opts.borrow_store), the rank's slab generated in place on the device"
        else:
            X0 = work.tensor(L, slab_of(work.X0, k0b, k0n, work.coo), device=True)
        dd = L.make_dist(rank, world, nid, k0b, w.K0)
        h = L.sambaten_init_factors_dist(X0, dd, w.R, w.s, w.r, w.seed, work.model[1], work.model[2],
                                         work.model[3], work.model[0], opts)
        parts = [L.sambaten_batch_partition(h, b.dims[2] if work.coo else b.shape[0]) for b in work.batches]
        local_batches = [slab_of(b, pb, pn, work.coo) for b, (pb, pn) in zip(work.batches, parts)]
        config["parallelism"] = f"sharded over {world} rank(s): time-mode slabs, rep rho on rank rho mod {world}"
        config["slab"] = [k0b, k0n]
    else:
        h = init_single(L, work, w, opts, config)
    if world > 1 and not sharded:
        config["parallelism"] = f"{world} independent replicas"
    L.sambaten_checkpoint(h)
    dbatches = [work.tensor(L, b, device=True) for b in local_batches]
    hbatches = [work.tensor(L, b, device=False, pin=True) for b in local_batches]
    out_A = torch.empty((w.I, w.R), dtype=torch.float32).pin_memory()
    out_B = torch.empty((w.J, w.R), dtype=torch.float32).pin_memory()
    out_C = torch.empty((w.K, w.R), dtype=torch.float32).pin_memory()
    out_l = torch.empty((w.R,), dtype=torch.float32).pin_memory()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nb = work.nb
    state = {"i": 0}

    def step(host=False):
        i = state["i"]
        state["i"] += 1
        if i % nb == 0 and i > 0:
            L.sambaten_restore(h)
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        with torch.cuda.stream(stream):
            ev0.record(stream)
            if host:
                info = L.sambaten_update(h, hbatches[i % nb], out_A, out_B, out_C, out_l)
            else:
                info = L.sambaten_update(h, dbatches[i % nb])
            ev1.record(stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1), info, work.entries[i % nb], i % nb

    # priming (untimed, before the W warm-up steps): one pass over every batch through both
    # entry points, so first-use costs (lazy kernel loading, per-shape ALS plans, workspace
    # growth as K grows) are paid before timing; then back to the K0 checkpoint
    for host in (False, True):
        for i in range(nb):
            with torch.cuda.stream(stream):
                L.sambaten_update(h, hbatches[i] if host else dbatches[i],
                                  *((out_A, out_B, out_C, out_l) if host else ()))
        L.sambaten_restore(h)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        step()
    clk = ClockSampler(local)
    clk.start()
    times, infos, ents, kts = [], [], [], []
    prof_step = os.environ.get("SBT_PROFILE_STEP")   # ncu --profile-from-start off: one timed step
    for si in range(args.steps):
        if prof_step is not None and si == int(prof_step):
            torch.cuda.cudart().cudaProfilerStart()
        ms, info, ne, bi = step()
        if prof_step is not None and si == int(prof_step):
            torch.cuda.cudart().cudaProfilerStop()
        times.append(ms)
        infos.append(info.as_dict())
        ents.append(ne)
    clocks = clk.stop()
    e2e_times, e2e_ents, e2e_in = [], [], []
    if not args.no_e2e:
        state["i"] = 0
        L.sambaten_restore(h)
        for _ in range(args.warmup):
            step(host=True)
        e2e_infos = []
        for _ in range(args.steps):
            ms, einfo, ne, bi = step(host=True)
            e2e_infos.append(einfo.as_dict())
            e2e_times.append(ms)
            e2e_ents.append(ne)
            lb = local_batches[bi]
            e2e_in.append((int(lb.nnz) * 16 if work.coo else int(lb.nbytes)) if sharded else work.bytes_in(bi))
    tot = sum(times) / 1000.0
    e2e_tot = sum(e2e_times) / 1000.0 if e2e_times else None
    if world > 1:
        t = torch.tensor([tot, e2e_tot or 0.0], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot, e2e_tot = float(t[0]), (float(t[1]) if e2e_times else None)
    reps = 1 if sharded else world      # replicas each ingest the whole batch
    value = reps * sum(ents) / tot

    peaks, peak_kind = measured_peaks()
    kern = kernel_rooflines(w, work, infos, peaks, peak_kind, world if sharded else 1,
                            ([k0n + sum(parts[j][1] for j in range((i % nb) + 1))
                              for i in range(args.warmup, args.warmup + args.steps)] if sharded else None),
                            args)
    dominant = max(kern, key=lambda k: kern[k]["ms_per_launch"] if kern[k].get("frac") is not None else -1)
    step_share = {f"a{k}": statistics.mean(inf["step_ms"][k] for inf in infos) for k in range(8)}
    line = {
        "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * tot / args.steps,
        "ms_per_step_min_max": [min(times), max(times)], "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded numpy generators; DESIGN.md 'Synthetic inputs')",
        "config": config,
        "roofline": dict(kern[dominant], step=dominant),
        "kernels": kern,
        "step_ms": step_share,
        "gpu_launches": int(sum(inf["kernel_launches"] for inf in infos)),
        "clocks": clocks,
        "fit_full_last": infos[-1]["fit_full"] if infos[-1]["fit_full"] != -1.0 else infos[-1]["fit_full_prev"],
        "fit_full_is_lag1": infos[-1]["fit_full"] == -1.0 and infos[-1]["fit_full_prev"] != -1.0,
        "fit_path_last": {0: "none", 1: "separate pass", 2: "lag-1 in a1", 3: "incremental",
                          4: "incremental plan -> full pass"}.get(infos[-1].get("fit_path", 0)),
        "fit_summary_last": infos[-1]["fit_summary"],
        "reps_rejected_last": bin(infos[-1]["reps_rejected_mask"]).count("1"),
    }
    if e2e_tot:
        hb = int(statistics.mean(e2e_in))
        db = 4 * (w.I + w.J + w.K + 1) * w.R
        line["e2e"] = {"value": reps * sum(e2e_ents) / e2e_tot, "unit": unit,
                       "h2d_bytes_per_step": hb, "d2h_bytes_per_step": db,
                       "ms_per_step": 1000.0 * e2e_tot / len(e2e_times),
                       "step_ms": {f"a{k}": statistics.mean(inf["step_ms"][k] for inf in e2e_infos)
                                   for k in range(8)}}
    if not args.no_recompute and not work.coo:
        # the paper's evaluation: CP_ALS recomputed on the current tensor (the
        # baseline arm; P:441 tol 1e-5, capped iterations) and Relative Fitness of the committed
        # model against it; device time of the recompute next to the update's
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        rf, es, eb = L.sambaten_relative_fitness(h, args.recompute_iters, 1e-5)
        e1.record(stream)
        torch.cuda.synchronize()
        t_rc = e0.elapsed_time(e1)
        line["relative_fitness"] = {
            "value": rf, "relerr_sambaten": es, "relerr_cp_als": eb, "cp_als_max_iters": args.recompute_iters,
            "cp_als_tol": 1e-5, "recompute_plus_fit_ms": t_rc,
            "update_ms": 1000.0 * tot / args.steps,
            "speedup_vs_recompute": t_rc / (1000.0 * tot / args.steps),
            "note": "P:417-421 Relative Fitness = ||X - X_SamBaTen|| / ||X - X_CP_ALS||; CP_ALS = full CP-ALS of "
                    "the current tensor from the R35 Philox point (sambaten_recompute; SURVEY 8(f) NEXT #3)"}
    line["als_iters_per_rep"] = statistics.mean(inf["als_iters_sum"] for inf in infos) / (w.r / (world if sharded else 1))
    line["als_plan_last"] = infos[-1]["als_plan"]
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if device_gen:
            tot_s, parts, desc = oracle_sampled_update(w, warm, line["als_iters_per_rep"])
            line["cpu_baseline"] = {"value": w.I * w.J * w.batch / tot_s, "unit": unit, "cores": threads_used(),
                                    "kind": "oracle", "sample": desc,
                                    "seconds_per_update_estimated": tot_s,
                                    "step_seconds": {k: round(v, 3) for k, v in parts.items()}}
        elif work.model is not None:
            v, dt, nbt = cpu_baseline_run(work, work.model, tau, warm)
            line["cpu_baseline"] = {"value": v, "unit": unit, "cores": threads_used(), "kind": "oracle",
                                    "sample": f"{nbt} consecutive oracle updates of {w.name} from the K0 state, {dt:.1f} s"}
    if world == 1 and not sharded and not args.no_variant:
        # variants of the same workload: a fresh handle with one option changed,
        # primed, W warm-up and K (GetRank: <= 5) timed steps exactly as above
        def run_variant(nsteps, **changes):
            nonlocal h
            L.sambaten_destroy(h)
            saved = {k: getattr(opts, k) for k in changes}
            for k, v in changes.items():
                setattr(opts, k, v)
            h = init_single(L, work, w, opts, config)
            L.sambaten_checkpoint(h)
            for i in range(nb):
                with torch.cuda.stream(stream):
                    L.sambaten_update(h, dbatches[i])
            L.sambaten_restore(h)
            state["i"] = 0
            for _ in range(args.warmup):
                step()
            vt, vi, ve = [], [], []
            for _ in range(nsteps):
                ms, info, ne, bi = step()
                vt.append(ms)
                vi.append(info.as_dict())
                ve.append(ne)
            for k, v in saved.items():
                setattr(opts, k, v)
            kv = kernel_rooflines(w, work, vi, peaks, peak_kind, 1, None, args)
            return {"value": sum(ve) / (sum(vt) / 1000.0), "unit": unit, "ms_per_step": statistics.mean(vt),
                    "steps": len(vt), "kernels": kv,
                    "fit_full_last": vi[-1]["fit_full"] if vi[-1]["fit_full"] != -1.0 else vi[-1]["fit_full_prev"],
                    "reps_rejected_last": bin(vi[-1]["reps_rejected_mask"]).count("1"),
                    "step_ms": {f"a{k}": statistics.mean(inf["step_ms"][k] for inf in vi) for k in range(8)},
                    "als_iters_mean": statistics.mean(inf["als_iters_sum"] / w.r for inf in vi),
                    "rep_rank_last": vi[-1]["rep_rank"][:w.r]}
        line["variants"] = {"incremental_marginals": dict(
            run_variant(args.steps, incremental_marginals=1),
            note="opts.incremental_marginals=1: a1 adds the batch's contribution to the committed int64 "
                 "marginals (bit-identical to the full pass; tests/test_gpu_incremental.py)")}
        if not work.coo:
            line["variants"]["pipelined"] = dict(
                run_variant(args.steps, pipelined=1),
                note="opts.pipelined=1 (SURVEY 8(f) NEXT #4, R36; P:173): samples from the marginals the previous "
                     "update committed, so a1 runs on a side stream overlapped with a2..a7; "
                     "tests/test_gpu_update.py::test_pipelined_parity")
            line["variants"]["pipelined_incremental"] = dict(
                run_variant(args.steps, pipelined=1, incremental_marginals=1),
                note="pipelined + incremental marginals: no pass over the whole tensor (the batch's slices, the "
                     "summaries and the incremental fit only)")
        if (device_gen or w.name == "C5") and warm:
            v = run_variant(args.steps, warm_start=0, accept_tau=0.0)
            v["roofline_a4"] = v.pop("kernels")["a4"]
            line["variants"]["cold_start_paper_literal"] = dict(
                v, note="cold summary ALS from the Philox point (P:213, R10), 30 iterations, paper-literal "
                        "merge tau = 0 (the r01 headline setting): the summaries do not converge and the "
                        "model decays (fit_full_last); a4 roofline of the cold 30-iteration run")
        if not work.coo and not device_gen:
            line["variants"]["warm_start"] = dict(
                run_variant(args.steps, warm_start=1),
                note="opts.warm_start=1 (SURVEY 8(f) NEXT #4, R34): summary ALS from the model's rows, "
                     "the config's tolerance; tests/test_gpu_update.py::test_warm_start_*")
            line["variants"]["getrank_in_update"] = dict(
                run_variant(min(args.steps, 5), getrank=1),
                note="opts.getrank=1 (P:266, Alg. 2; R33): a4 includes GetRank over ranks 1..R on every summary")
        for vv in line["variants"].values():
            vv.pop("kernels", None)
    L.sambaten_destroy(h)
    if rank == 0 and not work.coo and not args.no_getrank:
        line["getrank"] = getrank_timing(L, w, stream)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
