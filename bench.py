"""bench.py -- SamBaTen per-batch incremental CP update on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]

A step is one whole update (a0..a7: ingest, marginals, sampling, gather, batched CP-ALS,
matching, merge, full fit) of one batch of the BASELINE.json workload (default configs[1] =
C2: 500^3 dense, R=10, K0=450, batches of 10 slices, s=5, r=8, 30 ALS iterations), with
synthetic planted data.  The metric is BASELINE.json's: new tensor entries ingested per
second per update.  Rank 0 prints one JSON line.

Timing: W untimed warm-up steps, then K steps, each bracketed by a barrier and a device
synchronisation and timed with CUDA events on the library's stream; L2 is flushed (a 512 MB
write) before every step; the stream cycles through the config's batches, restoring the
K0 checkpoint (untimed) after the last one.  Multi-GPU (torchrun): every rank runs its own
replica of the update (weak scaling, no data-path collective yet) and the
time is the max over ranks.
"""
import argparse
import json
import math
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
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C2")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""
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
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
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


def make_workload(w):
    from synth import planted_dense, split_dense
    T, truth = planted_dense(w.I, w.J, w.K, w.R, noise=w.noise, seed=w.seed)
    T0, batches = split_dense(T, w.K0, w.batch)
    model = [np.asarray(x, np.float32) for x in (truth[0], truth[1], truth[2], truth[3][:w.K0])]
    return T0, batches, model


def cpu_baseline_run(w, T0, batches, model, max_batches=None):
    """The oracle as it stands (oracle/), on this host's cores: the config's updates from the
    K0 state (bounded sample: the first `max_batches` batches)."""
    from oracle import sambaten as O
    cfg = O.Config(R=w.R, s=(w.s,) * 3, r=w.r, seed=w.seed, maxit=w.maxit, tol=w.tol)
    st = O.init_factors(T0, cfg, *model, w.I * w.J * w.K)
    nb = len(batches) if max_batches is None else min(max_batches, len(batches))
    t0 = time.perf_counter()
    entries = 0
    for b in batches[:nb]:
        O.update(st, b)
        entries += b.size
    dt = time.perf_counter() - t0
    return entries / dt, dt, nb


def threads_used():
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count()


def main():
    args = parse()
    from synth import CONFIGS
    w = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    metric = "new tensor entries ingested/sec per update"
    unit = "entries/s"
    config = {"workload": f"{w.name}: dense {w.I}x{w.J}x{w.K}, K0={w.K0}, batch={w.batch} slices, "
                          f"R={w.R}, s={w.s}, r={w.r}, ALS {w.maxit} it tol {w.tol}",
              "l2": "flushed (512 MB write) before every step", "init": "planted truth factors"}

    if args.impl == "reference":
        if rank != 0:
            return
        T0, batches, model = make_workload(w)
        times = []
        per = w.I * w.J * w.batch
        for i in range(args.warmup + args.steps):
            from oracle import sambaten as O
            cfg = O.Config(R=w.R, s=(w.s,) * 3, r=w.r, seed=w.seed, maxit=w.maxit, tol=w.tol)
            st = O.init_factors(T0, cfg, *model, w.I * w.J * w.K)
            t0 = time.perf_counter()
            O.update(st, batches[0])
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
        tot = sum(times)
        val = per * len(times) / tot
        cores = threads_used()
        line = {"impl": "reference", "metric": metric, "value": val, "unit": unit, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / len(times),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic planted (numpy, seed 0)", "config": config,
                "cpu_baseline": {"value": val, "unit": unit, "cores": cores, "kind": "oracle",
                                 "sample": f"each step = one full oracle update of batch 0 from the K0 state"},
                "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1709_00668_b200 import _lib as L

    T0, batches, model = make_workload(w)
    stream = torch.cuda.Stream()
    opts = L.default_opts(als_max_iters=w.maxit, als_tol=w.tol, capacity=w.K, full_fit=1,
                          stream=stream.cuda_stream)
    h = L.sambaten_init_factors(L.dense(torch.from_numpy(T0).cuda()), w.R, w.s, w.r, w.seed,
                                model[1], model[2], model[3], model[0], opts)
    L.sambaten_checkpoint(h)
    dbatches = [torch.from_numpy(b).cuda() for b in batches]
    hbatches = [torch.from_numpy(b).pin_memory() for b in batches]
    out_A = torch.empty((w.I, w.R), dtype=torch.float32).pin_memory()
    out_B = torch.empty((w.J, w.R), dtype=torch.float32).pin_memory()
    out_C = torch.empty((w.K, w.R), dtype=torch.float32).pin_memory()
    out_l = torch.empty((w.R,), dtype=torch.float32).pin_memory()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nb = len(batches)
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
                info = L.sambaten_update(h, L.dense(hbatches[i % nb]), out_A, out_B, out_C, out_l)
            else:
                info = L.sambaten_update(h, L.dense(dbatches[i % nb]))
            ev1.record(stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1), info

    for _ in range(args.warmup):
        step()
    clk = ClockSampler(local)
    clk.start()
    times, infos = [], []
    for _ in range(args.steps):
        ms, info = step()
        times.append(ms)
        infos.append(info.as_dict())
    clocks = clk.stop()
    e2e_times = []
    if not args.no_e2e:
        state["i"] = 0
        L.sambaten_restore(h)
        for _ in range(args.warmup):
            step(host=True)
        for _ in range(args.steps):
            ms, _ = step(host=True)
            e2e_times.append(ms)
    tot = sum(times) / 1000.0
    e2e_tot = sum(e2e_times) / 1000.0 if e2e_times else None
    if world > 1:
        t = torch.tensor([tot, e2e_tot or 0.0], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot, e2e_tot = float(t[0]), (float(t[1]) if e2e_times else None)
    per_step_entries = w.I * w.J * w.batch
    value = world * per_step_entries * args.steps / tot

    peaks, peak_kind = measured_peaks()
    # dominant HBM-bound kernel of the step: the marginal pass a1 (one read of the whole tensor)
    a1_ms = statistics.mean(inf["step_ms"][1] for inf in infos)
    Kavg = statistics.mean(inf["k_total"] for inf in infos)
    a1_bytes = 4.0 * w.I * w.J * Kavg + 8.0 * (w.I + w.J + Kavg)
    achieved = a1_bytes / (a1_ms / 1000.0) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(w.name, {}).get("marg_dense_kernel")
        except Exception:
            traffic = None
    step_share = {f"a{k}": statistics.mean(inf["step_ms"][k] for inf in infos) for k in range(8)}
    line = {
        "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * tot / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic planted rank-R + 1% Gaussian noise (numpy, seed 0)",
        "config": config,
        "roofline": {"kernel": "marg_dense_kernel (a1)", "bound": "hbm", "achieved": achieved,
                     "peak": peaks["hbm_gbs"], "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                     "bytes_per_launch": a1_bytes, "ms_per_launch": a1_ms},
        "step_ms": step_share,
        "gpu_launches": int(sum(inf["kernel_launches"] for inf in infos)),
        "clocks": clocks,
        "fit_full_last": infos[-1]["fit_full"],
        "reps_rejected_last": bin(infos[-1]["reps_rejected_mask"]).count("1"),
    }
    if e2e_tot:
        hb = 4 * w.I * w.J * w.batch
        db = 4 * (w.I + w.J + w.K + 1) * w.R
        line["e2e"] = {"value": world * per_step_entries * args.steps / e2e_tot, "unit": unit,
                       "h2d_bytes_per_step": hb, "d2h_bytes_per_step": db}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, nbt = cpu_baseline_run(w, T0, batches, model)
        line["cpu_baseline"] = {"value": v, "unit": unit, "cores": threads_used(), "kind": "oracle",
                                "sample": f"{nbt} oracle updates (all batches of {w.name}) from the K0 state, {dt:.1f} s"}
    L.sambaten_destroy(h)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
