"""profiles/traffic.json from one-step ncu metric lists (dram__bytes_read.sum + dram__bytes_write.sum
per launch, single-pass metrics: no kernel replay).  Usage:
    python tools/traffic_json.py C4=gpurun_out/traffic_r02f_C4.csv C3=... [--tag r02f]
Per config and step: the DRAM bytes of the step's kernels in the one timed step (the bench's
`roofline.traffic` / `kernels.aN.traffic`)."""
import collections
import csv
import json
import os
import sys

STEP_OF = [("marg_stream", "a1"), ("margfit_stream", "a1"), ("marg_coo", "a1"), ("marg_rep_combine", "a1"),
           ("gather_dense", "a3"), ("gather_order", "a3"), ("coo_gather", "a3"),
           ("als_cluster", "a4"), ("coo_als_persist", "a4"), ("radix_", "a4"), ("permute", "a4"),
           ("fitcols", "a7"), ("fitrows", "a7"), ("fitinc", "a7"), ("coo_fitrows", "a7"), ("fit_stream", "a7")]


def parse(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    ui = h.index("Metric Unit")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024.0, "MB": 1024.0 ** 2,
             "GB": 1024.0 ** 3}
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        per[r[ii]][r[mi]] = v * scale.get(r[ui], 1.0)
        names[r[ii]] = r[ki]
    out = collections.defaultdict(float)
    for lid, m in per.items():
        name = names[lid]
        step = next((s for k, s in STEP_OF if k in name), None)
        if step is None:
            continue
        rd = m.get("dram__bytes_read.sum", 0.0)
        wr = m.get("dram__bytes_write.sum", 0.0)
        out[step] += rd + wr
    return dict(out)


def main():
    path = os.path.join(os.path.dirname(__file__), "..", "profiles", "traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    tag = "r02f"
    for a in sys.argv[1:]:
        if a.startswith("--tag="):
            tag = a.split("=", 1)[1]
            continue
        cfg, f = a.split("=", 1)
        data[cfg] = parse(f)
    data["_note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum of each step's kernels in one timed step, "
                     f"from a single-pass ncu metric list ({tag}; tools/gpu_r02f2.sh, tools/traffic_json.py)")
    json.dump(data, open(path, "w"), indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
