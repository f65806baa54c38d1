"""Write the round's ncu summaries under profiles/ (run here after tools/profile_round.sh).

    python tools/make_profiles.py r01
"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import launches, full  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STEP = {"marg_stream": "a1", "gather_dense": "a3", "als_cluster": "a4", "fit_stream": "a7"}
CFG = {"c2": "C2", "c4s": "C4s"}


def dram_bytes(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    import csv, io
    rows = list(csv.reader(io.StringIO(r.stdout)))
    h, u, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(m)
        tot += float(v[i].replace(",", "")) * scale.get(u[i], 1)
    return tot


def main(tag):
    out = os.path.join(ROOT, "profiles")
    go = os.path.join(ROOT, "gpurun_out")
    with open(os.path.join(out, f"{tag}_launches.txt"), "w") as f:
        f.write(launches(os.path.join(go, f"launches_{tag}.csv")) + "\n")
    traffic = {}
    tp = os.path.join(out, "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp))
    for cfg in CFG:
        for k, step in STEP.items():
            rep = os.path.join(go, f"prof_{tag}_{cfg}_{k}.ncu-rep")
            if not os.path.exists(rep):
                continue
            with open(os.path.join(out, f"{tag}_full_{cfg}_{k}.txt"), "w") as f:
                f.write(full(rep) + "\n")
            traffic.setdefault(CFG[cfg], {})[step] = dram_bytes(rep)
    traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch from one ncu --set full "
                        f"capture ({tag}); keys: BASELINE config -> step")
    json.dump(traffic, open(tp, "w"), indent=1, sort_keys=True)
    b = os.path.join(go, f"bench_{tag}.json")
    if os.path.exists(b):
        line = [ln for ln in open(b) if ln.startswith("{")][-1]
        open(os.path.join(out, f"{tag}_bench_c2.json"), "w").write(line)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
