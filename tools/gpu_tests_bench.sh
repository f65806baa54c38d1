# dev tool: full GPU test suite, C2 bench, C4 bench (logs in gpurun_out/)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t_pytest.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/t_bench_c2.log 2>&1
timeout 900 python bench.py --config C4 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/t_bench_c4.log 2>&1
tail -3 gpurun_out/t_pytest.log
python - <<'PY'
import json
for f in ("gpurun_out/t_bench_c2.log", "gpurun_out/t_bench_c4.log"):
    for ln in open(f):
        if ln.startswith("{"):
            d = json.loads(ln)
            print(f, round(d["ms_per_step"], 3), "value %.3g" % d["value"], "e2e %.3g" % d.get("e2e", {}).get("value", 0),
                  "frac %.3f" % d["roofline"]["frac"], {k: round(v, 3) for k, v in d["step_ms"].items()})
            v = d.get("variants", {}).get("incremental_marginals")
            if v: print("   incremental:", round(v["ms_per_step"], 3), "value %.3g" % v["value"], {k: round(x, 3) for k, x in v["step_ms"].items()})
PY
