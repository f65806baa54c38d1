# quick GPU iteration (dev tool): update parity tests, a short C2 bench, then ALS phase timing
# (the last step rebuilds the library with -DSBT_ALS_PHASES in the box's copy)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_update.py tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q_pytest.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/q_bench.log 2>&1
[ "${PHASES:-1}" = "1" ] && bash tools/probe_phases.sh ${CFG:-C2}
tail -3 gpurun_out/q_pytest.log
python - <<'PY'
import json
for ln in open("gpurun_out/q_bench.log"):
    if ln.startswith("{"):
        d = json.loads(ln); print("bench", round(d["ms_per_step"], 3), {k: round(v, 3) for k, v in d["step_ms"].items()})
PY
grep "als phases\|plan nI" gpurun_out/phases.log | head -4
