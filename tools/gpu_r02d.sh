#!/bin/bash
# round-2 (re-entry) evidence: full GPU suite, smoke, the default bench line (C4), C2 / C3 / C5,
# the reference arm, one-step launch lists (C4, C3, C5) and an ncu capture of the persistent COO ALS
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f_smoke.log
timeout 1500 python bench.py > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err
for c in C2 C3 C5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/f_bench_$c.json 2> gpurun_out/f_bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f_ref_c4.json 2> gpurun_out/f_ref_c4.err
FL="--steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
for C in C4 C3 C5; do
SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r02d_$C.csv python bench.py --config $C $FL > /dev/null 2>&1
done
SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --set full --import-source on -k regex:"coo_als_persist" -c 1 \
  -o gpurun_out/prof_r02d_c3_coo_als -f python bench.py --config C3 $FL > gpurun_out/ncu_r02d.log 2>&1
tail -n 3 gpurun_out/f_pytest.log gpurun_out/f_smoke.log
for f in gpurun_out/f_bench_*.json gpurun_out/f_ref_c4.json; do python -c "
import json,sys
d=json.loads([l for l in open('$f') if l.startswith('{')][-1])
print('$f', d.get('ms_per_step'), d.get('value'), d.get('e2e',{}).get('value'), (d.get('roofline') or {}).get('frac'), d.get('fit_full_last'), d.get('step_ms'))" 2>&1 | tail -1; done
