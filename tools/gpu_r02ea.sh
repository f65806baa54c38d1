#!/bin/bash
# payload-carrying COO sort: COO / getrank / dist GPU tests, C3 / C5 bench, C5 one-step launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "coo or getrank or dist or mttkrp" > gpurun_out/pytest_coo.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_coo.log
tail -2 gpurun_out/pytest_coo.log; grep -E '^E |FAILED' gpurun_out/pytest_coo.log | head
FL="--steps 8 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
for C in C3 C5; do
  timeout 600 python bench.py --config $C $FL > gpurun_out/bench_s_$C.json 2> gpurun_out/bench_s_$C.err
  python -c "
import json;d=json.load(open('gpurun_out/bench_s_$C.json'))
print('$C', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['step_ms'].items()}, 'fit', d.get('fit_full_last'))" 2>&1 | tail -1
done
FL1="--steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r02e_C5.csv python bench.py --config C5 $FL1 > /dev/null 2>&1
echo "launches rc=$?"
