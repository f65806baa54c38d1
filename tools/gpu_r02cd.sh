#!/bin/bash
# pair MTTKRP (half-warp short pieces): COO tests, C3 / C5 persistent vs per-mode pipeline
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "coo" > gpurun_out/pytest_coo.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_coo.log
tail -2 gpurun_out/pytest_coo.log
FL="--steps 8 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
for C in C3 C5; do
  timeout 600 python bench.py --config $C $FL > gpurun_out/bench_p_$C.json 2> gpurun_out/bench_p_$C.err
  SAMBATEN_COO_ALS_BPS=1 timeout 600 python bench.py --config $C $FL > gpurun_out/bench_p1_$C.json 2> gpurun_out/bench_p1_$C.err
  SAMBATEN_COO_ALS_MULTI=1 timeout 600 python bench.py --config $C $FL > gpurun_out/bench_m_$C.json 2> gpurun_out/bench_m_$C.err
  for V in p p1 m; do python -c "
import json;d=json.load(open('gpurun_out/bench_${V}_$C.json'))
print('$V $C', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['step_ms'].items()}, 'fit', d.get('fit_full_last'), 'it', d.get('als_iters_per_rep'))" 2>&1 | tail -1; done
done
FL1="--steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
SAMBATEN_COO_ALS_MULTI=1 SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r02cd_C3m.csv python bench.py --config C3 $FL1 > /dev/null 2>&1
echo "launches rc=$?"
