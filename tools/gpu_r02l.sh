#!/bin/bash
# one-step ncu launch lists of the COO configs (SBT_PROFILE_STEP=0)
mkdir -p gpurun_out
FL="--steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
for c in "C3 cold" "C5 cold" "C5 warm"; do
  set -- $c
  SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_$1_$2.csv python bench.py --config $1 --als-init $2 $FL > gpurun_out/ncu_$1_$2.log 2>&1
  echo "$c rc=$?"
done
