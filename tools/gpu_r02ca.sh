#!/bin/bash
# one timed step's launch list for C3, C2, C5 (cold serialised ncu times; shares only)
TAG=r02ca
mkdir -p gpurun_out
FL="--steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
for C in C3 C2 C5; do
SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_$C.csv python bench.py --config $C $FL > gpurun_out/ncu_${TAG}_$C.log 2>&1
echo "$C launches rc=$?"
done
