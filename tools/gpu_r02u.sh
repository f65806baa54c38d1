#!/bin/bash
mkdir -p gpurun_out
SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_C5w.csv python bench.py --config C5 --steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > /dev/null 2>&1
echo rc=$?
