#!/bin/bash
# ALS phase counters at C4 (warm, grid plan): rebuild with -DSBT_ALS_PHASES in the box's copy
mkdir -p gpurun_out
SBT_EXTRA_FLAGS=-DSBT_ALS_PHASES bash tools/build.sh > gpurun_out/phases_build.log 2>&1
SAMBATEN_DEBUG=1 timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > gpurun_out/ph.json 2> gpurun_out/ph.err
grep "als phases" gpurun_out/ph.err | tail -3
