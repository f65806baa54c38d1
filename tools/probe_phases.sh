# ALS phase timing (clock64 per phase, rank 0 of rep 0) on C2; rebuilds the library with
# -DSBT_ALS_PHASES in the box's copy of the repo (dev tool)
mkdir -p gpurun_out
SBT_EXTRA_FLAGS=-DSBT_ALS_PHASES bash tools/build.sh > gpurun_out/phases_build.log 2>&1
SAMBATEN_DEBUG=1 python tools/probe_update.py ${1:-C2} 8 > gpurun_out/phases.log 2>&1
