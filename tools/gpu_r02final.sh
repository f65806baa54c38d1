#!/bin/bash
# Round-2 closing evidence: one-step launch lists (C4, C3, C5) and full captures of the
# radix scatter at C5 (per-element and tile-local).  Usage: bash tools/gpu_r02final.sh   (logs in gpurun_out/)
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
for C in C4 C3 C5; do
  timeout 600 $B --config $C > /dev/null 2>&1 && \
  SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launch_final_$C.csv $B --config $C > /dev/null 2>&1
  echo "$C rc=$?"
done
for V in global local; do
  if [ $V = local ]; then export SAMBATEN_RADIX_LOCAL=1; fi
  SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:radix_scatter -c 1 -o gpurun_out/prof_final_radix_$V -f $B --config C5 > gpurun_out/ncu_radix_$V.log 2>&1
  echo "radix $V full rc=$?"
done
unset SAMBATEN_RADIX_LOCAL
