#!/bin/bash
# Round-2 profiles: C4 launch list (the bench command), ncu --set full captures of the hot
# kernels on the C4 stand-ins (C4p: the grid a4 plan; C4s), COO tests + C5/C3 benches.
TAG=r02
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_coo.py tests/test_gpu_getrank.py -q -p no:cacheprovider > gpurun_out/coo.log 2>&1; echo "rc=$?" >> gpurun_out/coo.log
CMDP="python bench.py --config C4p --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-variant --no-getrank --no-recompute"
timeout 900 $CMDP > gpurun_out/plain_c4p.log 2>&1
# launch skips: priming (device update, host update: the latter runs the marginal kernel twice
# and the incremental fit's four gated fitrows launches per update) -> the warm-up update
for KS in als_cluster:2 marg_stream:3 gather_dense:2 fitrows:8; do
  KN=${KS%%:*}; SK=${KS##*:}
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KN -s $SK -c 1 \
      -o gpurun_out/prof_${TAG}_c4p_$KN -f $CMDP > gpurun_out/ncu_${TAG}_c4p_$KN.log 2>&1
  echo "$KN rc=$?" >> gpurun_out/ncu_${TAG}_c4p_$KN.log
done
tail -n 2 gpurun_out/coo.log gpurun_out/ncu_*c4p*.log
