#!/bin/bash
# Round-2 profiles: C4 launch list (the bench command), ncu --set full captures of the hot
# kernels on the C4 stand-ins (C4p: the grid a4 plan; C4s), COO tests + C5/C3 benches.
TAG=r02
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_coo.py -q -p no:cacheprovider > gpurun_out/coo.log 2>&1; echo "rc=$?" >> gpurun_out/coo.log
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-variant --no-getrank --no-recompute"
timeout 900 $CMD > gpurun_out/plain_c4.log 2>&1
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c4.csv $CMD > gpurun_out/ncu_launch_c4.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launch_c4.log
CMDP="python bench.py --config C4p --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-variant --no-getrank --no-recompute"
timeout 900 $CMDP > gpurun_out/plain_c4p.log 2>&1
for KN in als_cluster marg_stream gather_dense fitrows; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KN -s 6 -c 1 \
      -o gpurun_out/prof_${TAG}_c4p_$KN -f $CMDP > gpurun_out/ncu_${TAG}_c4p_$KN.log 2>&1
  echo "$KN rc=$?" >> gpurun_out/ncu_${TAG}_c4p_$KN.log
done
timeout 1500 python bench.py --config C5 --steps 4 --warmup 2 --no-getrank --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --config C3 --steps 8 --warmup 3 --no-getrank > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
tail -n 2 gpurun_out/coo.log gpurun_out/ncu_*c4p*.log
