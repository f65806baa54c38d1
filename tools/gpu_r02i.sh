#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python bench.py --config C5 --steps 4 --warmup 2 --no-getrank --no-cpu-baseline --no-variant --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?" >> gpurun_out/bench_c5.err
timeout 900 python bench.py --config C3 --steps 8 --warmup 3 --no-getrank --no-cpu-baseline --no-variant --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "rc=$?" >> gpurun_out/bench_c3.err
CMD="python bench.py --config C5 --steps 1 --warmup 1 --no-getrank --no-cpu-baseline --no-variant --no-e2e"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/ncu_c5.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_c5.log
tail -n 2 gpurun_out/bench_c5.err gpurun_out/bench_c3.err gpurun_out/ncu_c5.log
