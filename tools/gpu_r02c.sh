#!/bin/bash
# fused a1 + lag-1 fit (32-bit path + REDUX row sums): tests, C4/C2 bench, ncu of the fused kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lagfit.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > gpurun_out/lag.log 2>&1; echo "lag rc=$?" >> gpurun_out/lag.log
timeout 1500 python bench.py --steps 6 --warmup 3 --no-getrank --no-variant > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?" >> gpurun_out/bench_c4.err
timeout 900 python bench.py --config C2 --steps 20 --warmup 5 --no-getrank --no-variant --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?" >> gpurun_out/bench_c2.err
CMD="python bench.py --config C4s --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-variant --no-getrank"
timeout 600 $CMD > gpurun_out/c4s_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:margfit -s 1 -c 1 -o gpurun_out/prof_margfit_c4s -f $CMD > gpurun_out/ncu_margfit.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_margfit.log
CMD2="python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-variant --no-getrank"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:margfit -s 3 -c 1 -o gpurun_out/prof_margfit_c2 -f $CMD2 > gpurun_out/ncu_margfit_c2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_margfit_c2.log
tail -5 gpurun_out/lag.log; tail -2 gpurun_out/bench_c4.err gpurun_out/bench_c2.err gpurun_out/ncu_margfit*.log
