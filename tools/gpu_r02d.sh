#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lagfit.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -p no:cacheprovider -x > gpurun_out/lag.log 2>&1; echo "lag rc=$?" >> gpurun_out/lag.log
timeout 1500 python bench.py --steps 6 --warmup 3 --no-getrank --no-variant --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?" >> gpurun_out/bench_c4.err
timeout 900 python bench.py --config C2 --steps 20 --warmup 5 --no-getrank --no-variant --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?" >> gpurun_out/bench_c2.err
tail -3 gpurun_out/lag.log
