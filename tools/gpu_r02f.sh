#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fitinc.py tests/test_gpu_recompute.py tests/test_gpu_dist.py -q -p no:cacheprovider > gpurun_out/fitinc.log 2>&1; echo "rc=$?" >> gpurun_out/fitinc.log
timeout 1500 python bench.py --steps 6 --warmup 3 --no-getrank --no-cpu-baseline --no-variant > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?" >> gpurun_out/bench_c4.err
timeout 900 python bench.py --config C2 --steps 20 --warmup 5 --no-getrank --no-variant --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?" >> gpurun_out/bench_c2.err
tail -n 3 gpurun_out/fitinc.log
