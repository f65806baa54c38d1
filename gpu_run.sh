#!/bin/bash
# Round-trip script for gpurun: tests, smoke, bench, ncu launch list + one full capture.
# Usage: bash gpu_run.sh [tag]     (logs in gpurun_out/)
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc >> gpurun_out/smi.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ "${EXTRA:-1}" = "1" ]; then
  timeout 600 python bench.py --sharded --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sharded.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sharded.log
  timeout 900 python bench.py --config C3 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
fi
if [ "${NCU:-1}" = "1" ]; then
  CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
  timeout 600 $CMD > gpurun_out/ncu_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch.log 2>&1
  echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
  for KN in ${NCU_KERNEL//,/ }; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KN -s ${NCU_SKIP:-2} -c ${NCU_COUNT:-1} \
        -o gpurun_out/prof_${TAG}_${KN} -f $CMD > gpurun_out/ncu_full_${KN}.log 2>&1
    echo "ncu full $KN rc=$?" >> gpurun_out/ncu_full_${KN}.log
  done
fi
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log; tail -3 gpurun_out/bench*.log; tail -2 gpurun_out/ncu_*.log
