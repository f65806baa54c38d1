# Round profile (dev tool): C2 bench line, then the ncu launch list of the same command and one
# --set full capture per hot kernel (C2 and the C4-row-shape stand-in C4s).  Usage:
#   bash tools/profile_round.sh TAG      -> gpurun_out/{bench,launches,prof}_TAG*
TAG=${1:-r01}
mkdir -p gpurun_out
if [ -n "$ONLY_MARG" ]; then   # re-capture only the marginal kernel
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-variant --no-getrank"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:marg_stream -s 16 -c 1 \
      -o gpurun_out/prof_${TAG}_c2_marg_stream -f $CMD > gpurun_out/ncu_${TAG}_c2_marg_stream.log 2>&1
  CMD4="python bench.py --config C4s --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-variant --no-getrank"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:marg_stream -s 18 -c 1 \
      -o gpurun_out/prof_${TAG}_c4s_marg_stream -f $CMD4 > gpurun_out/ncu_${TAG}_c4s_marg_stream.log 2>&1
  exit 0
fi
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err || exit 1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-variant --no-getrank"
timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
# launch skips: past the priming pass (device + host batches; a host batch launches the marginal
# kernel twice: old slices overlapped with its copy, then the batch) onto a device-path update
for KN in als_cluster marg_stream fit_stream gather_dense; do
  SK=12; [ $KN = marg_stream ] && SK=16
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KN -s $SK -c 1 \
      -o gpurun_out/prof_${TAG}_c2_$KN -f $CMD > gpurun_out/ncu_${TAG}_c2_$KN.log 2>&1
done
CMD4="python bench.py --config C4s --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-variant --no-getrank"
timeout 600 $CMD4 > gpurun_out/plain_${TAG}_c4s.log 2>&1 || exit 1
for KN in als_cluster marg_stream fit_stream gather_dense; do
  SK=12; [ $KN = marg_stream ] && SK=18
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KN -s $SK -c 1 \
      -o gpurun_out/prof_${TAG}_c4s_$KN -f $CMD4 > gpurun_out/ncu_${TAG}_c4s_$KN.log 2>&1
done
ls gpurun_out/prof_${TAG}_* | wc -l
