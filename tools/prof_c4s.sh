# dev tool: ncu --set full captures of the streaming kernels and the cluster ALS at the C4
# row shape (C4s: 3000 x 3000 x 300), after a plain run of the same command
mkdir -p gpurun_out
CMD="python bench.py --config C4s --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/c4s_plain.log 2>&1 || exit 1
for KN in fit_stream marg_stream als_cluster; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KN -s 12 -c 1 \
      -o gpurun_out/prof_c4s_$KN -f $CMD > gpurun_out/ncu_c4s_$KN.log 2>&1
  echo "$KN rc=$?" >> gpurun_out/ncu_c4s_$KN.log
done
tail -1 gpurun_out/ncu_c4s_*.log
