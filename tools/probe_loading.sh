mkdir -p gpurun_out
for cfg in C2 C3; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_${cfg}_w3.log 2>&1
  CUDA_MODULE_LOADING=EAGER timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_${cfg}_eager.log 2>&1
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/p_${cfg}_w10.log 2>&1
done
