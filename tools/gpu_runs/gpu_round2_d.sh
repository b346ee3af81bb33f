set -x
for v in default fmanopin; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_$v.so
  LORENZ_LIB=$lib python tools/tune.py --tag $v --integrator rk4fma --kib 65536 100000 131072 262144 --sched seg >> gpurun_out/tune_fma2.jsonl 2>&1
  LORENZ_LIB=$lib python tools/tune.py --tag $v --integrator rk4 --kib 65536 1048576 >> gpurun_out/tune_fma2.jsonl 2>&1
done
python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_r02d.json 2>&1
echo done
