set -x
for rep in 1 2; do
for v in default consth; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_$v.so
  LORENZ_LIB=$lib python tools/tune.py --tag $v --integrator rk4 --kib 65536 131072 1048576 >> gpurun_out/tune_consth.jsonl 2>&1
  LORENZ_LIB=$lib python tools/tune.py --tag $v --integrator euler --kib 65536 1048576 >> gpurun_out/tune_consth.jsonl 2>&1
done
done
echo done
