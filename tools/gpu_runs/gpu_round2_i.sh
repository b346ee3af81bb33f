set -x
for v in default uni uniimm imm; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_$v.so
  LORENZ_LIB=$lib python tools/tune.py --tag $v --integrator rk4 --kib 65536 131072 1048576 >> gpurun_out/tune_var.jsonl 2>&1
  LORENZ_LIB=$lib python tools/tune.py --tag $v --integrator rk4fma --kib 65536 262144 >> gpurun_out/tune_var.jsonl 2>&1
  LORENZ_LIB=$lib python tools/tune.py --tag $v --integrator euler --kib 65536 >> gpurun_out/tune_var.jsonl 2>&1
done
echo done
