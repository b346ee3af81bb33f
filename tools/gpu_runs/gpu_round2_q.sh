set -x
for rep in 1 2; do
for v in default pf; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_$v.so
  LORENZ_LIB=$lib python tools/tune.py --tag $v --integrator rk4 --kib 65536 131072 1048576 >> gpurun_out/tune_pf.jsonl 2>&1
  LORENZ_LIB=$lib python tools/tune.py --tag $v --integrator euler --kib 65536 1048576 >> gpurun_out/tune_pf.jsonl 2>&1
  LORENZ_LIB=$lib python tools/tune.py --tag $v --integrator rk4 --kib 37888 >> gpurun_out/tune_pf.jsonl 2>&1
done
done
for v in default pf; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_$v.so
  echo "{\"lib\": \"$v\"}" >> gpurun_out/e2e_pf.jsonl
  LORENZ_LIB=$lib python tools/e2e_probe.py --mib 64 128 --staged-chunks 1 >> gpurun_out/e2e_pf.jsonl 2>&1
done
echo done
