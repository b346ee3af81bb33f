set -x
python -m pytest tests/test_gpu_spectra.py -q -x > gpurun_out/pytest_spectra.log 2>&1
python tools/spectra.py --sizes 1024 2048 4096 --reps 10 --oracle-side 0 --fig 256 > gpurun_out/spectra_r02.jsonl 2>&1
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > gpurun_out/pytest_gpu_r02e.log 2>&1
for v in default nopin pinrk4; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_$v.so
  LORENZ_LIB=$lib python tools/tune.py --tag $v --integrator rk4 --kib 65536 1048576 >> gpurun_out/tune_pin.jsonl 2>&1
  LORENZ_LIB=$lib python tools/tune.py --tag $v --integrator euler --kib 65536 1048576 >> gpurun_out/tune_pin.jsonl 2>&1
  LORENZ_LIB=$lib python tools/tune.py --tag $v --integrator euler --kib 65536 1048576 --sched seg >> gpurun_out/tune_pin.jsonl 2>&1
done
python tools/tune.py --tag fma-seg --integrator rk4fma --kib 65536 131072 262144 524288 1048576 --sched seg >> gpurun_out/tune_pin.jsonl 2>&1
python tools/tune.py --tag fma-wave --integrator rk4fma --kib 131072 262144 524288 1048576 --sched wave >> gpurun_out/tune_pin.jsonl 2>&1
echo done
