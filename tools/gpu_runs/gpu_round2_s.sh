set -x
LORENZ_LIB=tools/variants/liblorenz_e8.so python -m pytest tests/test_gpu_spectra.py -q -x > gpurun_out/pytest_e8.log 2>&1
for v in default e8 default e8; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_$v.so
  echo "{\"lib\": \"$v\"}" >> gpurun_out/spectra_e8.jsonl
  LORENZ_LIB=$lib python tools/spectra.py --sizes 2048 4096 --reps 10 --oracle-side 0 --fig 256 >> gpurun_out/spectra_e8.jsonl 2>&1
done
echo done
