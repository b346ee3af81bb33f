# spectra: four-step stage 2 with 4 columns per 64-thread CTA (8 per SM) against 8 per 128-thread CTA;
# parity of the variant, A/B timings
set -x
LORENZ_LIB=tools/variants/liblorenz_sp_s2cta64.so timeout 600 python -m pytest tests/test_gpu_spectra.py -q -x > gpurun_out/pytest_sp_ak.log 2>&1
tail -1 gpurun_out/pytest_sp_ak.log
for rep in 1 2 3; do
for v in default sp_s2cta64; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_$v.so
  echo "{\"lib\": \"$v\"}" >> gpurun_out/spectra_ak.jsonl
  LORENZ_LIB=$lib timeout 300 python tools/spectra.py --sizes 4096 --reps 20 --oracle-side 0 --fig 0 >> gpurun_out/spectra_ak.jsonl 2>&1
done
done
echo done
