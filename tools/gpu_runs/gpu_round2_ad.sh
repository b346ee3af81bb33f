# spectra: 2048-point row passes and stage 2 compiled for 5 / 6 resident 128-thread CTAs per SM (register
# caps 102 / 85) against 4; parity of the variants, A/B timings.
set -x
for v in sp_m5 sp_m6; do
  LORENZ_LIB=tools/variants/liblorenz_$v.so timeout 600 python -m pytest tests/test_gpu_spectra.py -q -x > gpurun_out/pytest_sp_ad_$v.log 2>&1
done
tail -1 gpurun_out/pytest_sp_ad_*.log
for rep in 1 2; do
for v in default sp_m5 sp_m6; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_$v.so
  echo "{\"lib\": \"$v\"}" >> gpurun_out/spectra_ad.jsonl
  LORENZ_LIB=$lib timeout 300 python tools/spectra.py --sizes 4096 --reps 20 --oracle-side 0 --fig 0 >> gpurun_out/spectra_ad.jsonl 2>&1
done
done
echo done
