# spectra: 128-thread CTAs for the 2048-point row passes (one row per CTA) and for the four-step stage 2
# (8 columns per CTA) against the 256-thread default; parity of both variants, A/B timings.
set -x
timeout 600 python -m pytest tests/test_gpu_spectra.py -q -x > gpurun_out/pytest_sp_aa.log 2>&1
for v in sp_row128 sp_s2cta128; do
  LORENZ_LIB=tools/variants/liblorenz_$v.so timeout 600 python -m pytest tests/test_gpu_spectra.py -q -x > gpurun_out/pytest_sp_aa_$v.log 2>&1
done
tail -1 gpurun_out/pytest_sp_aa*.log
for rep in 1 2; do
for v in default sp_row128 sp_s2cta128; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_$v.so
  echo "{\"lib\": \"$v\"}" >> gpurun_out/spectra_aa.jsonl
  LORENZ_LIB=$lib timeout 300 python tools/spectra.py --sizes 1024 2048 4096 --reps 20 --oracle-side 0 --fig 0 >> gpurun_out/spectra_aa.jsonl 2>&1
done
done
echo done
