# spectra: the TMA column pass for H = 2048 too (128-thread CTAs) and the unrolled byte sum;
# parity, A/B timings against LZ_COL_TMA=0, launch list, full captures.
set -x
timeout 600 python -m pytest tests/test_gpu_spectra.py -q -x > gpurun_out/pytest_sp_z.log 2>&1
tail -3 gpurun_out/pytest_sp_z.log
grep -q " passed" gpurun_out/pytest_sp_z.log && ! grep -q "failed\|error" gpurun_out/pytest_sp_z.log || exit 1
for rep in 1 2; do
for v in base nocol default; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_sp_$v.so
  echo "{\"lib\": \"$v\"}" >> gpurun_out/spectra_z.jsonl
  LORENZ_LIB=$lib timeout 300 python tools/spectra.py --sizes 1024 2048 4096 --reps 20 --oracle-side 0 --fig 0 >> gpurun_out/spectra_z.jsonl 2>&1
done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/spectra_launches_z.csv python tools/spectra.py --sizes 2048 4096 --reps 1 --oracle-side 0 --fig 0 > gpurun_out/ncu_z.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fft_col_tma|byte_sum" -c 2 -o gpurun_out/spectra_full_z \
    python tools/spectra.py --sizes 4096 --reps 1 --oracle-side 0 --fig 0 > gpurun_out/ncu_z_full.log 2>&1
echo done
