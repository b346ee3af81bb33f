# spectra: register-paired C2R input + the TMA column pass of the autocorrelation (4096 rows).
# Parity first (bounded by timeout: an mbarrier that never completes would hang), then A/B timings,
# the launch list and one full capture of the TMA kernel.
set -x
timeout 600 python -m pytest tests/test_gpu_spectra.py -q -x > gpurun_out/pytest_sp_v.log 2>&1
tail -3 gpurun_out/pytest_sp_v.log
grep -q " passed" gpurun_out/pytest_sp_v.log && ! grep -q "failed\|error" gpurun_out/pytest_sp_v.log || exit 1
for rep in 1 2; do
for v in base notma default; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_sp_$v.so
  echo "{\"lib\": \"$v\"}" >> gpurun_out/spectra_v.jsonl
  LORENZ_LIB=$lib timeout 300 python tools/spectra.py --sizes 2048 4096 --reps 20 --oracle-side 0 --fig 0 >> gpurun_out/spectra_v.jsonl 2>&1
done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/spectra_launches_v.csv python tools/spectra.py --sizes 4096 --reps 1 --oracle-side 0 --fig 0 > gpurun_out/ncu_v.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_col_tma -c 1 -o gpurun_out/spectra_tma_v \
    python tools/spectra.py --sizes 4096 --reps 1 --oracle-side 0 --fig 0 > gpurun_out/ncu_v_full.log 2>&1
echo done
