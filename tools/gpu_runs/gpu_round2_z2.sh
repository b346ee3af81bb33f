# spectra: byte sum with one atomic per CTA, col0 unpacking + flatness in one kernel;
# parity, timings against the round-start library, launch list.
set -x
timeout 600 python -m pytest tests/test_gpu_spectra.py -q -x > gpurun_out/pytest_sp_z2.log 2>&1
tail -3 gpurun_out/pytest_sp_z2.log
grep -q " passed" gpurun_out/pytest_sp_z2.log && ! grep -q "failed\|error" gpurun_out/pytest_sp_z2.log || exit 1
for rep in 1 2; do
for v in base default; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_sp_$v.so
  echo "{\"lib\": \"$v\"}" >> gpurun_out/spectra_z2.jsonl
  LORENZ_LIB=$lib timeout 300 python tools/spectra.py --sizes 1024 2048 4096 --reps 20 --oracle-side 0 --fig 0 >> gpurun_out/spectra_z2.jsonl 2>&1
done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/spectra_launches_z2.csv python tools/spectra.py --sizes 2048 4096 --reps 1 --oracle-side 0 --fig 0 > gpurun_out/ncu_z2.log 2>&1
timeout 600 python tools/spectra.py --sizes 256 1024 2048 4096 --reps 20 > gpurun_out/spectra_final_z2.jsonl 2>&1
echo done
