# spectra round-2 follow-up: register-paired R2C / C2R unpacking and the chunked rows + stage-1
# interleave (L2-resident stage 1). Parity on the default library, then A/B timings of the variants.
set -x
python -m pytest tests/test_gpu_spectra.py -q -x > gpurun_out/pytest_sp_u.log 2>&1
tail -3 gpurun_out/pytest_sp_u.log
for rep in 1 2; do
for v in base p1 pc1 c2 default c8; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_sp_$v.so
  echo "{\"lib\": \"$v\"}" >> gpurun_out/spectra_u.jsonl
  LORENZ_LIB=$lib timeout 300 python tools/spectra.py --sizes 2048 4096 --reps 20 --oracle-side 0 --fig 0 >> gpurun_out/spectra_u.jsonl 2>&1
done
done
for v in base default; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_sp_$v.so
  LORENZ_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/spectra_launches_u_$v.csv python tools/spectra.py --sizes 4096 --reps 1 --oracle-side 0 --fig 0 > gpurun_out/ncu_u_$v.log 2>&1
done
echo done
