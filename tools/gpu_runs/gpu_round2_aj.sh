# spectra: the TMA column pass's second transform reads its real input (|X|^2, 0) as real (8-byte loads, zero
# imaginary parts as constants) against the previous library; parity, A/B timings, launch list
set -x
timeout 600 python -m pytest tests/test_gpu_spectra.py -q -x > gpurun_out/pytest_sp_aj.log 2>&1
tail -1 gpurun_out/pytest_sp_aj.log
for rep in 1 2 3; do
for v in prev default; do
  lib=""; [ $v != default ] && lib=tools/variants/liblorenz_$v.so
  echo "{\"lib\": \"$v\"}" >> gpurun_out/spectra_aj.jsonl
  LORENZ_LIB=$lib timeout 300 python tools/spectra.py --sizes 2048 4096 --reps 20 --oracle-side 0 --fig 0 >> gpurun_out/spectra_aj.jsonl 2>&1
done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/spectra_launches_aj.csv python tools/spectra.py --sizes 4096 --reps 1 --oracle-side 0 --fig 0 > gpurun_out/ncu_aj.log 2>&1
echo done
