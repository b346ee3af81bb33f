# spectra: the adopted 128-thread CTAs (2048-point rows, stage 2) as the default; parity, timings, launch list
set -x
timeout 600 python -m pytest tests/test_gpu_spectra.py -q -x > gpurun_out/pytest_sp_ab.log 2>&1
tail -1 gpurun_out/pytest_sp_ab.log
timeout 600 python tools/spectra.py --sizes 256 1024 2048 4096 --reps 20 > gpurun_out/spectra_final_ab.jsonl 2>&1
timeout 300 python tools/spectra.py --sizes 4096 --reps 20 --oracle-side 0 --fig 0 >> gpurun_out/spectra_final_ab.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/spectra_launches_ab.csv python tools/spectra.py --sizes 2048 4096 --reps 1 --oracle-side 0 --fig 0 > gpurun_out/ncu_ab.log 2>&1
echo done
