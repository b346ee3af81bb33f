set -x
python -m pytest tests/test_gpu_spectra.py -q > gpurun_out/pytest_spectra_h.log 2>&1
python tools/spectra.py --sizes 1024 2048 4096 --reps 10 --oracle-side 128 --fig 1024 > gpurun_out/spectra_r02h.jsonl 2>&1
python tools/spectra.py --sizes 4096 --reps 2 --oracle-side 0 --fig 256 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/spectra_launches_r02h.csv python tools/spectra.py --sizes 4096 --reps 1 --oracle-side 0 --fig 256 > gpurun_out/ncu_s1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fft_col_stage1|fft_pass_kernel" -c 6 -o gpurun_out/spectra_full_r02h python tools/spectra.py --sizes 4096 --reps 1 --oracle-side 0 --fig 256 > gpurun_out/ncu_s2.log 2>&1
echo done
