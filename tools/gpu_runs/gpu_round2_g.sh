set -x
python -m pytest tests/test_gpu_spectra.py -q -x > gpurun_out/pytest_spectra_g.log 2>&1
python tools/spectra.py --sizes 1024 2048 4096 --reps 10 --oracle-side 0 --fig 256 > gpurun_out/spectra_r02g.jsonl 2>&1
python tools/spectra.py --sizes 4096 --reps 2 --oracle-side 0 --fig 256 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/spectra_launches_r02g.csv python tools/spectra.py --sizes 4096 --reps 1 --oracle-side 0 --fig 256 > gpurun_out/ncu_s1.log 2>&1
echo done
