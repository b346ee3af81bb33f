set -x
python tools/spectra.py --sizes 4096 --reps 2 --oracle-side 0 --fig 256 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/spectra_launches_r02b.csv python tools/spectra.py --sizes 4096 --reps 2 --oracle-side 0 --fig 256 > gpurun_out/ncu_s1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cluster -c 2 -o gpurun_out/spectra_cluster_r02 python tools/spectra.py --sizes 4096 --reps 1 --oracle-side 0 --fig 256 > gpurun_out/ncu_s2.log 2>&1
echo done
