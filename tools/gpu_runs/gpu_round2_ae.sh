# final library: one ncu --set full capture of the 4096^2 spectrum's row pass, stage 1, stage 2 and the
# autocorrelation's R2C rows, TMA column pass and C2R rows (the kernels profiles/spectra_final_r02.json summarises)
set -x
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fft_pass_kernel|fft_col" -c 6 -o gpurun_out/spectra_full_final \
    python tools/spectra.py --sizes 4096 --reps 1 --oracle-side 0 --fig 0 > gpurun_out/ncu_final_full.log 2>&1
ncu -i gpurun_out/spectra_full_final.ncu-rep --page raw --csv > gpurun_out/spectra_full_final_raw.csv 2>/dev/null
ncu -i gpurun_out/spectra_full_final.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/spectra_full_final_source.csv 2>/dev/null
gzip -f gpurun_out/spectra_full_final_source.csv
echo done
