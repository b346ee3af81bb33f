# validation after the round's spectra follow-up: smoke, every GPU test, the C4 bench line, the spectra
# timings and launch list of the final library
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final3.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu_final3.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final3_c4.json 2> gpurun_out/bench_final3_c4.err
timeout 600 python tools/spectra.py --sizes 256 1024 2048 4096 --reps 20 > gpurun_out/spectra_final3.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/spectra_launches_final3.csv python tools/spectra.py --sizes 2048 4096 --reps 1 --oracle-side 0 --fig 0 > gpurun_out/ncu_final3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fft_col_tma|byte_sum" -c 2 -o gpurun_out/spectra_full_final3 \
    python tools/spectra.py --sizes 4096 --reps 1 --oracle-side 0 --fig 0 > gpurun_out/ncu_final3_full.log 2>&1
echo done
