# final validation of the round (after the squaring fused into the TMA column pass): smoke, every GPU test,
# the C4 bench line, the spectra timings and launch list
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final7.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu_final7.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final7_c4.json 2> gpurun_out/bench_final7_c4.err
timeout 600 python tools/spectra.py --sizes 256 1024 2048 4096 --reps 20 > gpurun_out/spectra_final7.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/spectra_launches_final7.csv python tools/spectra.py --sizes 2048 4096 --reps 1 --oracle-side 0 --fig 0 > gpurun_out/ncu_final7.log 2>&1
echo done
