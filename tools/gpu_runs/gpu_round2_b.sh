set -x
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > gpurun_out/pytest_gpu_r02c.log 2>&1
./tools/rk4_occupancy > gpurun_out/rk4_occupancy_r02.json 2> gpurun_out/rk4_occupancy.err
python bench.py --workload c5 --steps 3 --warmup 3 > gpurun_out/bench_c5_r02b.json 2>&1
python bench.py --workload c3 --integrator rk4fma --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_fma_r02.json 2>&1
python tools/spectra.py --sizes 4096 --reps 5 --oracle-side 0 --fig 256 > gpurun_out/spectra_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/spectra_launches_r02.csv python tools/spectra.py --sizes 4096 --reps 2 --oracle-side 0 --fig 256 > gpurun_out/ncu_s1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fft_pass -c 5 -o gpurun_out/spectra_full_r02 python tools/spectra.py --sizes 4096 --reps 2 --oracle-side 0 --fig 256 > gpurun_out/ncu_s2.log 2>&1
echo done
