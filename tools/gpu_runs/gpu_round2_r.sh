set -x
python bench.py --workload c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c3_r02.csv python bench.py --workload c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c3a.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lorenz_chain_seg_kernel -s 1 -c 1 -o gpurun_out/c3_full_r02 python bench.py --workload c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c3b.log 2>&1
echo done
