set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.log 2>&1
python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu_r02b.log 2>&1
python bench.py > gpurun_out/bench_c4_r02.json 2> gpurun_out/bench_c4_r02.err
python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_r02.json 2>&1
python bench.py --workload c5 --steps 3 --warmup 3 > gpurun_out/bench_c5_r02.json 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lorenz_chain_seg_kernel -s 1 -c 1 -o gpurun_out/chain_full_r02 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu2.log 2>&1 && \
ncu --set full --import-source on -k regex:lorenz_chain_seg_kernel -s 1 -c 1 -o gpurun_out/chain_full_baseclock_r02 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
echo done
